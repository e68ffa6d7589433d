"""Thin Python binding of include/ub.h -- argument marshalling only.

Every step of the hot path runs inside libub.so (hand-written sm_100a CUDA + NCCL);
PyTorch only supplies device memory, streams and process groups.  Names follow the C
ABI (and the paper's vocabulary: batch_offset == cu_seqlens).
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from ._lib import (EncoderParams, UB_BAL_EXACT_SMALL, UB_BAL_LPT, UB_BAL_PAPER, UB_BAL_SNAKE, UB_BAL_STAY, UB_BF16, UB_FP32,
                   UB_IPC_HANDLE_BYTES, FmhaParams, check, lib)

BAL_MODES = {"paper": UB_BAL_PAPER, "snake": UB_BAL_SNAKE, "exact_small": UB_BAL_EXACT_SMALL, "lpt": UB_BAL_LPT,
             "stay": UB_BAL_STAY}
UB_BAL_LOCALITY = 0x100


def _mode(mode: str) -> int:
    """'paper', 'snake', 'lpt', 'exact_small', each optionally '+locality' (UB_BAL_LOCALITY)."""
    base, _, flag = mode.partition("+")
    if flag not in ("", "locality"):
        raise ValueError(f"bad balance mode {mode!r}")
    return BAL_MODES[base] | (UB_BAL_LOCALITY if flag else 0)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _np_ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


_ws_cache = {}


def _workspace(nbytes: int, device, tag: str) -> torch.Tensor:
    key = (tag, str(device))
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = buf
    return buf


def version() -> str:
    return lib().ub_version().decode()


PROF_FWD, PROF_BWD, PROF_PAD, PROF_UNPAD, PROF_DAL_FWD, PROF_DAL_BWD = 0, 1, 2, 3, 4, 5


def profile_events(kernel_id: int, start=None, stop=None):
    """Record torch.cuda.Event `start`/`stop` around every launch of one internal kernel
    (0 fwd main, 1 bwd main, 2 pad, 3 unpad, 4 DAL fwd, 5 DAL bwd incl. its reduction); None clears.  Bench/profiling hook."""
    for e in (start, stop):
        if e is not None and not e.cuda_event:
            e.record()            # torch creates the cudaEvent_t lazily on first record
    check(lib().ub_profile_events(int(kernel_id), start.cuda_event if start is not None else None,
                                  stop.cuda_event if stop is not None else None))


def dropout_effective_p(p: float, bits: int = 8) -> float:
    """The drop rate the kernels apply for a requested p: floor(2^bits p) / 2^bits (8-bit
    attention decisions, R5; 16-bit Dropout_Add_LayerNorm decisions, R21)."""
    return float(lib().ub_dropout_effective_p(float(p), int(bits)))


# ------------------------------------------------------------------ batch_offset
def cu_seqlens(lengths, max_seqlen: int) -> np.ndarray:
    """Host prefix sum with validation; returns int32 [B+1]."""
    L = np.ascontiguousarray(np.asarray(lengths, dtype=np.int32))
    out = np.zeros(L.size + 1, dtype=np.int32)
    check(lib().ub_cu_seqlens(_np_ptr(L), L.size, int(max_seqlen), _np_ptr(out)))
    return out


def lengths_from_mask(mask) -> np.ndarray:
    m = np.ascontiguousarray(np.asarray(mask, dtype=np.int32))
    out = np.zeros(m.shape[0], dtype=np.int32)
    check(lib().ub_lengths_from_mask(_np_ptr(m), m.shape[0], m.shape[1], _np_ptr(out)))
    return out


# ------------------------------------------------------------------ unpad / pad
def unpad(padded: torch.Tensor, cu: torch.Tensor, T: int, out: torch.Tensor | None = None, stream=None):
    """Gather: padded [B, S, *row] -> packed [T, *row]."""
    B, S = padded.shape[0], padded.shape[1]
    row_bytes = padded[0, 0].numel() * padded.element_size()
    if out is None:
        out = torch.empty((T,) + tuple(padded.shape[2:]), dtype=padded.dtype, device=padded.device)
    check(lib().ub_unpad(_ptr(padded), _ptr(out), _ptr(cu), B, S, int(T), row_bytes, _stream(stream)))
    return out


def pad(packed: torch.Tensor, cu: torch.Tensor, B: int, S: int, pad_row: torch.Tensor | None = None,
        out: torch.Tensor | None = None, stream=None):
    """Scatter: packed [T, *row] -> padded [B, S, *row] (pad_row or zeros elsewhere)."""
    T = packed.shape[0]
    row_bytes = packed[0].numel() * packed.element_size() if T > 0 else \
        int(np.prod(packed.shape[1:])) * packed.element_size()
    if out is None:
        out = torch.empty((B, S) + tuple(packed.shape[1:]), dtype=packed.dtype, device=packed.device)
    check(lib().ub_pad(_ptr(packed), _ptr(out), _ptr(cu), B, S, int(T), row_bytes, _ptr(pad_row), _stream(stream)))
    return out


# ------------------------------------------------------------------ varlen FMHA
def fmha_params(B, T, max_seqlen, heads, head_dim, dtype, scale=None, p_dropout=0.0, seed=0, offset=0,
                num_ctas=0, dropout_mask=None, schedule=None):
    return FmhaParams(B=int(B), T=int(T), max_seqlen=int(max_seqlen), heads=int(heads), head_dim=int(head_dim),
                      scale=float(scale if scale is not None else 1.0 / math.sqrt(head_dim)),
                      p_dropout=float(p_dropout), seed=int(seed), offset=int(offset),
                      dtype=UB_BF16 if dtype == torch.bfloat16 else UB_FP32, num_ctas=int(num_ctas),
                      dropout_mask=(dropout_mask.data_ptr() if dropout_mask is not None else None),
                      schedule=(schedule.data_ptr() if schedule is not None else None))


def fmha_schedule(lengths, heads: int, max_seqlen: int, grid: int, is_bwd: bool, out=None) -> np.ndarray:
    """ub_fmha_schedule: the host LPT schedule (int32 numpy array) of one direction's work items
    for a batch with these lengths and a persistent grid of `grid` CTAs; copy it to the device and
    pass it as schedule=... .  out: a preallocated int32 numpy array (e.g. a pinned tensor's view)."""
    a = np.ascontiguousarray(np.asarray(lengths, dtype=np.int32).reshape(-1))
    n = int(lib().ub_fmha_schedule_ints(a.size, heads, max_seqlen, grid, 1 if is_bwd else 0))
    if out is None:
        out = np.zeros(n, dtype=np.int32)
    assert out.dtype == np.int32 and out.flags["C_CONTIGUOUS"]       # size: checked by the library
    check(lib().ub_fmha_schedule(_np_ptr(a), a.size, heads, max_seqlen, grid, 1 if is_bwd else 0, _np_ptr(out),
                                 out.size))
    return out


def dropout_mask(cu: torch.Tensor, T: int, heads: int, max_seqlen: int, p_dropout: float, seed=0, offset=0,
                 out=None, stream=None):
    """R5's keep bits for a batch (ub_dropout_mask): a uint8 CUDA tensor to pass to the forward
    and the backward (dropout_mask=...), so neither regenerates it.  Query-major words first,
    then key-major (see include/ub.h)."""
    B = cu.numel() - 1
    prm = fmha_params(B, T, max_seqlen, heads, 64, torch.bfloat16, None, p_dropout, seed, offset)
    n = lib().ub_dropout_mask_bytes(C.byref(prm))
    if out is None:
        out = torch.empty(n, dtype=torch.uint8, device=cu.device)
    assert out.numel() >= n
    check(lib().ub_dropout_mask(C.byref(prm), _ptr(cu), _ptr(out), _stream(stream)))
    return out


def varlen_fmha_fwd(qkv: torch.Tensor, cu: torch.Tensor, max_seqlen: int, scale=None, p_dropout=0.0, seed=0,
                    offset=0, out=None, lse=None, stream=None, num_ctas=0, padded=None, dropout_mask=None,
                    schedule=None):
    """Eq. (1) over packed qkv [T, 3, H, D]; returns (out [T,H,D], lse [H,T] fp32).
    padded: optional [B, S, H, D] tensor that the forward also fills with O in the padded
    layout, zeros past each length (a9 fused into the epilogue, ub_varlen_fmha_fwd_pad)."""
    T, three, H, D = qkv.shape
    assert three == 3
    B = cu.numel() - 1
    prm = fmha_params(B, T, max_seqlen, H, D, qkv.dtype, scale, p_dropout, seed, offset, num_ctas, dropout_mask,
                      schedule)
    if out is None:
        out = torch.empty((T, H, D), dtype=qkv.dtype, device=qkv.device)
    if lse is None:
        lse = torch.empty((H, T), dtype=torch.float32, device=qkv.device)
    ws = _workspace(lib().ub_fmha_workspace_bytes(C.byref(prm), 0), qkv.device, "fmha_fwd")
    if padded is not None:
        check(lib().ub_varlen_fmha_fwd_pad(C.byref(prm), _ptr(qkv), _ptr(cu), _ptr(out), _ptr(lse), _ptr(padded),
                                           int(padded.shape[1]), _ptr(ws), _stream(stream)))
    else:
        check(lib().ub_varlen_fmha_fwd(C.byref(prm), _ptr(qkv), _ptr(cu), _ptr(out), _ptr(lse), _ptr(ws),
                                       _stream(stream)))
    return out, lse


def varlen_fmha_bwd(qkv, out, lse, dout, cu, max_seqlen: int, scale=None, p_dropout=0.0, seed=0, offset=0,
                    dqkv=None, stream=None, num_ctas=0, dropout_mask=None, schedule=None):
    """Backward of varlen_fmha_fwd; returns dqkv [T, 3, H, D]."""
    T, _, H, D = qkv.shape
    B = cu.numel() - 1
    prm = fmha_params(B, T, max_seqlen, H, D, qkv.dtype, scale, p_dropout, seed, offset, num_ctas, dropout_mask,
                      schedule)
    if dqkv is None:
        dqkv = torch.empty_like(qkv)
    ws = _workspace(lib().ub_fmha_workspace_bytes(C.byref(prm), 1), qkv.device, "fmha_bwd")
    check(lib().ub_varlen_fmha_bwd(C.byref(prm), _ptr(qkv), _ptr(out), _ptr(lse), _ptr(dout), _ptr(cu),
                                   _ptr(dqkv), _ptr(ws), _stream(stream)))
    return dqkv


# ------------------------------------------------------------------ pre-marshalled calls (hot loops)
class BoundFmha:
    """The varlen FMHA forward (+ fused pad) and backward on fixed buffers, with every pointer,
    the stream and the parameter struct marshalled once: a call only updates T (and the
    dropout seed) and invokes the C entry point.  Same ABI calls as varlen_fmha_fwd / _bwd --
    argument marshalling hoisted out of a training loop whose buffers do not change.
    qkv / dout / out / dqkv: capacity-sized tensors whose first T rows are used; lse: a buffer
    of at least H * T floats, used as a dense [H, T] array."""

    def __init__(self, qkv, cu, max_seqlen, out, lse, dout=None, dqkv=None, scale=None, p_dropout=0.0, seed=0,
                 offset=0, stream=None, num_ctas=0, padded=None, dropout_mask=None):
        cap, three, H, D = qkv.shape
        B = cu.numel() - 1
        self.prm = fmha_params(B, cap, max_seqlen, H, D, qkv.dtype, scale, p_dropout, seed, offset, num_ctas,
                               dropout_mask)
        self._p = C.byref(self.prm)
        L = lib()
        ws_f = _workspace(L.ub_fmha_workspace_bytes(self._p, 0), qkv.device, "fmha_fwd")
        ws_b = _workspace(L.ub_fmha_workspace_bytes(self._p, 1), qkv.device, "fmha_bwd")
        self._keep = (qkv, cu, out, lse, dout, dqkv, padded, ws_f, ws_b, dropout_mask)   # keep the buffers alive
        st = _stream(stream)
        if padded is not None:
            self._fwd = L.ub_varlen_fmha_fwd_pad
            self._fwd_args = (self._p, _ptr(qkv), _ptr(cu), _ptr(out), _ptr(lse), _ptr(padded), int(padded.shape[1]),
                              _ptr(ws_f), st)
        else:
            self._fwd = L.ub_varlen_fmha_fwd
            self._fwd_args = (self._p, _ptr(qkv), _ptr(cu), _ptr(out), _ptr(lse), _ptr(ws_f), st)
        self._bwd = L.ub_varlen_fmha_bwd
        self._bwd_args = (self._p, _ptr(qkv), _ptr(out), _ptr(lse), _ptr(dout), _ptr(cu), _ptr(dqkv), _ptr(ws_b), st)
        self.cap = cap
        self._sched = (None, None)

    def _set(self, T, seed):
        assert 0 < T <= self.cap
        self.prm.T = T
        if seed is not None:
            self.prm.seed = seed

    def set_schedules(self, fwd_sched=None, bwd_sched=None):
        """Device int32 tensors from fmha_schedule (fwd / bwd direction) for the next calls, or
        None for the kernels' snake deal (same results)."""
        self._sched = (fwd_sched.data_ptr() if fwd_sched is not None else None,
                       bwd_sched.data_ptr() if bwd_sched is not None else None)

    def fwd(self, T: int, seed=None):
        self._set(T, seed)
        self.prm.schedule = self._sched[0]
        st = self._fwd(*self._fwd_args)
        if st:
            check(st)

    def bwd(self, T: int, seed=None):
        self._set(T, seed)
        self.prm.schedule = self._sched[1]
        st = self._bwd(*self._bwd_args)
        if st:
            check(st)


class BoundDropoutMask:
    """ub_dropout_mask on a fixed output buffer, marshalled once: call with (T, seed).  Size
    the buffer for the largest T (dropout_mask_bytes(cap, ...))."""

    def __init__(self, cu, cap, heads, max_seqlen, p_dropout, out, offset=0, stream=None, overlap_previous=False):
        """overlap_previous: UB_MASK_OVERLAP_PREVIOUS (the caller guarantees the previous kernel on
        the stream neither writes cu nor touches `out`)."""
        B = cu.numel() - 1
        self.prm = fmha_params(B, cap, max_seqlen, heads, 64, torch.bfloat16, None, p_dropout, 0, offset)
        assert out.numel() >= lib().ub_dropout_mask_bytes(C.byref(self.prm))
        self._keep = (cu, out)
        self._args = (C.byref(self.prm), _ptr(cu), _ptr(out), 1 if overlap_previous else 0, _stream(stream))
        self._f = lib().ub_dropout_mask_ex
        self.cap = cap

    def __call__(self, T: int, seed: int):
        assert 0 < T <= self.cap
        self.prm.T = T
        self.prm.seed = seed
        st = self._f(*self._args)
        if st:
            check(st)


def dropout_mask_bytes(T: int, heads: int, max_seqlen: int) -> int:
    prm = fmha_params(1, T, max_seqlen, heads, 64, torch.bfloat16, None, 0.1)
    return int(lib().ub_dropout_mask_bytes(C.byref(prm)))


class BoundUnpad:
    """ub_unpad on fixed buffers (padded [B, S, *row] -> out), marshalled once; call with T."""

    def __init__(self, padded, cu, out, stream=None):
        self._keep = (padded, cu, out)
        B, S = padded.shape[0], padded.shape[1]
        row = padded[0, 0].numel() * padded.element_size()
        self._args = [_ptr(padded), _ptr(out), _ptr(cu), B, S, 0, row, _stream(stream)]
        self._f = lib().ub_unpad

    def __call__(self, T: int):
        a = self._args
        a[5] = int(T)
        st = self._f(*a)
        if st:
            check(st)


# ------------------------------------------------------------------ Dropout_Add_LayerNorm
def dal_fwd(a: torch.Tensor, res: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, p_dropout=0.0, eps=1e-12,
            seed=0, offset=0, out=None, mean=None, rstd=None, stream=None):
    """y = LayerNorm(res + dropout(a)) * gamma + beta over packed rows (R21).
    a, res [T, E] bf16; gamma, beta [E] bf16.  Returns (y [T, E] bf16, mean [T], rstd [T] fp32)."""
    T, E = a.shape
    y = out if out is not None else torch.empty_like(a)
    mean = mean if mean is not None else torch.empty(T, dtype=torch.float32, device=a.device)
    rstd = rstd if rstd is not None else torch.empty(T, dtype=torch.float32, device=a.device)
    check(lib().ub_dal_fwd(_ptr(a), _ptr(res), _ptr(gamma), _ptr(beta), int(T), int(E), float(p_dropout), float(eps),
                           int(seed), int(offset), _ptr(y), _ptr(mean), _ptr(rstd), _stream(stream)))
    return y, mean, rstd


def dal_bwd(dy: torch.Tensor, a: torch.Tensor, res: torch.Tensor, gamma: torch.Tensor, mean: torch.Tensor,
            rstd: torch.Tensor, p_dropout=0.0, seed=0, offset=0, stream=None):
    """Backward of dal_fwd: returns (da, dres [T, E] bf16, dgamma, dbeta [E] fp32)."""
    T, E = a.shape
    da, dres = torch.empty_like(a), torch.empty_like(a)
    dgamma = torch.empty(E, dtype=torch.float32, device=a.device)
    dbeta = torch.empty(E, dtype=torch.float32, device=a.device)
    ws = _workspace(lib().ub_dal_bwd_workspace_bytes(int(T), int(E)), a.device, "dal_bwd")
    check(lib().ub_dal_bwd(_ptr(dy), _ptr(a), _ptr(res), _ptr(gamma), _ptr(mean), _ptr(rstd), int(T), int(E),
                           float(p_dropout), int(seed), int(offset), _ptr(da), _ptr(dres), _ptr(dgamma), _ptr(dbeta),
                           _ptr(ws), _stream(stream)))
    return da, dres, dgamma, dbeta


# ------------------------------------------------------------------ embedding (NEXT-4)
def embedding_fwd(ids, pos, seg, w_word, w_pos, w_type, out=None, stream=None):
    """out[t] = W_word[ids[t]] + W_pos[pos[t]] + W_type[seg[t]] on packed tokens."""
    T, E = ids.numel(), w_word.shape[1]
    out = out if out is not None else torch.empty((T, E), dtype=w_word.dtype, device=w_word.device)
    check(lib().ub_embedding_fwd(_ptr(ids), _ptr(pos), _ptr(seg), _ptr(w_word), _ptr(w_pos), _ptr(w_type), int(T),
                                 int(E), _ptr(out), _stream(stream)))
    return out


def embedding_bwd(dout, ids, pos, seg, dw_word, dw_pos, dw_type, stream=None):
    """Accumulate dout rows into the (zeroed) fp32 or bf16 table gradients."""
    T, E = dout.shape
    gd = UB_FP32 if dw_word.dtype == torch.float32 else UB_BF16
    check(lib().ub_embedding_bwd(_ptr(dout), _ptr(ids), _ptr(pos), _ptr(seg), int(T), int(E), int(dw_type.shape[0]),
                                 gd, _ptr(dw_word), _ptr(dw_pos), _ptr(dw_type), _stream(stream)))
    return dw_word, dw_pos, dw_type


# ------------------------------------------------------------------ Linear (cuBLASLt) and the encoder sub-layer
def linear_fwd(x: torch.Tensor, W: torch.Tensor, b: torch.Tensor | None = None, out=None, stream=None):
    """y[T, N] = x[T, K] W[N, K]^T + b."""
    T, K = x.shape
    N = W.shape[0]
    y = out if out is not None else torch.empty((T, N), dtype=x.dtype, device=x.device)
    ws = _workspace(lib().ub_linear_workspace_bytes(), x.device, "linear")
    check(lib().ub_linear_fwd(_ptr(x), _ptr(W), _ptr(b), int(T), int(K), int(N), _ptr(y), _ptr(ws), _stream(stream)))
    return y


def linear_bwd(dy: torch.Tensor, x: torch.Tensor, W: torch.Tensor, res_grad: torch.Tensor | None = None, stream=None):
    """(dx = dy W (+ res_grad), dW = dy^T x (fp32), db = sum_t dy (fp32)) -- P:410."""
    T, N = dy.shape
    K = W.shape[1]
    dx = torch.empty((T, K), dtype=dy.dtype, device=dy.device)
    dW = torch.empty((N, K), dtype=torch.float32, device=dy.device)
    db = torch.empty(N, dtype=torch.float32, device=dy.device)
    ws = _workspace(lib().ub_linear_workspace_bytes(), dy.device, "linear")
    check(lib().ub_linear_bwd(_ptr(dy), _ptr(x), _ptr(W), _ptr(res_grad), int(T), int(K), int(N), _ptr(dx), _ptr(dW),
                              _ptr(db), _ptr(ws), _stream(stream)))
    return dx, dW, db


def encoder_params(B, T, max_seqlen, hidden=1024, heads=16, p_attn=0.0, p_hidden=0.0, eps=1e-12, seed=0, offset=0,
                   num_ctas=0):
    return EncoderParams(B=int(B), T=int(T), max_seqlen=int(max_seqlen), hidden=int(hidden), heads=int(heads),
                         p_attn=float(p_attn), p_hidden=float(p_hidden), eps=float(eps), seed=int(seed),
                         offset=int(offset), num_ctas=int(num_ctas))


def encoder_attn_fwd(x, cu, max_seqlen, w_qkv, b_qkv, w_o, b_o, gamma, beta, heads=16, p_attn=0.0, p_hidden=0.0,
                     eps=1e-12, seed=0, offset=0, saved=None, out=None, stream=None, num_ctas=0):
    """Unpadded encoder attention sub-layer forward (NEXT-1): returns (y, saved) where saved
    holds the activations the backward reads (qkv, ctx, lse, a, mean, rstd)."""
    T, hid = x.shape
    prm = encoder_params(cu.numel() - 1, T, max_seqlen, hid, heads, p_attn, p_hidden, eps, seed, offset, num_ctas)
    dev = x.device
    if saved is None:
        saved = {"qkv": torch.empty((T, 3 * hid), dtype=x.dtype, device=dev),
                 "ctx": torch.empty((T, hid), dtype=x.dtype, device=dev),
                 "lse": torch.empty((heads, T), dtype=torch.float32, device=dev),
                 "a": torch.empty((T, hid), dtype=x.dtype, device=dev),
                 "mean": torch.empty(T, dtype=torch.float32, device=dev),
                 "rstd": torch.empty(T, dtype=torch.float32, device=dev)}
    y = out if out is not None else torch.empty_like(x)
    ws = _workspace(lib().ub_encoder_attn_workspace_bytes(C.byref(prm), 0), dev, "encoder_fwd")
    check(lib().ub_encoder_attn_fwd(C.byref(prm), _ptr(x), _ptr(cu), _ptr(w_qkv), _ptr(b_qkv), _ptr(w_o), _ptr(b_o),
                                    _ptr(gamma), _ptr(beta), _ptr(saved["qkv"]), _ptr(saved["ctx"]), _ptr(saved["lse"]),
                                    _ptr(saved["a"]), _ptr(saved["mean"]), _ptr(saved["rstd"]), _ptr(y), _ptr(ws),
                                    _stream(stream)))
    return y, saved


def encoder_attn_bwd(dy, x, cu, max_seqlen, w_qkv, w_o, gamma, saved, heads=16, p_attn=0.0, p_hidden=0.0, eps=1e-12,
                     seed=0, offset=0, stream=None, num_ctas=0):
    """Backward of encoder_attn_fwd: returns dict dx, dw_qkv, db_qkv, dw_o, db_o, dgamma, dbeta."""
    T, hid = x.shape
    prm = encoder_params(cu.numel() - 1, T, max_seqlen, hid, heads, p_attn, p_hidden, eps, seed, offset, num_ctas)
    dev = x.device
    f32 = lambda *shape: torch.empty(shape, dtype=torch.float32, device=dev)
    g = {"dx": torch.empty_like(x), "dw_qkv": f32(3 * hid, hid), "db_qkv": f32(3 * hid), "dw_o": f32(hid, hid),
         "db_o": f32(hid), "dgamma": f32(hid), "dbeta": f32(hid)}
    ws = _workspace(lib().ub_encoder_attn_workspace_bytes(C.byref(prm), 1), dev, "encoder_bwd")
    check(lib().ub_encoder_attn_bwd(C.byref(prm), _ptr(x), _ptr(cu), _ptr(w_qkv), _ptr(w_o), _ptr(gamma),
                                    _ptr(saved["qkv"]), _ptr(saved["ctx"]), _ptr(saved["lse"]), _ptr(saved["a"]),
                                    _ptr(saved["mean"]), _ptr(saved["rstd"]), _ptr(dy), _ptr(g["dx"]), _ptr(g["dw_qkv"]),
                                    _ptr(g["db_qkv"]), _ptr(g["dw_o"]), _ptr(g["db_o"]), _ptr(g["dgamma"]),
                                    _ptr(g["dbeta"]), _ptr(ws), _stream(stream)))
    return g


# ------------------------------------------------------------------ balancer
def balance_plan(all_lengths, W: int, B: int, max_seqlen: int, mode: str = "paper") -> dict:
    """Host planner: perm, rank_tokens, send_samples [W*W], send_tokens [W*W]."""
    a = np.ascontiguousarray(np.asarray(all_lengths, dtype=np.int32).reshape(-1))
    perm = np.zeros(W * B, dtype=np.int32)
    rt = np.zeros(W, dtype=np.int64)
    ss = np.zeros(W * W, dtype=np.int32)
    st = np.zeros(W * W, dtype=np.int64)
    check(lib().ub_balance_plan(_np_ptr(a), W, B, int(max_seqlen), _mode(mode), _np_ptr(perm), _np_ptr(rt),
                                _np_ptr(ss), _np_ptr(st)))
    return {"perm": perm, "rank_tokens": rt, "send_samples": ss, "send_tokens": st}


def balance_relabel(all_lengths, perm, W: int, B: int):
    """Locality relabeling of a plan (R24): returns (new perm, kept tokens before, after)."""
    a = np.ascontiguousarray(np.asarray(all_lengths, dtype=np.int32).reshape(-1))
    p = np.ascontiguousarray(np.asarray(perm, dtype=np.int32)).copy()
    kb, ka = C.c_int64(0), C.c_int64(0)
    check(lib().ub_balance_relabel(_np_ptr(a), W, B, _np_ptr(p), C.byref(kb), C.byref(ka)))
    return p, int(kb.value), int(ka.value)


def balance_plan_weighted(all_lengths, W: int, B: int, max_seqlen: int, alpha: int, beta: int) -> dict:
    """Cost-aware planner (NEXT-2): LPT + swaps on alpha*L + beta*L^2; perm, rank_cost."""
    a = np.ascontiguousarray(np.asarray(all_lengths, dtype=np.int32).reshape(-1))
    perm = np.zeros(W * B, dtype=np.int32)
    rc = np.zeros(W, dtype=np.int64)
    check(lib().ub_balance_plan_weighted(_np_ptr(a), W, B, int(max_seqlen), int(alpha), int(beta), _np_ptr(perm),
                                         _np_ptr(rc)))
    return {"perm": perm, "rank_cost": rc}


def exchange_tables(all_lengths, perm, W: int, B: int, rank: int, unpack: bool):
    a = np.ascontiguousarray(np.asarray(all_lengths, dtype=np.int32).reshape(-1))
    p = np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
    tab = np.zeros(5 * B, dtype=np.int64)
    counts = np.zeros(W, dtype=np.int64)
    scounts = np.zeros(W, dtype=np.int64)
    total = np.zeros(1, dtype=np.int64)
    check(lib().ub_exchange_tables(_np_ptr(a), _np_ptr(p), W, B, rank, int(unpack), _np_ptr(tab), _np_ptr(counts),
                                   _np_ptr(scounts), _np_ptr(total)))
    return tab, counts, scounts, int(total[0])


def exchange_copy(src_tokens, dst_tokens, src_samples, dst_samples, d_tab, B, rec_bytes, srec_bytes, stream=None):
    check(lib().ub_exchange_copy(_ptr(src_tokens), _ptr(dst_tokens), _ptr(src_samples), _ptr(dst_samples),
                                 _ptr(d_tab), B, int(rec_bytes), int(srec_bytes), _stream(stream)))


# ------------------------------------------------------------------ checked mode
def set_checked(on: bool):
    """Validate device cu_seqlens before every unpad / pad / FMHA launch (syncs; tests only)."""
    check(lib().ub_set_checked(1 if on else 0))


def validate_cu_seqlens(cu: torch.Tensor, B: int, max_seqlen: int, T: int, stream=None) -> int:
    """0 valid, 1 cu[0] != 0, 2 not monotone, 3 a length > max_seqlen, 4 cu[B] > T (syncs)."""
    flag = torch.full((1,), -1, dtype=torch.int32, device=cu.device)
    check(lib().ub_validate_cu_seqlens(_ptr(cu), B, max_seqlen, int(T), _ptr(flag), _stream(stream)))
    return int(flag.item())


# ------------------------------------------------------------------ pull exchange (NEXT-3)
def ipc_export(t: torch.Tensor) -> bytes:
    """Handle (UB_IPC_HANDLE_BYTES) of the device buffer starting at t, for the other ranks."""
    buf = (C.c_uint8 * UB_IPC_HANDLE_BYTES)()
    check(lib().ub_ipc_export(_ptr(t), C.cast(buf, C.c_void_p)))
    return bytes(buf)


def ipc_import(handle: bytes):
    """Maps a peer's exported buffer: returns (device pointer, mapping base for ipc_close)."""
    raw = (C.c_uint8 * UB_IPC_HANDLE_BYTES)(*handle)
    ptr, base = C.c_void_p(), C.c_void_p()
    check(lib().ub_ipc_import(C.cast(raw, C.c_void_p), C.byref(ptr), C.byref(base)))
    return ptr.value, base.value


def ipc_close(base: int):
    check(lib().ub_ipc_close(C.c_void_p(base)))


def exchange_pull_table(all_lengths, perm, W: int, B: int, rank: int):
    """Pull table [6*B] int64 of rank `rank` (see include/ub.h) and its received records."""
    a = np.ascontiguousarray(np.asarray(all_lengths, dtype=np.int32).reshape(-1))
    p = np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
    tab = np.zeros(6 * B, dtype=np.int64)
    total = np.zeros(1, dtype=np.int64)
    check(lib().ub_exchange_pull_table(_np_ptr(a), _np_ptr(p), W, B, rank, _np_ptr(tab), _np_ptr(total)))
    return tab, int(total[0])


def exchange_pull(d_peer_tokens: torch.Tensor, d_peer_samples, d_tab: torch.Tensor, B: int, rec_bytes: int,
                  srec_bytes: int, out_tokens: torch.Tensor, out_samples=None, d_ready=None, wait_value: int = 0,
                  stream=None):
    """d_peer_tokens / d_peer_samples / d_ready: int64 CUDA tensors [W] of device pointers."""
    check(lib().ub_exchange_pull(_ptr(d_peer_tokens), _ptr(d_peer_samples), _ptr(d_ready), int(wait_value),
                                 _ptr(d_tab), B, int(rec_bytes), int(srec_bytes), _ptr(out_tokens), _ptr(out_samples),
                                 _stream(stream)))


def signal(flag: torch.Tensor, value: int, stream=None):
    """flag: a uint32 / int32 CUDA tensor element (its first element is set)."""
    check(lib().ub_signal(_ptr(flag), int(value), _stream(stream)))


def wait_flags(d_flags: torch.Tensor, value: int, stream=None):
    """d_flags: int64 CUDA tensor [n] of device pointers to uint32 flags."""
    check(lib().ub_wait_flags(_ptr(d_flags), int(d_flags.numel()), int(value), _stream(stream)))


class Comm:
    """NCCL communicator owned by the library (ub_comm).  Bootstrap: rank 0 creates the
    unique id, the caller broadcasts it over a torch.distributed group."""

    def __init__(self, world: int, rank: int, group=None):
        import torch.distributed as dist
        idbuf = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            raw = (C.c_uint8 * 128)()
            check(lib().ub_comm_unique_id(C.cast(raw, C.c_void_p)))
            idbuf = torch.tensor(list(bytes(raw)), dtype=torch.uint8)
        if world > 1:
            dev_buf = idbuf.cuda() if dist.get_backend(group) == "nccl" else idbuf
            dist.broadcast(dev_buf, 0, group=group)
            idbuf = dev_buf.cpu()
        raw = (C.c_uint8 * 128)(*idbuf.tolist())
        h = C.c_void_p()
        check(lib().ub_comm_init(C.byref(h), C.cast(raw, C.c_void_p), world, rank))
        self.handle, self.world, self.rank = h, world, rank

    def set_options(self, force_nccl: bool = False, host_profile: bool = False):
        """force_nccl: the self chunk and a one-rank all-gather also go through NCCL
        (UB_COMM_FORCE_NCCL), so the collective data plane runs on one GPU.  host_profile:
        accumulate the host time of each exchange-finish phase (UB_COMM_HOST_PROFILE)."""
        check(lib().ub_comm_set_options(self.handle, (1 if force_nccl else 0) | (2 if host_profile else 0)))

    HOST_PHASES = ("wait_lengths", "plan", "wait_staging", "tables", "pack", "nccl_p2p", "gather_cu")

    def host_profile(self) -> dict:
        """Mean host microseconds per exchange finish, per phase (ub_comm_host_profile)."""
        out = (C.c_double * 7)()
        n = C.c_int64(0)
        check(lib().ub_comm_host_profile(self.handle, out, 7, C.byref(n)))
        k = max(int(n.value), 1)
        return {"finishes": int(n.value), **{name: out[i] / k for i, name in enumerate(self.HOST_PHASES)}}

    def nccl_ops(self) -> int:
        """NCCL calls (all-gathers, sends, receives) this communicator has enqueued."""
        v = C.c_int64(0)
        check(lib().ub_comm_nccl_ops(self.handle, C.byref(v)))
        return int(v.value)

    def allgather_lengths(self, d_lengths: torch.Tensor, out=None, stream=None):
        B = d_lengths.numel()
        if out is None:
            out = torch.empty(self.world * B, dtype=torch.int32, device=d_lengths.device)
        check(lib().ub_allgather_lengths(self.handle, _ptr(d_lengths), _ptr(out), B, _stream(stream)))
        return out

    def balance_exchange(self, d_lengths, d_tokens, d_samples, capacity_tokens, max_seqlen, mode="paper",
                         out_tokens=None, out_samples=None, out_cu=None, stream=None):
        """One step of the exchange on `stream`.  Returns
        (out_tokens, out_samples, out_cu, T_out, perm)."""
        B = d_lengths.numel()
        rec = d_tokens[0].numel() * d_tokens.element_size() if d_tokens.shape[0] else \
            int(np.prod(d_tokens.shape[1:])) * d_tokens.element_size()
        srec = d_samples[0].numel() * d_samples.element_size() if d_samples is not None else 0
        dev = d_lengths.device
        if out_tokens is None:
            out_tokens = torch.empty((capacity_tokens,) + tuple(d_tokens.shape[1:]), dtype=d_tokens.dtype, device=dev)
        if out_samples is None and d_samples is not None:
            out_samples = torch.empty_like(d_samples)
        if out_cu is None:
            out_cu = torch.empty(B + 1, dtype=torch.int32, device=dev)
        ws = _workspace(lib().ub_exchange_workspace_bytes(self.world, B, capacity_tokens, rec, srec), dev,
                        f"exchange{self.rank}")
        perm = np.zeros(self.world * B, dtype=np.int32)
        T_out = C.c_int64(0)
        check(lib().ub_balance_exchange(self.handle, _mode(mode), B, int(max_seqlen), _ptr(d_lengths),
                                        _ptr(d_tokens), _ptr(d_samples), rec, srec, int(capacity_tokens),
                                        _ptr(out_tokens), _ptr(out_samples), _ptr(out_cu), _np_ptr(perm),
                                        C.byref(T_out), _ptr(ws), _stream(stream)))
        return out_tokens, out_samples, out_cu, int(T_out.value), perm

    SLOTS = 8    # UB_EXCHANGE_SLOTS

    def _ws(self, B, capacity_tokens, rec, srec, dev):
        return _workspace(lib().ub_exchange_workspace_bytes(self.world, B, capacity_tokens, rec, srec), dev,
                          f"exchange{self.rank}")

    def exchange_begin(self, slot: int, d_lengths, capacity_tokens, rec, srec, stream=None):
        """Phase 1 (no host wait): all-gather of the lengths into pinned slot `slot`."""
        ws = self._ws(d_lengths.numel(), capacity_tokens, rec, srec, d_lengths.device)
        check(lib().ub_exchange_begin(self.handle, int(slot), d_lengths.numel(), _ptr(d_lengths), _ptr(ws),
                                      _stream(stream)))

    def exchange_finish(self, slot: int, B, d_tokens, d_samples, capacity_tokens, max_seqlen, mode, out_tokens,
                        out_samples, out_cu, stream=None):
        """Phase 2: plan, pack, all-to-all-v, unpack; returns (T_out, perm)."""
        rec = int(np.prod(d_tokens.shape[1:])) * d_tokens.element_size()
        srec = int(np.prod(d_samples.shape[1:])) * d_samples.element_size() if d_samples is not None else 0
        ws = self._ws(B, capacity_tokens, rec, srec, out_tokens.device)
        perm = np.zeros(self.world * B, dtype=np.int32)
        T_out = C.c_int64(0)
        check(lib().ub_exchange_finish(self.handle, int(slot), _mode(mode), B, int(max_seqlen), _ptr(d_tokens),
                                       _ptr(d_samples), rec, srec, int(capacity_tokens), _ptr(out_tokens),
                                       _ptr(out_samples), _ptr(out_cu), _np_ptr(perm), C.byref(T_out), _ptr(ws),
                                       _stream(stream)))
        return int(T_out.value), perm

    def bind_finish(self, slot: int, B, d_tokens, d_samples, capacity_tokens, max_seqlen, mode, out_tokens,
                    out_samples, out_cu, stream=None):
        """exchange_finish on fixed buffers, marshalled once: returns a callable () -> (T_out,
        perm) (perm: this binding's own int32 array, overwritten by the next call)."""
        rec = int(np.prod(d_tokens.shape[1:])) * d_tokens.element_size()
        srec = int(np.prod(d_samples.shape[1:])) * d_samples.element_size() if d_samples is not None else 0
        ws = self._ws(B, capacity_tokens, rec, srec, out_tokens.device)
        perm = np.zeros(self.world * B, dtype=np.int32)
        T_out = C.c_int64(0)
        args = (self.handle, int(slot), _mode(mode), B, int(max_seqlen), _ptr(d_tokens), _ptr(d_samples), rec, srec,
                int(capacity_tokens), _ptr(out_tokens), _ptr(out_samples), _ptr(out_cu), _np_ptr(perm), C.byref(T_out),
                _ptr(ws), _stream(stream))
        f = lib().ub_exchange_finish
        keep = (d_tokens, d_samples, out_tokens, out_samples, out_cu, ws)

        def call():
            st = f(*args)
            if st:
                check(st)
            return T_out.value, perm
        call.keep = keep
        call.perm = perm                                 # the array each call refreshes
        return call

    def slot_lengths(self, slot: int, B: int, out=None) -> np.ndarray:
        """ub_exchange_slot_lengths: the W*B all-gathered lengths of the slot's last finished
        exchange (host int32 array)."""
        if out is None:
            out = np.zeros(self.world * B, dtype=np.int32)
        check(lib().ub_exchange_slot_lengths(self.handle, int(slot), int(B), _np_ptr(out)))
        return out

    def bind_fmha_schedule(self, slot: int, perm: np.ndarray, B: int, heads: int, max_seqlen: int, grid: int,
                           is_bwd: bool, h_sched: torch.Tensor, d_sched: torch.Tensor, stream=None):
        """ub_exchange_fmha_schedule marshalled once: a callable () that builds the FMHA schedule of
        the batch the slot's last finish delivered (its perm array: bind_finish's, refreshed by
        each call) into pinned h_sched and uploads it to d_sched on `stream`."""
        assert perm.dtype == np.int32 and h_sched.is_pinned() and d_sched.is_cuda
        args = (self.handle, int(slot), _np_ptr(perm), int(B), int(heads), int(max_seqlen), int(grid),
                1 if is_bwd else 0, _ptr(h_sched), int(h_sched.numel()), _ptr(d_sched), _stream(stream))
        f = lib().ub_exchange_fmha_schedule

        def call():
            st = f(*args)
            if st:
                check(st)
        call.keep = (perm, h_sched, d_sched)
        return call

    def bind_begin(self, slot: int, d_lengths, capacity_tokens, rec, srec, stream=None):
        """exchange_begin marshalled once: returns a callable ()."""
        ws = self._ws(d_lengths.numel(), capacity_tokens, rec, srec, d_lengths.device)
        args = (self.handle, int(slot), d_lengths.numel(), _ptr(d_lengths), _ptr(ws), _stream(stream))
        f = lib().ub_exchange_begin

        def call():
            st = f(*args)
            if st:
                check(st)
        call.keep = (d_lengths, ws)
        return call

    def close(self):
        if self.handle:
            check(lib().ub_comm_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
