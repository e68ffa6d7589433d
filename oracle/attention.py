"""Multi-head self-attention, Eq. (1) of the paper (§III-A):

    Attention(Q, K, V) = softmax(Q K^T / sqrt(d_k)) V,   d_k = head dimension

computed per sequence on the padded batch with the padding keys masked out, which is
what the unpadded FMHA must reproduce on valid tokens (§IV-A-1).
ORACLE: test infrastructure only.  numpy, float64, one (sequence, head) at a time.

Readings: R1 scale is a parameter (default 1/sqrt(d_k)); R2 no
cross-sequence attention; R3 padded query rows output 0; R4 inverted dropout on the
post-softmax probabilities, LSE taken before dropout; R5 Philox mask (oracle.philox).

Forward, for each sequence b (length L) and head h:
    S   = scale * Q K^T                      (S x S, S = max_seq_len)
    S[:, j >= L] = -inf                      (padding keys masked)
    m_i = max_j S_ij ;  l_i = sum_j exp(S_ij - m_i)
    P   = exp(S - m) / l ;   LSE_i = m_i + log l_i
    Pd  = P * M * r         if p > 0 else P  (M = keep mask, r = 1 / (1 - floor(256 p) / 256), R5)
    O   = Pd V ;  O[i >= L] = 0
Backward (chain rule through the same steps):
    dV  = Pd^T dO ;  dPd = dO V^T ;  dP = dPd * M * r
    Delta_i = sum_j P_ij dP_ij  (= sum_d dO_id O_id)
    dS  = P * (dP - Delta)      ;  dQ = scale * dS K ;  dK = scale * dS^T Q

Pins (tests/test_oracle_attention.py): closed forms (one token -> V row; identical keys
-> mean of V; d_k=1 two-token hand case; Q=0 -> mean of V), padded == unpadded,
softmax rows sum to 1, no leakage from padding, torch CPU fp64
scaled_dot_product_attention (an independent library routine) forward and autograd
backward, central finite differences, sum_j dK_j = 0, sum dV = sum dO at p=0, L=1 ->
dQ = dK = 0.  Parity pinned.
"""
from __future__ import annotations

import math

import numpy as np

from . import philox, varlen


def _keep_full(keep_block, L: int, S: int) -> np.ndarray:
    full = np.ones((S, S), dtype=bool)
    if keep_block is not None:
        full[:L, :L] = keep_block
    return full


def mha_fwd_padded(q, k, v, lengths, scale, p=0.0, keep=None):
    """Padded-masked forward.

    q, k, v: [B, S, H, D] float64.  keep: None or callable keep(b, h) -> [L, L] bool.
    Returns O [B, S, H, D] and LSE [B, H, S] (LSE of padded rows left at 0).
    """
    B, S, H, D = q.shape
    O = np.zeros_like(q)
    LSE = np.zeros((B, H, S))
    for b in range(B):
        L = int(lengths[b])
        for h in range(H):
            Sm = scale * (q[b, :, h, :] @ k[b, :, h, :].T)
            Sm[:, L:] = -np.inf
            m = np.max(Sm, axis=1, keepdims=True)
            e = np.exp(Sm - m)
            l = np.sum(e, axis=1, keepdims=True)
            P = e / l
            LSE[b, h, :L] = (m + np.log(l))[:L, 0]
            if p > 0.0:
                M = _keep_full(keep(b, h), L, S)
                P = P * M * philox.dropout_scale(p)
            Ob = P @ v[b, :, h, :]
            Ob[L:, :] = 0.0
            O[b, :, h, :] = Ob
    return O, LSE


def mha_bwd_padded(q, k, v, dout, lengths, scale, p=0.0, keep=None):
    """Analytic backward of mha_fwd_padded.  Returns dQ, dK, dV [B, S, H, D]."""
    B, S, H, D = q.shape
    dQ = np.zeros_like(q)
    dK = np.zeros_like(k)
    dV = np.zeros_like(v)
    for b in range(B):
        L = int(lengths[b])
        for h in range(H):
            Sm = scale * (q[b, :, h, :] @ k[b, :, h, :].T)
            Sm[:, L:] = -np.inf
            m = np.max(Sm, axis=1, keepdims=True)
            e = np.exp(Sm - m)
            P = e / np.sum(e, axis=1, keepdims=True)
            P[L:, :] = 0.0                      # padded query rows produce nothing (R3)
            if p > 0.0:
                M = _keep_full(keep(b, h), L, S)
                Pd = P * M * philox.dropout_scale(p)
            else:
                M = None
                Pd = P
            dO = dout[b, :, h, :].copy()
            dO[L:, :] = 0.0
            dV[b, :, h, :] = Pd.T @ dO
            dPd = dO @ v[b, :, h, :].T
            dP = dPd * M * philox.dropout_scale(p) if p > 0.0 else dPd
            Delta = np.sum(P * dP, axis=1, keepdims=True)
            dS = P * (dP - Delta)
            dQ[b, :, h, :] = scale * (dS @ k[b, :, h, :])
            dK[b, :, h, :] = scale * (dS.T @ q[b, :, h, :])
    return dQ, dK, dV


def mha_fwd_unpadded(q, k, v, offsets, scale):
    """Unpadded form: each sequence slice of the packed [T, H, D] tensors attends
    only within itself; no masks exist because no padding exists.  Returns O [T,H,D]."""
    T, H, D = q.shape
    O = np.zeros_like(q)
    for b in range(len(offsets) - 1):
        s, e_ = int(offsets[b]), int(offsets[b + 1])
        for h in range(H):
            Sm = scale * (q[s:e_, h, :] @ k[s:e_, h, :].T)
            w = np.exp(Sm - Sm.max(axis=1, keepdims=True))
            w = w / w.sum(axis=1, keepdims=True)
            O[s:e_, h, :] = w @ v[s:e_, h, :]
    return O


def attention_probs(q, k, lengths, scale):
    """Softmax rows P [B, H, S, S] (masked columns 0) -- used by the row-sum pin."""
    B, S, H, D = q.shape
    out = np.zeros((B, H, S, S))
    for b in range(B):
        L = int(lengths[b])
        for h in range(H):
            Sm = scale * (q[b, :, h, :] @ k[b, :, h, :].T)
            Sm[:, L:] = -np.inf
            e = np.exp(Sm - Sm.max(axis=1, keepdims=True))
            out[b, h] = e / e.sum(axis=1, keepdims=True)
    return out


def _keep_fn(offsets, seed, offset, p, t_base=0):
    def keep(b, h):
        L = int(offsets[b + 1] - offsets[b])
        return philox.keep_mask_block(seed, offset, t_base + int(offsets[b]), L, h, p)
    return keep


def varlen_fwd(qkv, offsets, max_seq_len, scale, p=0.0, seed=0, offset=0, t_base=0):
    """The library's forward contract on packed inputs, via pad -> padded-masked -> unpad.

    qkv: [T, 3, H, D] (any float dtype; computed in float64).  offsets = batch_offset.
    t_base: packed-row index of qkv[0] in the full batch (dropout coordinates are
    absolute rows, R5), so a slice of sequences can be checked on its own.
    Returns O [T, H, D] and LSE [H, T] (natural log), both float64.
    """
    qkv = np.asarray(qkv, dtype=np.float64)
    lengths = np.diff(np.asarray(offsets))
    padded = varlen.pad(qkv, offsets, max_seq_len, 0.0)          # [B, S, 3, H, D]
    q, k, v = padded[:, :, 0], padded[:, :, 1], padded[:, :, 2]
    keep = _keep_fn(offsets, seed, offset, p, t_base) if p > 0.0 else None
    O, LSE = mha_fwd_padded(q, k, v, lengths, scale, p, keep)
    O_packed = varlen.unpad(O, lengths)
    LSE_packed = varlen.unpad(np.transpose(LSE, (0, 2, 1)), lengths)  # [T, H]
    return O_packed, np.ascontiguousarray(LSE_packed.T)


def varlen_bwd(qkv, dout, offsets, max_seq_len, scale, p=0.0, seed=0, offset=0, t_base=0):
    """Backward contract on packed inputs (t_base as in varlen_fwd).  Returns dqkv
    [T, 3, H, D] float64."""
    qkv = np.asarray(qkv, dtype=np.float64)
    dout = np.asarray(dout, dtype=np.float64)
    lengths = np.diff(np.asarray(offsets))
    padded = varlen.pad(qkv, offsets, max_seq_len, 0.0)
    dO = varlen.pad(dout, offsets, max_seq_len, 0.0)
    q, k, v = padded[:, :, 0], padded[:, :, 1], padded[:, :, 2]
    keep = _keep_fn(offsets, seed, offset, p, t_base) if p > 0.0 else None
    dQ, dK, dV = mha_bwd_padded(q, k, v, dO, lengths, scale, p, keep)
    d = np.stack([dQ, dK, dV], axis=2)                          # [B, S, 3, H, D]
    return varlen.unpad(d, lengths)


def default_scale(head_dim: int) -> float:
    """1/sqrt(d_k) (reading R1)."""
    return 1.0 / math.sqrt(head_dim)
