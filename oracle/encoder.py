"""Unpadded encoder attention sub-layer (BASELINE config 4) -- forward
and backward.  ORACLE: test infrastructure only.  numpy fp64.

    qkv = x Wqkv^T + bqkv                (Linear)
    ctx = Eq. (1) per sequence and head  (oracle.attention; dropout R4/R5)
    a   = ctx Wo^T + bo                  (Linear)
    y   = LayerNorm(x + dropout(a))      (oracle.dal; R21)
backward by the chain rule in the reverse order; the residual gradient of x (the LayerNorm
input's branch) is added to the QKV projection's data gradient (P:416 computes that sum
through the GEMM's beta -- the value is the same).

round_bf16=True rounds every tensor the device stores in bf16 (qkv, ctx, a, and the
gradients da, dres, dctx, dqkv) to bf16 (RNE) at the point it is stored -- the storage
precision of reading R6 ("O2 mixed precision"), not a change of the arithmetic, which stays
fp64.  Without it the oracle is the exact fp64 composition.

Pins (tests/test_oracle_encoder.py): torch CPU fp64 autograd of the same composition built
from torch's own scaled_dot_product_attention and layer_norm (independent routines), with
the hidden-dropout mask applied by hand.  Parity pinned.
"""
from __future__ import annotations

import numpy as np
import torch

from . import attention as oatt
from . import dal as odal


def _bf16(x: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).double().numpy()


def encoder_attn_fwd(x, off, S, w_qkv, b_qkv, w_o, b_o, gamma, beta, heads, p_attn=0.0, p_hidden=0.0, eps=1e-12,
                     seed=0, offset=0, round_bf16=False):
    """Returns (y, saved) with saved = dict(qkv, ctx, lse, a, mean, rstd), fp64."""
    rnd = _bf16 if round_bf16 else (lambda t: t)
    x = np.asarray(x, np.float64)
    T, hid = x.shape
    D = hid // heads
    qkv = rnd(x @ np.asarray(w_qkv, np.float64).T + np.asarray(b_qkv, np.float64))
    O, LSE = oatt.varlen_fwd(qkv.reshape(T, 3, heads, D), off, S, 1.0 / np.sqrt(D), p_attn, seed, offset)
    ctx = rnd(O.reshape(T, hid))
    a = rnd(ctx @ np.asarray(w_o, np.float64).T + np.asarray(b_o, np.float64))
    y, mean, rstd = odal.dal_fwd(a, x, gamma, beta, p_hidden, eps, seed, offset)
    return y, {"qkv": qkv, "ctx": ctx, "lse": LSE, "a": a, "mean": mean, "rstd": rstd}


def encoder_attn_bwd(dy, x, off, S, w_qkv, w_o, gamma, saved, heads, p_attn=0.0, p_hidden=0.0, eps=1e-12, seed=0,
                     offset=0, round_bf16=False):
    """Returns dict dx, dw_qkv, db_qkv, dw_o, db_o, dgamma, dbeta (fp64)."""
    rnd = _bf16 if round_bf16 else (lambda t: t)
    x = np.asarray(x, np.float64)
    T, hid = x.shape
    D = hid // heads
    w_qkv = np.asarray(w_qkv, np.float64)
    w_o = np.asarray(w_o, np.float64)
    da, dres, dgamma, dbeta = odal.dal_bwd(dy, saved["a"], x, gamma, p_hidden, eps, seed, offset)
    da, dres = rnd(da), rnd(dres)
    dw_o = da.T @ saved["ctx"]
    db_o = da.sum(axis=0)
    dctx = rnd(da @ w_o)
    dqkv = oatt.varlen_bwd(saved["qkv"].reshape(T, 3, heads, D), dctx.reshape(T, heads, D), off, S,
                           1.0 / np.sqrt(D), p_attn, seed, offset)
    dqkv = rnd(dqkv.reshape(T, 3 * hid))
    return {"dx": dqkv @ w_qkv + dres, "dw_qkv": dqkv.T @ x, "db_qkv": dqkv.sum(axis=0), "dw_o": dw_o, "db_o": db_o,
            "dgamma": dgamma, "dbeta": dbeta}
