"""Dropout_Add_LayerNorm (§IV-C-1 "Dropout_Add_LayerNorm Fusion") -- forward and
backward.  ORACLE: test infrastructure only.  numpy, fp64.

The paper fuses Dropout, Add and LayerNorm of the BERT encoder into one forward kernel and
two backward kernels (Table table:kernel-fusion: 3 -> 1 and 5 -> 2) and gives no formulas;
the computation is the textbook one (reading R21 in DESIGN.md):

    z    = res + a * keep * r                          (inverted dropout on the sublayer output a,
                                                        r = 1 / (1 - thr / 65536), the exact inverse
                                                        keep probability of the 16-bit decision)
    mu   = mean_j z_j,   var = mean_j (z_j - mu)^2,    rstd = 1 / sqrt(var + eps)
    y    = (z - mu) * rstd * gamma + beta

backward, with xhat = (z - mu) * rstd and g = dy * gamma:
    dz     = rstd * (g - mean_j g_j - xhat * mean_j (g_j xhat_j))
    dres   = dz,     da = dz * keep * r
    dgamma = sum_t dy * xhat,   dbeta = sum_t dy

Dropout mask (reading R21, same Philox4x32-10 as the attention mask R5, own salt):
    key = (seed mod 2^32, seed >> 32),  ctr = (col >> 3, t, 0xDA100000, offset mod 2^32)
    r16 = 16-bit half (col & 1) of word ((col & 7) >> 1);  keep <=> r16 >= floor(p * 65536)
with t the packed row index and col the column.

Pins (tests/test_oracle_dal.py): torch CPU fp64 layer_norm (an independent library routine)
and its autograd backward with the same mask applied by hand, central finite differences,
sum_j dz_j = 0 (LayerNorm is invariant to shifting z), p = 0 keeps everything, keep fraction
within the binomial bounds.  Parity pinned.
"""
from __future__ import annotations

import numpy as np

from .philox import MASK32, philox4x32_10

DAL_SALT = 0xDA100000


def dal_threshold(p: float) -> int:
    """thr = floor(p * 65536), p taken as the float32 the API carries (R21)."""
    return int(np.floor(float(np.float32(p)) * 65536.0))


def dal_dropout_scale(p: float) -> float:
    """r = 1 / (1 - thr / 65536): a 16-bit value is >= thr with probability exactly
    (65536 - thr) / 65536, so E[keep * r] = 1 (R21; the applied drop rate is thr / 65536)."""
    return 1.0 / (1.0 - dal_threshold(p) / 65536.0) if p > 0 else 1.0


def dal_keep_mask(seed: int, offset: int, T: int, E: int, p: float) -> np.ndarray:
    """keep[t, col] (bool) for rows 0..T-1, columns 0..E-1 -- R21."""
    if p <= 0.0:
        return np.ones((T, E), dtype=bool)
    thr = dal_threshold(p)                                    # 16-bit decisions (R21)
    t = np.arange(T, dtype=np.uint64)[:, None]
    c = np.arange(E, dtype=np.uint64)[None, :]
    tt, cc = np.broadcast_arrays(t, c)
    w = philox4x32_10(cc >> np.uint64(3), tt, np.full(tt.shape, DAL_SALT, np.uint64),
                      np.full(tt.shape, offset & MASK32, np.uint64),
                      np.uint64(seed & MASK32), np.uint64((seed >> 32) & MASK32))
    word = np.choose(((cc & np.uint64(7)) >> np.uint64(1)).astype(np.int64), w)
    r16 = (word >> (np.uint64(16) * (cc & np.uint64(1)))) & np.uint64(0xFFFF)
    return r16 >= np.uint64(thr)


def dal_fwd(a, res, gamma, beta, p=0.0, eps=1e-12, seed=0, offset=0):
    """Returns (y, mean, rstd) in fp64; a, res [T, E]; gamma, beta [E]."""
    a = np.asarray(a, np.float64)
    res = np.asarray(res, np.float64)
    T, E = a.shape
    keep = dal_keep_mask(seed, offset, T, E, p)
    scale = dal_dropout_scale(p)
    z = res + np.where(keep, a * scale, 0.0)
    mu = z.mean(axis=1)
    var = ((z - mu[:, None]) ** 2).mean(axis=1)
    rstd = 1.0 / np.sqrt(var + eps)
    y = (z - mu[:, None]) * rstd[:, None] * np.asarray(gamma, np.float64)[None, :] + np.asarray(beta, np.float64)[None, :]
    return y, mu, rstd


def dal_bwd(dy, a, res, gamma, p=0.0, eps=1e-12, seed=0, offset=0):
    """Returns (da, dres, dgamma, dbeta) in fp64 (mean / rstd recomputed from a, res)."""
    dy = np.asarray(dy, np.float64)
    a = np.asarray(a, np.float64)
    res = np.asarray(res, np.float64)
    gamma = np.asarray(gamma, np.float64)
    T, E = a.shape
    keep = dal_keep_mask(seed, offset, T, E, p)
    scale = dal_dropout_scale(p)
    z = res + np.where(keep, a * scale, 0.0)
    mu = z.mean(axis=1, keepdims=True)
    rstd = 1.0 / np.sqrt(((z - mu) ** 2).mean(axis=1, keepdims=True) + eps)
    xhat = (z - mu) * rstd
    g = dy * gamma[None, :]
    dz = rstd * (g - g.mean(axis=1, keepdims=True) - xhat * (g * xhat).mean(axis=1, keepdims=True))
    da = np.where(keep, dz * scale, 0.0)
    return da, dz, (dy * xhat).sum(axis=0), dy.sum(axis=0)
