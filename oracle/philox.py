"""Philox4x32-10 and the attention-dropout keep mask.  ORACLE: test infrastructure only.

The paper never describes attention dropout (reading R4 in DESIGN.md); BASELINE's
signature requires a dropout seed, so the mask convention is ours (reading R5):

    key  = (seed mod 2^32, seed >> 32)
    ctr  = (j >> 4, t, h, offset mod 2^32)      t = packed query row (batch_offset[b] + i)
                                                j = key index inside the sequence
    w    = Philox4x32-10(ctr, key)              four 32-bit words
    r8   = (w[(j & 15) >> 2] >> (8 * (j & 3))) & 0xFF
    keep <=> r8 >= thr,  thr = floor(p * 256)   (p taken as the float32 the API passes)
    kept values are scaled by 1 / (1 - thr / 256), the exact inverse keep probability

so the mask is a pure function of absolute coordinates (independent of tiling,
bucketing or work order), one Philox call serves 16 consecutive keys of one row (8-bit
decisions, as FlashAttention's uint8 threshold: half the Philox work of 16-bit ones), and
the estimator stays unbiased for any p (revision of R5 made for the kernels' cost, see
DESIGN.md).

Philox4x32-10 follows Salmon et al., "Parallel random numbers: as easy as 1, 2, 3"
(SC'11): round(ctr,key) = (hi(M1*c2) ^ c1 ^ k0, lo(M1*c2), hi(M0*c0) ^ c3 ^ k1, lo(M0*c0)),
key bumped by (W0, W1) between the 10 rounds.

Pins (tests/test_oracle_philox.py): the Random123 known-answer vectors, keep
fraction vs the binomial CI, p=0 keeps all.  Parity pinned.
"""
from __future__ import annotations

import numpy as np

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = 0xFFFFFFFF


def _mulhilo(a: int, b: np.ndarray):
    prod = np.uint64(a) * b.astype(np.uint64)
    return prod >> np.uint64(32), prod & np.uint64(MASK32)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 on uint64 arrays holding 32-bit values.

    Returns a tuple of four uint64 arrays (each < 2^32)."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & np.uint64(MASK32) for x in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64) & np.uint64(MASK32)
    k1 = np.asarray(k1, dtype=np.uint64) & np.uint64(MASK32)
    for r in range(10):
        if r > 0:
            k0 = (k0 + np.uint64(W0)) & np.uint64(MASK32)
            k1 = (k1 + np.uint64(W1)) & np.uint64(MASK32)
        hi0, lo0 = _mulhilo(M0, c0)
        hi1, lo1 = _mulhilo(M1, c2)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def dropout_threshold(p: float) -> int:
    """thr = floor(p * 256) with p rounded to float32 first (the API carries a float)."""
    p32 = float(np.float32(p))
    return int(np.floor(p32 * 256.0))


def dropout_scale(p: float) -> float:
    """Inverted-dropout scale 1 / (1 - thr / 256): kept values over the keep probability."""
    return 1.0 / (1.0 - dropout_threshold(p) / 256.0)


def keep_mask_block(seed: int, offset: int, t0: int, L: int, h: int, p: float) -> np.ndarray:
    """Keep mask [L, L] (query i, key j) for the sequence whose first packed row is t0."""
    thr = dropout_threshold(p)
    i = np.arange(L, dtype=np.uint64)[:, None]
    j = np.arange(L, dtype=np.uint64)[None, :]
    t = np.uint64(t0) + i
    ii, jj = np.broadcast_arrays(t, j)
    w = philox4x32_10(jj >> np.uint64(4), ii, np.full(ii.shape, h, np.uint64),
                      np.full(ii.shape, offset & MASK32, np.uint64),
                      np.uint64(seed & MASK32), np.uint64((seed >> 32) & MASK32))
    word_idx = (jj & np.uint64(15)) >> np.uint64(2)
    word = np.choose(word_idx.astype(np.int64), w)
    r8 = (word >> (np.uint64(8) * (jj & np.uint64(3)))) & np.uint64(0xFF)
    return r8 >= np.uint64(thr)
