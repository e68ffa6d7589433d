"""Unpad storage (§IV-A-1, Fig. fig-storage), gather/scatter and
nonzero_indices (§IV-B-2).  ORACLE: test infrastructure only.

Pins (tests/test_oracle_varlen.py): SPEC worked examples,
round trips, differencing, nonzero cross-check.  Parity pinned.
"""
from __future__ import annotations

import numpy as np


def batch_offset(lengths) -> np.ndarray:
    """Prefix-sum array of P:302: ``[0, L0, L0+L1, ...]`` (B+1 entries, int64).

    Written as the plain running sum, one sample at a time.
    Raises ValueError on an empty list or a length < 1 (reading R8).
    """
    lengths = [int(x) for x in lengths]
    if len(lengths) == 0:
        raise ValueError("empty lengths")
    out = [0]
    for L in lengths:
        if L < 1:
            raise ValueError("sequence length must be >= 1")
        out.append(out[-1] + L)
    return np.asarray(out, dtype=np.int64)


def unpad(padded: np.ndarray, lengths) -> np.ndarray:
    """Gather: padded ``[B, S, ...]`` -> packed ``[sum L, ...]``.

    Row i of sequence b goes to packed row ``offset[b] + i`` for i < L_b.
    """
    lengths = [int(x) for x in lengths]
    B, S = padded.shape[0], padded.shape[1]
    if len(lengths) != B:
        raise ValueError("lengths / batch mismatch")
    rows = []
    for b in range(B):
        if lengths[b] > S:
            raise ValueError("length exceeds max_seq_len")
        for i in range(lengths[b]):
            rows.append(padded[b, i])
    if not rows:
        return np.zeros((0,) + padded.shape[2:], dtype=padded.dtype)
    return np.stack(rows, axis=0)


def pad(packed: np.ndarray, offsets, max_seq_len: int, pad_value=0) -> np.ndarray:
    """Scatter: packed ``[T, ...]`` -> padded ``[B, max_seq_len, ...]``.

    Positions i >= L_b hold ``pad_value`` (a scalar or a row of the trailing shape).
    Raises ValueError when a length exceeds ``max_seq_len`` (capacity error).
    """
    offsets = [int(x) for x in offsets]
    B = len(offsets) - 1
    out = np.empty((B, max_seq_len) + packed.shape[1:], dtype=packed.dtype)
    out[...] = pad_value
    for b in range(B):
        L = offsets[b + 1] - offsets[b]
        if L > max_seq_len:
            raise ValueError("capacity: length exceeds max_seq_len")
        for i in range(L):
            out[b, i] = packed[offsets[b] + i]
    return out


def nonzero_indices(mask: np.ndarray) -> np.ndarray:
    """Row-major flat positions where ``input_mask`` is non-zero."""
    flat = np.asarray(mask).reshape(-1)
    return np.asarray([i for i in range(flat.size) if flat[i] != 0], dtype=np.int64)


def lengths_from_mask(mask: np.ndarray) -> np.ndarray:
    """Valid-token count per row of a prefix ``input_mask`` ("The valid input
    token number can be obtained from the input tensor input_mask").  Raises on a
    non-prefix row."""
    mask = np.asarray(mask)
    out = []
    for row in mask:
        L = int(np.sum(row != 0))
        if np.any(row[:L] == 0) or np.any(row[L:] != 0):
            raise ValueError("non-prefix mask")
        out.append(L)
    return np.asarray(out, dtype=np.int64)
