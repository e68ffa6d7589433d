"""Unpadded BERT embedding forward and backward ("the embedding ... runs on unpadded
tokens", "Embedding Operator Optimization").
ORACLE: test infrastructure only.  numpy fp64.

Forward, per packed token t (reading R23 in DESIGN.md):
    out[t, :] = W_word[ids[t], :] + W_pos[pos[t], :] + W_type[seg[t], :]
Backward -- the operation the paper optimises ("the output's gradient from the same
index should be accumulated to get the weight's gradient"):
    dW_word[v, :] = sum over t with ids[t] = v of dout[t, :]     (likewise dW_pos, dW_type)
written here with np.add.at, the library routine for exactly that scatter-add.

Pins (tests/test_oracle_embedding.py): a hand-worked example, the one-hot matrix form
dW = onehot(ids)^T dout, conservation (the column sums of dW equal those of dout), and
tokens that never occur get zero gradient.  Parity pinned.
"""
from __future__ import annotations

import numpy as np


def embedding_fwd(ids, pos, seg, w_word, w_pos, w_type):
    ids, pos, seg = (np.asarray(a, np.int64) for a in (ids, pos, seg))
    return (np.asarray(w_word, np.float64)[ids] + np.asarray(w_pos, np.float64)[pos]
            + np.asarray(w_type, np.float64)[seg])


def embedding_bwd(dout, ids, pos, seg, vocab, n_pos, n_type):
    dout = np.asarray(dout, np.float64)
    E = dout.shape[1]
    out = []
    for idx, n in ((ids, vocab), (pos, n_pos), (seg, n_type)):
        d = np.zeros((n, E))
        np.add.at(d, np.asarray(idx, np.int64), dout)
        out.append(d)
    return tuple(out)


def packed_positions(offsets) -> np.ndarray:
    """Position of every packed token inside its sequence: 0..L_b-1 per sequence."""
    offsets = np.asarray(offsets, np.int64)
    T = int(offsets[-1])
    return np.arange(T) - np.repeat(offsets[:-1], np.diff(offsets))
