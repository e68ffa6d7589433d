"""In-process simulation of the padding exchange's data movement (P:355-359 steps 1
and 3; S:359 simulates the all-gather in-process).  ORACLE: test infrastructure only.

Every rank r holds B samples: valid lengths[r][k], packed token records
tokens[r] ([sum_k L, rec] bytes, sample k at batch_offset[k]) and per-sample
records samples[r] ([B, srec] bytes).  After the exchange rank d holds the samples
perm[d*B + 0 .. d*B + B-1] in that order: its packed tokens are the concatenation of
those samples' token rows, its sample records likewise, and its batch_offset is the
prefix sum of their lengths.  Pinned by tests/test_oracle_balance.py::test_exchange_simulation (multiset
of rows preserved, per-sample byte identity, cardinality).
"""
from __future__ import annotations

import numpy as np

from . import varlen


def exchange(lengths, tokens, samples, perm, W, B):
    """lengths: [W][B]; tokens: list of W uint8 arrays [T_r, rec]; samples: list of W
    uint8 arrays [B, srec]; perm: [W*B] global ids (g = r*B + k).
    Returns a list of W dicts {tokens, samples, cu}."""
    offs = [varlen.batch_offset(lengths[r]) for r in range(W)]
    out = []
    for d in range(W):
        tok_rows, smp_rows, lens = [], [], []
        for k in range(B):
            g = int(perm[d * B + k])
            src, kk = divmod(g, B)
            s, e = int(offs[src][kk]), int(offs[src][kk + 1])
            tok_rows.append(tokens[src][s:e])
            smp_rows.append(samples[src][kk:kk + 1])
            lens.append(e - s)
        out.append({"tokens": np.concatenate(tok_rows, axis=0),
                    "samples": np.concatenate(smp_rows, axis=0),
                    "cu": varlen.batch_offset(lens)})
    return out
