"""Randomised GPU parity sweep (tcgen05 FMHA fwd + bwd, with and without dropout, plain and
fused-pad forward) against the fp64 oracle on sampled sequences: random batch sizes,
lengths (all buckets, ragged tails), head counts and seeds."""
import math

import numpy as np
import pytest
import torch

from gpu_util import assert_close, make_batch, oracle_seq_slice, TOL_LSE

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ub():
    import paper_2208_08124_b200 as m
    return m


@pytest.mark.parametrize("case", range(6))
def test_random_batches(ub, case):
    rng = np.random.default_rng(1000 + case)
    B = int(rng.integers(1, 40))
    H = int(rng.choice([1, 2, 4, 16]))
    S = int(rng.choice([128, 256, 512]))
    L = rng.integers(1, S + 1, size=B).astype(np.int32)
    p = float(rng.choice([0.0, 0.1, 0.25]))
    seed = int(rng.integers(0, 2**40))
    lengths, off, qkv, dout = make_batch(L, H, 64, seed=int(rng.integers(0, 10000)))
    qd, gd = qkv.cuda(), dout.cuda()
    cu = torch.tensor(off.astype(np.int32)).cuda()
    scale = 1.0 / math.sqrt(64)
    padded = torch.empty((B, S, H, 64), dtype=torch.bfloat16, device="cuda") if case % 2 else None
    o, lse = ub.varlen_fmha_fwd(qd, cu, S, scale, p, seed, 3, padded=padded)
    d = ub.varlen_fmha_bwd(qd, o, lse, gd, cu, S, scale, p, seed, 3)
    torch.cuda.synchronize()
    seqs = sorted(set(rng.choice(B, size=min(B, 4), replace=False).tolist()))
    ref = oracle_seq_slice(qkv, dout, off, seqs, scale, p, seed, 3)
    oc, lc, dc = o.float().cpu().numpy(), lse.cpu().numpy(), d.float().cpu().numpy()
    for b in seqs:
        s, e = int(off[b]), int(off[b + 1])
        O, LSE, dq = ref[b]
        assert_close(oc[s:e], O, f"O seq{b}")
        assert np.max(np.abs(lc[:, s:e] - LSE)) <= TOL_LSE
        for i, name in enumerate("qkv"):
            assert_close(dc[s:e, i], dq[:, i], f"d{name} seq{b}")
    if padded is not None:
        assert torch.equal(padded.view(torch.int16), ub.pad(o, cu, B, S).view(torch.int16))
