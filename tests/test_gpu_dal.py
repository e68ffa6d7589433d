"""GPU parity of Dropout_Add_LayerNorm (reading R21) against the fp64 oracle."""
import numpy as np
import pytest
import torch

import synth
from gpu_util import assert_close
from oracle import dal as odal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ub():
    import paper_2208_08124_b200 as m
    return m


def _inputs(T, E, seed):
    a = synth.gen_normal((T, E), seed, torch.bfloat16)
    res = synth.gen_normal((T, E), seed + 1, torch.bfloat16)
    gamma = (1.0 + 0.1 * synth.gen_normal((E,), seed + 2)).to(torch.bfloat16)
    beta = (0.1 * synth.gen_normal((E,), seed + 3)).to(torch.bfloat16)
    dy = synth.gen_normal((T, E), seed + 4, torch.bfloat16)
    return a, res, gamma, beta, dy


@pytest.mark.parametrize("T,E,p", [(1, 1024, 0.0), (37, 1024, 0.1), (300, 1024, 0.1), (129, 768, 0.0),
                                   (64, 2048, 0.25), (33, 8, 0.1)])
def test_dal_fwd_bwd_parity(ub, T, E, p):
    a, res, gamma, beta, dy = _inputs(T, E, 50 + T)
    eps, seed, off = 1e-12, 0x2208 + T, 7
    y, mean, rstd = ub.dal_fwd(a.cuda(), res.cuda(), gamma.cuda(), beta.cuda(), p, eps, seed, off)
    da, dres, dg, db = ub.dal_bwd(dy.cuda(), a.cuda(), res.cuda(), gamma.cuda(), mean, rstd, p, seed, off)
    torch.cuda.synchronize()
    f64 = lambda t: t.double().numpy()
    Y, MU, RS = odal.dal_fwd(f64(a), f64(res), f64(gamma), f64(beta), p, eps, seed, off)
    DA, DRES, DG, DB = odal.dal_bwd(f64(dy), f64(a), f64(res), f64(gamma), p, eps, seed, off)
    assert_close(y.float().cpu().numpy(), Y, "y")
    assert np.max(np.abs(mean.cpu().numpy() - MU)) < 1e-4
    assert np.max(np.abs(rstd.cpu().numpy() / RS - 1)) < 1e-4
    assert_close(da.float().cpu().numpy(), DA, "da")
    assert_close(dres.float().cpu().numpy(), DRES, "dres")
    # parameter grads sum T rows in fp32: tolerance scales with sqrt(T)
    tol = 2e-2 * max(1.0, np.sqrt(T) / 4)
    assert_close(dg.cpu().numpy(), DG, "dgamma", max_abs=tol)
    assert_close(db.cpu().numpy(), DB, "dbeta", max_abs=tol)
    # the dropout mask, bit-exact: da is exactly zero where the oracle drops (and the
    # kept entries are nonzero unless dz rounds to 0)
    keep = odal.dal_keep_mask(seed, off, T, E, p)
    dah = da.float().cpu().numpy()
    assert np.all(dah[~keep] == 0.0)
    assert np.array_equal((dah != 0) | (np.abs(DRES) < 1e-3), keep | (np.abs(DRES) < 1e-3))


def test_dal_bert_large_full_size_sampled(ub):
    """T = 15 157 rows (a config-2 batch) x E = 1024 at p = 0.1: sampled rows vs the oracle,
    dgamma / dbeta in full; deterministic across calls."""
    L = synth.gen_lengths("mlperf_like_v0", 56, 0)
    T, E, p, seed = int(L.sum()), 1024, 0.1, 99
    a, res, gamma, beta, dy = _inputs(T, E, 7)
    ad, rd, gd, bd, dyd = a.cuda(), res.cuda(), gamma.cuda(), beta.cuda(), dy.cuda()
    y, mean, rstd = ub.dal_fwd(ad, rd, gd, bd, p, 1e-12, seed, 0)
    da, dres, dg, db = ub.dal_bwd(dyd, ad, rd, gd, mean, rstd, p, seed, 0)
    da2, dres2, dg2, db2 = ub.dal_bwd(dyd, ad, rd, gd, mean, rstd, p, seed, 0)
    torch.cuda.synchronize()
    assert torch.equal(dg, dg2) and torch.equal(db, db2) and torch.equal(da, da2)
    rows = np.random.default_rng(3).choice(T, 64, replace=False)
    f64 = lambda t: t.double().numpy()
    Y, _, _ = odal.dal_fwd(f64(a), f64(res), f64(gamma), f64(beta), p, 1e-12, seed, 0)
    assert_close(y.float().cpu().numpy()[rows], Y[rows], "y sampled")
    DA, DRES, DG, DB = odal.dal_bwd(f64(dy), f64(a), f64(res), f64(gamma), p, 1e-12, seed, 0)
    assert_close(dres.float().cpu().numpy()[rows], DRES[rows], "dres sampled")
    assert_close(da.float().cpu().numpy()[rows], DA[rows], "da sampled")
    assert_close(dg.cpu().numpy(), DG, "dgamma", max_abs=1.0)
    assert_close(db.cpu().numpy(), DB, "dbeta", max_abs=1.0)


def test_dal_bwd_growing_width(ub):
    """Backward calls with E growing across calls (the shared-memory attribute is set once
    per kernel for its largest width)."""
    for E in (64, 1024, 2048):
        a, res, gamma, beta, dy = _inputs(16, E, E)
        y, mean, rstd = ub.dal_fwd(a.cuda(), res.cuda(), gamma.cuda(), beta.cuda())
        da, dres, dg, db = ub.dal_bwd(dy.cuda(), a.cuda(), res.cuda(), gamma.cuda(), mean, rstd)
        torch.cuda.synchronize()
        f64 = lambda t: t.double().numpy()
        DA, DRES, DG, DB = odal.dal_bwd(f64(dy), f64(a), f64(res), f64(gamma))
        assert_close(dres.float().cpu().numpy(), DRES, f"dres E={E}")


def test_dal_invalid_arguments(ub):
    from paper_2208_08124_b200 import UbError
    a = torch.zeros((4, 12), dtype=torch.bfloat16, device="cuda")
    g = torch.zeros(12, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(UbError) as e:
        ub.dal_fwd(a, a, g, g)                     # E = 12 not a multiple of 8
    assert e.value.status == 5
    a = torch.zeros((4, 16), dtype=torch.bfloat16, device="cuda")
    g = torch.zeros(16, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(UbError) as e:
        ub.dal_fwd(a, a, g, g, p_dropout=1.0)
    assert e.value.status == 1
