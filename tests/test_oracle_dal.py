"""Pins for oracle.dal (Dropout_Add_LayerNorm; reading R21) -- CPU only."""
import numpy as np
import torch

from oracle import dal


def _inputs(T=7, E=48, seed=0):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((T, E)), rng.standard_normal((T, E)), 1.0 + 0.1 * rng.standard_normal(E),
            0.1 * rng.standard_normal(E), rng.standard_normal((T, E)))


def _torch_ref(a, res, gamma, beta, dy, keep, p, eps):
    """Independent route: torch fp64 layer_norm + autograd, the mask applied by hand."""
    at = torch.tensor(a, requires_grad=True)
    rt = torch.tensor(res, requires_grad=True)
    gt = torch.tensor(gamma, requires_grad=True)
    bt = torch.tensor(beta, requires_grad=True)
    m = torch.tensor(keep, dtype=torch.float64) * dal.dal_dropout_scale(p)   # scale pinned below
    y = torch.nn.functional.layer_norm(rt + at * m, (a.shape[1],), gt, bt, eps)
    y.backward(torch.tensor(dy))
    return y.detach().numpy(), at.grad.numpy(), rt.grad.numpy(), gt.grad.numpy(), bt.grad.numpy()


def test_matches_torch_layer_norm_and_autograd():
    for p in (0.0, 0.1, 0.5):
        a, res, gamma, beta, dy = _inputs(seed=int(p * 10))
        keep = dal.dal_keep_mask(3, 9, a.shape[0], a.shape[1], p)
        y, mu, rstd = dal.dal_fwd(a, res, gamma, beta, p, 1e-5, 3, 9)
        da, dres, dg, db = dal.dal_bwd(dy, a, res, gamma, p, 1e-5, 3, 9)
        ry, rda, rdres, rdg, rdb = _torch_ref(a, res, gamma, beta, dy, keep, p, 1e-5)
        for got, exp in ((y, ry), (da, rda), (dres, rdres), (dg, rdg), (db, rdb)):
            assert np.allclose(got, exp, rtol=1e-10, atol=1e-10)


def test_finite_differences():
    a, res, gamma, beta, dy = _inputs(T=3, E=16, seed=4)
    p, eps, h = 0.25, 1e-5, 1e-6
    da, dres, dg, db = dal.dal_bwd(dy, a, res, gamma, p, eps, 1, 2)
    f = lambda a_, r_, g_, b_: float((dal.dal_fwd(a_, r_, g_, b_, p, eps, 1, 2)[0] * dy).sum())
    for (t, j) in ((0, 0), (1, 7), (2, 15)):
        e = np.zeros_like(a); e[t, j] = h
        assert abs((f(a + e, res, gamma, beta) - f(a - e, res, gamma, beta)) / (2 * h) - da[t, j]) < 1e-6
        assert abs((f(a, res + e, gamma, beta) - f(a, res - e, gamma, beta)) / (2 * h) - dres[t, j]) < 1e-6
    for j in (0, 9):
        e = np.zeros_like(gamma); e[j] = h
        assert abs((f(a, res, gamma + e, beta) - f(a, res, gamma - e, beta)) / (2 * h) - dg[j]) < 1e-6
        assert abs((f(a, res, gamma, beta + e) - f(a, res, gamma, beta - e)) / (2 * h) - db[j]) < 1e-6


def test_invariants_and_mask():
    a, res, gamma, beta, dy = _inputs(T=50, E=64, seed=5)
    da, dres, dg, db = dal.dal_bwd(dy, a, res, gamma, 0.1, 1e-12, 7, 0)
    assert np.allclose(dres.sum(axis=1), 0.0, atol=1e-9)       # LN is shift-invariant in z
    y, mu, rstd = dal.dal_fwd(a, res, np.ones(64), np.zeros(64), 0.1, 1e-12, 7, 0)
    assert np.allclose(y.mean(axis=1), 0.0, atol=1e-9) and np.allclose((y ** 2).mean(axis=1), 1.0, atol=1e-6)
    assert dal.dal_keep_mask(1, 0, 4, 32, 0.0).all()
    k = dal.dal_keep_mask(11, 5, 256, 1024, 0.1)
    n = k.size
    frac = k.mean()
    assert abs(frac - 0.9) < 5 * np.sqrt(0.09 / n) + 1.0 / 65536     # binomial bound (+ threshold rounding)
    # coordinate-pure: a sub-block equals the same rows/cols of a bigger mask
    assert np.array_equal(dal.dal_keep_mask(11, 5, 100, 64, 0.1), k[:100, :64])
    # dropped entries of a do not reach y: da is exactly zero there
    keep = dal.dal_keep_mask(7, 0, 50, 64, 0.1)
    assert np.all(da[~keep] == 0.0)


def test_scale_is_exact_inverse_keep_probability():
    """R21: a kept value is scaled by 1 / P(keep).  P(keep) by brute force over the whole
    16-bit space (r >= thr for r = 0..65535), so E[keep * r] = 1 exactly, for p on and off
    the 1/65536 grid; and the empirical keep fraction of a large mask matches it."""
    r16 = np.arange(65536)
    for p in (0.1, 0.25, 0.5, 1.0 / 3.0, 0.9, 3.0 / 65536):
        pk = np.count_nonzero(r16 >= dal.dal_threshold(p)) / 65536.0
        assert abs(dal.dal_dropout_scale(p) * pk - 1.0) < 1e-15, p
    assert dal.dal_dropout_scale(0.0) == 1.0
    k = dal.dal_keep_mask(2, 0, 512, 1024, 0.1)
    pk = np.count_nonzero(r16 >= dal.dal_threshold(0.1)) / 65536.0
    assert abs(k.mean() - pk) < 5 * np.sqrt(pk * (1 - pk) / k.size)
