"""Pins for oracle.attention (Eq. 1; unpadded equivalence) -- CPU only.

Each pin is chosen so that a plausible mistake (dropped term, wrong sign, wrong
index, transposed operand, missing scale, mask on the wrong axis) fails at least one.
"""
import math

import numpy as np
import pytest
import torch

from oracle import attention, philox, varlen
import synth


def _rand_padded(rng, lengths, S, H, D):
    B = len(lengths)
    q, k, v = (rng.standard_normal((B, S, H, D)) for _ in range(3))
    return q, k, v


def test_two_token_hand_case(golden):
    ex = golden["spec_worked_examples"]["attention_two_token"][0]
    q = np.zeros((1, 2, 1, 1)); k = np.zeros((1, 2, 1, 1)); v = np.zeros((1, 2, 1, 1))
    q[0, 0, 0, 0] = ex["q"]
    k[0, :, 0, 0] = ex["k"]
    v[0, :, 0, 0] = ex["v"]
    O, LSE = attention.mha_fwd_padded(q, k, v, [2], scale=1.0)
    e = math.e
    assert abs(O[0, 0, 0, 0] - (2 + 5 * e) / (1 + e)) < 1e-14, ex["cite"]
    assert abs(LSE[0, 0, 0] - math.log(1 + e)) < 1e-14


def test_closed_forms():
    rng = np.random.default_rng(0)
    q, k, v = _rand_padded(rng, [1, 5], 6, 2, 4)
    O, _ = attention.mha_fwd_padded(q, k, v, [1, 5], scale=0.5)
    assert np.allclose(O[0, 0], v[0, 0], atol=1e-15)          # one valid token -> V row
    assert np.all(O[0, 1:] == 0) and np.all(O[1, 5:] == 0)     # padded query rows -> 0 (R3)
    k2 = k.copy(); k2[1, :, :, :] = k2[1, 0:1, :, :]             # identical keys -> mean of V
    O2, _ = attention.mha_fwd_padded(q, k2, v, [1, 5], scale=0.5)
    assert np.allclose(O2[1, :5], v[1, :5].mean(axis=0, keepdims=True), atol=1e-13)
    O3, L3 = attention.mha_fwd_padded(np.zeros_like(q), k, v, [1, 5], scale=0.5)  # Q=0 -> uniform
    assert np.allclose(O3[1, :5], v[1, :5].mean(axis=0, keepdims=True), atol=1e-13)
    assert np.allclose(L3[1, :, :5], math.log(5), atol=1e-13)


def test_rows_sum_to_one_and_no_leakage():
    rng = np.random.default_rng(1)
    lens = [3, 7, 1, 5]
    q, k, v = _rand_padded(rng, lens, 8, 2, 8)
    P = attention.attention_probs(q, k, lens, 1 / math.sqrt(8))
    for b, L in enumerate(lens):
        assert np.allclose(P[b, :, :, :].sum(-1), 1.0, atol=1e-12)
        assert np.all(P[b, :, :, L:] == 0)
    O, LSE = attention.mha_fwd_padded(q, k, v, lens, 1 / math.sqrt(8))
    q2, k2, v2 = q.copy(), k.copy(), v.copy()
    for b, L in enumerate(lens):                     # perturb padding only
        q2[b, L:] += 100.0; k2[b, L:] -= 50.0; v2[b, L:] = 1e6
    O2, LSE2 = attention.mha_fwd_padded(q2, k2, v2, lens, 1 / math.sqrt(8))
    assert np.array_equal(O, O2) and np.array_equal(LSE, LSE2)


def test_padded_equals_unpadded_and_permutation():
    rng = np.random.default_rng(2)
    lens = [2, 5, 7]
    off = varlen.batch_offset(lens)
    T, H, D = int(off[-1]), 2, 4
    qkv = rng.standard_normal((T, 3, H, D))
    O, _ = attention.varlen_fwd(qkv, off, 8, 0.5)
    Ou = attention.mha_fwd_unpadded(qkv[:, 0], qkv[:, 1], qkv[:, 2], off, 0.5)
    assert np.max(np.abs(O - Ou)) <= 1e-10 * max(1.0, np.max(np.abs(Ou)))
    # block independence: reversing the sequence order permutes the output blocks
    order = [2, 1, 0]
    qkv_p = np.concatenate([qkv[off[b]:off[b + 1]] for b in order])
    off_p = varlen.batch_offset([lens[b] for b in order])
    Op, _ = attention.varlen_fwd(qkv_p, off_p, 8, 0.5)
    for j, b in enumerate(order):
        assert np.allclose(Op[off_p[j]:off_p[j + 1]], O[off[b]:off[b + 1]], atol=1e-14)


def _torch_sdpa_seq(qkv_seq, scale):
    """Independent library routine: torch CPU fp64 SDPA on one sequence [L,3,H,D]."""
    t = torch.tensor(qkv_seq, dtype=torch.float64, requires_grad=True)
    q, k, v = (t[:, i].permute(1, 0, 2).unsqueeze(0) for i in range(3))
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, scale=scale)
    return t, o[0].permute(1, 0, 2)


def test_forward_and_backward_vs_torch_sdpa():
    rng = np.random.default_rng(3)
    lens = [3, 7, 1, 5]                       # BASELINE config 1 shape: H=2, D=8
    off = varlen.batch_offset(lens)
    T, H, D = int(off[-1]), 2, 8
    scale = 1 / math.sqrt(D)
    qkv = rng.standard_normal((T, 3, H, D))
    dout = rng.standard_normal((T, H, D))
    O, LSE = attention.varlen_fwd(qkv, off, 7, scale)
    dqkv = attention.varlen_bwd(qkv, dout, off, 7, scale)
    for b in range(len(lens)):
        s, e = off[b], off[b + 1]
        t, o = _torch_sdpa_seq(qkv[s:e], scale)
        assert np.allclose(O[s:e], o.detach().numpy(), atol=1e-12)
        (o * torch.tensor(dout[s:e])).sum().backward()
        assert np.allclose(dqkv[s:e], t.grad.numpy(), atol=1e-12)
        # LSE via torch logsumexp of the scaled logits
        qq = torch.tensor(qkv[s:e, 0]); kk = torch.tensor(qkv[s:e, 1])
        lse = torch.logsumexp(scale * torch.einsum("ihd,jhd->hij", qq, kk), dim=-1)
        assert np.allclose(LSE[:, s:e], lse.numpy(), atol=1e-12)


@pytest.mark.parametrize("p", [0.0, 0.3])
def test_backward_central_finite_differences(p):
    rng = np.random.default_rng(4)
    lens = [3, 2]
    S, H, D = 4, 2, 3
    q, k, v = _rand_padded(rng, lens, S, H, D)
    G = rng.standard_normal((2, S, H, D))
    keep = None
    if p > 0:
        keep = lambda b, h: philox.keep_mask_block(7, 0, 10 * b, lens[b], h, p)
    f = lambda q_, k_, v_: float(np.sum(attention.mha_fwd_padded(q_, k_, v_, lens, 0.7, p, keep)[0] * G))
    dQ, dK, dV = attention.mha_bwd_padded(q, k, v, G, lens, 0.7, p, keep)
    h_ = 1e-6
    for X, dX, which in ((q, dQ, 0), (k, dK, 1), (v, dV, 2)):
        num = np.zeros_like(X)
        it = np.nditer(X, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            Xp = X.copy(); Xp[idx] += h_
            Xm = X.copy(); Xm[idx] -= h_
            args_p = [q, k, v]; args_p[which] = Xp
            args_m = [q, k, v]; args_m[which] = Xm
            num[idx] = (f(*args_p) - f(*args_m)) / (2 * h_)
        assert np.max(np.abs(num - dX)) < 1e-6 * max(1.0, np.max(np.abs(dX))), which


def test_backward_invariants():
    rng = np.random.default_rng(5)
    lens = [1, 6, 4]
    off = varlen.batch_offset(lens)
    T, H, D = int(off[-1]), 2, 4
    qkv = rng.standard_normal((T, 3, H, D))
    dout = rng.standard_normal((T, H, D))
    d = attention.varlen_bwd(qkv, dout, off, 6, 0.5)
    for b in range(3):
        s, e = off[b], off[b + 1]
        assert np.allclose(d[s:e, 1].sum(axis=0), 0.0, atol=1e-12)           # sum_j dK_j = 0
        assert np.allclose(d[s:e, 2].sum(axis=0), dout[s:e].sum(axis=0), atol=1e-12)  # sum dV = sum dO
    assert np.allclose(d[0, 0], 0.0) and np.allclose(d[0, 1], 0.0)           # L=1: dQ = dK = 0
    assert np.allclose(d[0, 2], dout[0])                                      # L=1: dV = dO
    d2 = attention.varlen_bwd(qkv, 2.5 * dout, off, 6, 0.5)                   # linear in dO
    assert np.allclose(d2, 2.5 * d, atol=1e-12)


def test_delta_identity():
    """Delta_i = sum_j P_ij dP_ij equals sum_d dO_id O_id (used by the backward)."""
    rng = np.random.default_rng(6)
    lens = [5]
    q, k, v = _rand_padded(rng, lens, 5, 1, 3)
    dO = rng.standard_normal((1, 5, 1, 3))
    O, _ = attention.mha_fwd_padded(q, k, v, lens, 0.9)
    P = attention.attention_probs(q, k, lens, 0.9)[0, 0]
    dP = dO[0, :, 0] @ v[0, :, 0].T
    assert np.allclose((P * dP).sum(1), (dO[0, :, 0] * O[0, :, 0]).sum(1), atol=1e-13)


def test_dropout_unbiased_and_p0_identity():
    rng = np.random.default_rng(7)
    lens = [64]
    off = varlen.batch_offset(lens)
    qkv = rng.standard_normal((64, 3, 1, 8))
    O0, L0 = attention.varlen_fwd(qkv, off, 64, 0.35)
    Oz, Lz = attention.varlen_fwd(qkv, off, 64, 0.35, p=0.0, seed=99)
    assert np.array_equal(O0, Oz) and np.array_equal(L0, Lz)
    acc = np.zeros_like(O0)
    n = 200
    for s in range(n):
        Od, Ld = attention.varlen_fwd(qkv, off, 64, 0.35, p=0.2, seed=s)
        assert np.array_equal(Ld, L0)                   # LSE is taken before dropout (R4)
        acc += Od
    assert np.max(np.abs(acc / n - O0)) < 0.15          # E[O] = O (inverted dropout)
