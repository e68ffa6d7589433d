"""Parity of the CUDA varlen FMHA (through the C ABI) against the fp64 oracle.  -m gpu."""
import math

import numpy as np
import pytest
import torch

import synth
from gpu_util import assert_close, errors, make_batch, oracle_seq_slice, TOL_LSE
from oracle import attention as oatt

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ub():
    import paper_2208_08124_b200 as ub
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return ub


def _run(ub, lengths, H, D, dtype, p=0.0, seed=7, max_seqlen=None, bwd=True):
    lengths, off, qkv, dout = make_batch(lengths, H, D, dtype)
    cu = torch.tensor(off.astype(np.int32)).cuda()
    ms = int(max_seqlen or lengths.max())
    scale = 1.0 / math.sqrt(D)
    qd, gd = qkv.cuda(), dout.cuda()
    o, lse = ub.varlen_fmha_fwd(qd, cu, ms, scale, p, seed, 0)
    d = ub.varlen_fmha_bwd(qd, o, lse, gd, cu, ms, scale, p, seed, 0) if bwd else None
    torch.cuda.synchronize()
    return lengths, off, qkv, dout, o.cpu(), lse.cpu(), (d.cpu() if d is not None else None), scale


# BASELINE config 1: 4 sequences {3,7,1,5}, 2 heads x 8, fp32, vs CPU fp64 padded-masked attention
@pytest.mark.parametrize("p", [0.0, 0.1])
def test_config1_tiny_fp32(ub, p):
    lengths, off, qkv, dout, o, lse, d, scale = _run(ub, [3, 7, 1, 5], 2, 8, torch.float32, p=p)
    q64, g64 = qkv.double().numpy(), dout.double().numpy()
    O, LSE = oatt.varlen_fwd(q64, off, 7, scale, p, 7, 0)
    dq = oatt.varlen_bwd(q64, g64, off, 7, scale, p, 7, 0)
    assert_close(o.numpy(), O, "O", 1e-5, 1e-5)
    assert_close(lse.numpy(), LSE, "LSE", 1e-5, 1e-5)
    assert_close(d.numpy(), dq, "dqkv", 1e-4, 1e-5)


# tile edges; also the backward's warpgroup skip (a last query tile of <= 64 rows: 64, 65, 192,
# 193, 448, 449 sit on both sides of it at one, two and four tiles)
EDGE_LENGTHS = [1, 127, 128, 129, 255, 256, 300, 512, 64, 2, 383, 384, 385, 65, 192, 193, 448, 449]


@pytest.mark.parametrize("p", [0.0, 0.1])
def test_bf16_edge_lengths_fwd_bwd(ub, p):
    lengths, off, qkv, dout, o, lse, d, scale = _run(ub, EDGE_LENGTHS, 2, 64, torch.bfloat16, p=p, max_seqlen=512)
    q64, g64 = qkv.double().numpy(), dout.double().numpy()
    O, LSE = oatt.varlen_fwd(q64, off, 512, scale, p, 7, 0)
    assert_close(o.float().numpy(), O, "O")
    assert_close(lse.numpy(), LSE, "LSE", TOL_LSE, 1.0)
    dq = oatt.varlen_bwd(q64, g64, off, 512, scale, p, 7, 0)
    for i, name in enumerate("qkv"):
        assert_close(d[:, i].float().numpy(), dq[:, i], "d" + name)


def test_bf16_longer_than_in_kernel_delta(ub):
    """max_seqlen > 512: the backward takes its Delta from the separate row-dot kernel instead
    of computing it per item in shared memory; both paths against the oracle (L = 700, 129)."""
    lengths, off, qkv, dout, o, lse, d, scale = _run(ub, [700, 129, 5], 2, 64, torch.bfloat16, p=0.1,
                                                     max_seqlen=768)
    q64, g64 = qkv.double().numpy(), dout.double().numpy()
    O, LSE = oatt.varlen_fwd(q64, off, 768, scale, 0.1, 7, 0)
    assert_close(o.float().numpy(), O, "O")
    dq = oatt.varlen_bwd(q64, g64, off, 768, scale, 0.1, 7, 0)
    for i, name in enumerate("qkv"):
        assert_close(d[:, i].float().numpy(), dq[:, i], "d" + name)


def test_bf16_fwd_deterministic_and_single_sequence(ub):
    lengths, off, qkv, dout = make_batch([200, 77], 3, 64)
    cu = torch.tensor(off.astype(np.int32)).cuda()
    qd = qkv.cuda()
    o1, l1 = ub.varlen_fmha_fwd(qd, cu, 512)
    o2, l2 = ub.varlen_fmha_fwd(qd, cu, 512)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    # L = 1: output equals the V row exactly up to bf16 rounding
    lengths, off, qkv, dout = make_batch([1, 1, 1], 2, 64)
    cu = torch.tensor(off.astype(np.int32)).cuda()
    o, lse = ub.varlen_fmha_fwd(qkv.cuda(), cu, 512)
    torch.cuda.synchronize()
    assert torch.equal(o.cpu(), qkv[:, 2])
    d = ub.varlen_fmha_bwd(qkv.cuda(), o, lse, dout.cuda(), cu, 512)
    torch.cuda.synchronize()
    d = d.cpu().float()
    # L=1: dQ = dK = 0 (dS = P (dP - Delta) with P = 1 and dP = Delta up to fp32 summation order)
    assert float(d[:, 0].abs().max()) < 1e-5 and float(d[:, 1].abs().max()) < 1e-5
    assert torch.equal(d[:, 2], dout.float())                         # dV = dO


@pytest.mark.parametrize("p", [0.0, 0.1])
def test_bf16_config2_full_batch_every_sequence(ub, p):
    """BASELINE config 2 (56 x mlperf_like_v0 lengths up to 512, 16 heads x 64, bf16, persistent
    grid), at p = 0 and at BERT-large's attention dropout p = 0.1: EVERY sequence's O, LSE, dQ,
    dK, dV element by element against the fp64 oracle (per sequence, absolute dropout
    coordinates), under the BASELINE tolerance.  (bench.py's launch configuration gives these
    results bitwise: test_bench_launch_configuration_bitwise.)"""
    L = synth.gen_lengths("mlperf_like_v0", 56, 0)
    seed = 0x2208
    lengths, off, qkv, dout, o, lse, d, scale = _run(ub, L, 16, 64, torch.bfloat16, p=p, seed=seed, max_seqlen=512)
    ref = oracle_seq_slice(qkv, dout, off, range(len(L)), scale, p=p, seed=seed, offset=0)
    worst = {}
    for b in range(len(L)):
        s, e = int(off[b]), int(off[b + 1])
        O, LSE, dq = ref[b]
        worst.setdefault("O", []).append(assert_close(o[s:e].float().numpy(), O, f"O seq{b} L={e - s}"))
        assert_close(lse[:, s:e].numpy(), LSE, f"LSE seq{b}", TOL_LSE, 1.0)
        for i, name in enumerate("qkv"):
            worst.setdefault(name, []).append(assert_close(d[s:e, i].float().numpy(), dq[:, i],
                                                           f"d{name} seq{b} L={e - s}"))
    # the whole batch as one tensor, too (rel-L2 over all 56 sequences)
    O_all = np.concatenate([ref[b][0] for b in range(len(L))])
    D_all = np.concatenate([ref[b][2] for b in range(len(L))])
    assert_close(o.float().numpy(), O_all, "O batch")
    assert_close(d.float().numpy(), D_all, "dqkv batch")


@pytest.mark.parametrize("dist,seed", [("mlperf_like_v0", 0), ("uniform", 1), ("bimodal", 2)])
def test_bf16_bert_large_full_size_sampled(ub, dist, seed):
    """BASELINE config 2 / 5 at full size (56 x up to 512, 16 heads x 64) in the launch
    configuration bench.py times; the oracle checks a sample of sequences one by one
    (longest, shortest and a few in between), plus size-independent invariants."""
    L = synth.gen_lengths(dist, 56, seed)
    lengths, off, qkv, dout, o, lse, d, scale = _run(ub, L, 16, 64, torch.bfloat16, p=0.0, max_seqlen=512)
    order = np.argsort(L)
    seqs = sorted(set([int(order[0]), int(order[-1]), int(order[len(order) // 2]), int(order[len(order) // 4]),
                       int(order[3 * len(order) // 4])]))
    ref = oracle_seq_slice(qkv, dout, off, seqs, scale)
    for b in seqs:
        s, e = int(off[b]), int(off[b + 1])
        O, LSE, dq = ref[b]
        assert_close(o[s:e].float().numpy(), O, f"O seq{b}")
        assert_close(lse[:, s:e].numpy(), LSE, f"LSE seq{b}", TOL_LSE, 1.0)
        for i, name in enumerate("qkv"):
            assert_close(d[s:e, i].float().numpy(), dq[:, i], f"d{name} seq{b}")
    # invariants at full size: sum_j dK_j = 0 and sum_j dV_j = sum_i dO_i per (seq, head)
    d32, g32 = d.float(), dout.float()
    for b in range(len(L)):
        s, e = int(off[b]), int(off[b + 1])
        dk_sum = d32[s:e, 1].sum(0)
        assert float(dk_sum.abs().max()) < 0.05 * max(1.0, math.sqrt(e - s)), b
        assert_close(d32[s:e, 2].sum(0).numpy(), g32[s:e].sum(0).numpy(), f"sum dV seq{b}", 0.05 * math.sqrt(e - s), 2e-2)


def test_bf16_dropout_mask_matches_oracle(ub):
    """The dropout mask of BOTH kernels equals the oracle's Philox mask (R5) bitwise, at all
    16 heads and at several packed-row offsets (the counter words t, h of R5):
      forward  -- V rows one-hot (v_j = e_j): O[i, d=j] = P~[i, j], kept <=> O != 0;
      backward -- dO rows one-hot (dO_i = e_i): dV[j, d=i] = P~[i, j], kept <=> dV != 0."""
    Ls, H, D = [64, 40, 64, 17], 16, 64
    lengths, off, qkv, dout = make_batch(Ls, H, D)
    qkv[:, 2] = 0
    dout[:] = 0
    for b, L in enumerate(Ls):
        s = int(off[b])
        for j in range(L):
            qkv[s + j, 2, :, j] = 1.0                   # v_j = e_j
            dout[s + j, :, j] = 1.0                     # dO_j = e_j
    qd = qkv.cuda()
    cu = torch.tensor(off.astype(np.int32)).cuda()
    p, seed, offs = 0.3, 1234, 5
    o, lse = ub.varlen_fmha_fwd(qd, cu, 512, None, p, seed, offs)
    d = ub.varlen_fmha_bwd(qd, o, lse, dout.cuda(), cu, 512, None, p, seed, offs)
    torch.cuda.synchronize()
    o, dv = o.float().cpu().numpy(), d[:, 2].float().cpu().numpy()
    from oracle import philox
    for b, L in enumerate(Ls):
        s = int(off[b])
        for h in range(H):
            keep = philox.keep_mask_block(seed, offs, s, L, h, p)          # [query i, key j]
            assert np.array_equal(o[s:s + L, h, :L] != 0, keep), (b, h)
            assert np.array_equal((dv[s:s + L, h, :L] != 0).T, keep), (b, h)


def test_invalid_arguments(ub):
    from paper_2208_08124_b200._lib import UbError
    lengths, off, qkv, dout = make_batch([5], 2, 32)
    cu = torch.tensor(off.astype(np.int32)).cuda()
    with pytest.raises(UbError) as e:
        ub.varlen_fmha_fwd(qkv.cuda(), cu, 512)       # bf16 path supports head_dim 64 only
    assert e.value.status == 5
    lengths, off, qkv, dout = make_batch([5], 2, 64)
    cu = torch.tensor(off.astype(np.int32)).cuda()
    with pytest.raises(UbError) as e:
        ub.varlen_fmha_fwd(qkv.cuda(), cu, 512, p_dropout=1.0)
    assert e.value.status == 1
    with pytest.raises(UbError) as e:                     # p < 1/256: R5's 8-bit decisions drop nothing
        ub.varlen_fmha_fwd(qkv.cuda(), cu, 512, p_dropout=0.003)
    assert e.value.status == 1



def test_bwd_repeatable_across_changing_batches(ub):
    """Back-to-back backward calls on batches of different T (shared cached workspace)
    give bit-identical dQ, dK, dV for the same inputs: every reduction has a fixed order
    (dQ partials are added pass by pass by one CTA, R16), and no state leaks between calls."""
    outs = []
    for L in ([300, 45, 512, 129], [512, 512, 3], [300, 45, 512, 129]):
        lengths, off, qkv, dout = make_batch(L, 4, 64, seed=77)
        cu = torch.tensor(off.astype(np.int32)).cuda()
        qd, gd = qkv.cuda(), dout.cuda()
        o, lse = ub.varlen_fmha_fwd(qd, cu, 512)
        d = ub.varlen_fmha_bwd(qd, o, lse, gd, cu, 512)
        torch.cuda.synchronize()
        outs.append(d.cpu())
    assert torch.equal(outs[0], outs[2])


def test_bf16_more_sequences_than_smem_plan(ub):
    """B > kPlanCap (512): the kernels fall back to the separate plan kernel and the
    global-memory work decode; results must match the oracle on sampled sequences."""
    rng = np.random.default_rng(3)
    L = rng.integers(1, 60, size=1100)
    L[0], L[1] = 200, 129
    lengths, off, qkv, dout, o, lse, d, scale = _run(ub, L, 2, 64, torch.bfloat16, p=0.0, max_seqlen=256)
    seqs = [0, 1, 2, 500, 1099]
    ref = oracle_seq_slice(qkv, dout, off, seqs, scale)
    for b in seqs:
        s, e = int(off[b]), int(off[b + 1])
        O, LSE, dq = ref[b]
        assert_close(o[s:e].float().numpy(), O, f"O seq{b}")
        for i, name in enumerate("qkv"):
            assert_close(d[s:e, i].float().numpy(), dq[:, i], f"d{name} seq{b}")


def test_item_table_overflow_same_results(ub):
    """With 2 CTAs every CTA owns more items than its shared-memory item table holds, so the
    kernels take the global-plan decode path: forward and backward must be bitwise the same
    as with the full grid (the per-item arithmetic does not depend on the CTA)."""
    rng = np.random.default_rng(11)
    L = rng.integers(1, 513, size=40).astype(np.int32)
    lengths, off, qkv, dout = make_batch(L, 4, 64, seed=5)
    cu = torch.tensor(off.astype(np.int32)).cuda()
    qd, gd = qkv.cuda(), dout.cuda()
    res = []
    for n in (0, 2):
        o, lse = ub.varlen_fmha_fwd(qd, cu, 512, num_ctas=n)
        d = ub.varlen_fmha_bwd(qd, o, lse, gd, cu, 512, num_ctas=n)
        torch.cuda.synchronize()
        res.append((o.cpu(), lse.cpu(), d.cpu()))
    for a, b in zip(res[0], res[1]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("p", [0.0, 0.1])
def test_fwd_with_fused_pad(ub, p):
    """ub_varlen_fmha_fwd_pad (a7 + a9): out / lse identical to the plain forward, padded
    identical (bitwise) to ub_pad of out -- zeros past each length, including whole padded
    tiles, sequences of one token and EMPTY sequences (no work item: zero-filled by the
    kernel's otherwise idle warp)."""
    L = np.array([1, 31, 32, 33, 127, 128, 129, 300, 0, 512, 64, 0], np.int32)   # incl. empty sequences
    off = np.concatenate([[0], np.cumsum(L)]).astype(np.int64)      # (the oracle rejects L = 0, R8)
    qkv = synth.gen_normal((int(off[-1]), 3, 4, 64), 1000)
    qd = qkv.cuda()
    cu = torch.tensor(off.astype(np.int32)).cuda()
    S = 512
    o1, l1 = ub.varlen_fmha_fwd(qd, cu, S, None, p, 3, 0)
    padded = torch.full((len(L), S, 4, 64), float("nan"), dtype=torch.bfloat16, device="cuda")
    o2, l2 = ub.varlen_fmha_fwd(qd, cu, S, None, p, 3, 0, padded=padded)
    ref = ub.pad(o1, cu, len(L), S)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    assert torch.equal(padded.view(torch.int16), ref.view(torch.int16))


def test_dropout_mask_layouts_match_oracle(ub):
    """ub_dropout_mask (R5 materialised): both bit layouts equal the oracle's Philox mask
    bitwise for every (head, query, key) of a batch with sequences of 1..300 tokens."""
    from oracle import philox
    L = [300, 1, 33, 128, 129, 64]
    off = np.concatenate([[0], np.cumsum(L)]).astype(np.int64)
    T, H, MT, p, seed, offs = int(off[-1]), 3, 3, 0.1, 0x1234_5678_9ABC, 77
    cu = torch.tensor(off.astype(np.int32)).cuda()
    m = ub.api.dropout_mask(cu, T, H, 384, p, seed, offs)
    torch.cuda.synchronize()
    words = m.cpu().numpy().view(np.uint32)
    half = words.size // 2
    mq = words[:H * T * MT * 4].reshape(H, MT, 4, T).transpose(0, 3, 1, 2)     # -> [H, T, MT, 4]
    mk = words[half:half + H * T * MT * 4].reshape(H, MT, 4, T).transpose(0, 3, 1, 2)
    for b, Lb in enumerate(L):
        s = int(off[b])
        nt = (Lb + 127) // 128
        for h in range(H):
            keep = philox.keep_mask_block(seed, offs, s, Lb, h, p)          # [query, key]
            qbits = np.unpackbits(np.ascontiguousarray(mq[h, s:s + Lb, :nt]).reshape(Lb, -1).view(np.uint8), axis=1,
                                  bitorder="little")
            kbits = np.unpackbits(np.ascontiguousarray(mk[h, s:s + Lb, :nt]).reshape(Lb, -1).view(np.uint8), axis=1,
                                  bitorder="little")
            assert np.array_equal(qbits[:, :Lb].astype(bool), keep), (b, h)
            assert np.array_equal(kbits[:, :Lb].astype(bool), keep.T), (b, h)


def test_external_dropout_mask_same_results(ub):
    """A mask materialised once (ub_dropout_mask) and passed to both directions gives bitwise
    the results of the calls that materialise it themselves."""
    L = [512, 300, 45, 129, 1]
    lengths, off, qkv, dout = make_batch(L, 4, 64, seed=21)
    cu = torch.tensor(off.astype(np.int32)).cuda()
    qd, gd = qkv.cuda(), dout.cuda()
    T = int(off[-1])
    o1, l1 = ub.varlen_fmha_fwd(qd, cu, 512, None, 0.1, 9, 3)
    d1 = ub.varlen_fmha_bwd(qd, o1, l1, gd, cu, 512, None, 0.1, 9, 3)
    m = ub.api.dropout_mask(cu, T, 4, 512, 0.1, 9, 3)
    o2, l2 = ub.varlen_fmha_fwd(qd, cu, 512, None, 0.1, 9, 3, dropout_mask=m)
    d2 = ub.varlen_fmha_bwd(qd, o2, l2, gd, cu, 512, None, 0.1, 9, 3, dropout_mask=m)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2) and torch.equal(d1, d2)


def test_overlapped_mask_behind_backward(ub):
    """UB_MASK_OVERLAP_PREVIOUS: the next step's mask launched right behind a backward that
    reads the other mask buffer (the bench's step pipeline) equals the plain mask bitwise, and
    the next step's results are bitwise those with the plain mask."""
    from paper_2208_08124_b200 import api
    H = 16
    L1 = synth.gen_lengths("mlperf_like_v0", 56, 31)
    L2 = synth.gen_lengths("mlperf_like_v0", 56, 32)
    _, off1, qkv1, dout1 = make_batch(L1, H, 64, seed=41)
    _, off2, qkv2, dout2 = make_batch(L2, H, 64, seed=42)
    cu1, cu2 = (torch.tensor(o.astype(np.int32)).cuda() for o in (off1, off2))
    T1, T2 = int(off1[-1]), int(off2[-1])
    q1, g1, q2, g2 = qkv1.cuda(), dout1.cuda(), qkv2.cuda(), dout2.cuda()
    cap = max(T1, T2)
    bufs = [torch.zeros(api.dropout_mask_bytes(cap, H, 512), dtype=torch.uint8, device="cuda") for _ in range(2)]
    m1 = api.BoundDropoutMask(cu1, cap, H, 512, 0.1, bufs[0])
    m2 = api.BoundDropoutMask(cu2, cap, H, 512, 0.1, bufs[1], overlap_previous=True)
    m1(T1, 5)
    o, lse = ub.varlen_fmha_fwd(q1, cu1, 512, None, 0.1, 5, 0, dropout_mask=bufs[0])
    ub.varlen_fmha_bwd(q1, o, lse, g1, cu1, 512, None, 0.1, 5, 0, dropout_mask=bufs[0])
    m2(T2, 6)                                            # behind the backward, overlapping its tail
    o2, l2 = ub.varlen_fmha_fwd(q2, cu2, 512, None, 0.1, 6, 0, dropout_mask=bufs[1])
    d2 = ub.varlen_fmha_bwd(q2, o2, l2, g2, cu2, 512, None, 0.1, 6, 0, dropout_mask=bufs[1])
    torch.cuda.synchronize()
    # (words of rows past a sequence end stay unwritten: both buffers start zeroed)
    plain = torch.zeros_like(bufs[1])
    api.BoundDropoutMask(cu2, cap, H, 512, 0.1, plain)(T2, 6)
    torch.cuda.synchronize()
    assert torch.equal(bufs[1], plain)
    o3, l3 = ub.varlen_fmha_fwd(q2, cu2, 512, None, 0.1, 6, 0, dropout_mask=plain)
    d3 = ub.varlen_fmha_bwd(q2, o3, l3, g2, cu2, 512, None, 0.1, 6, 0, dropout_mask=plain)
    torch.cuda.synchronize()
    assert torch.equal(o2, o3) and torch.equal(l2, l3) and torch.equal(d2, d3)


def test_bench_launch_configuration_bitwise(ub):
    """The launch configuration bench.py times -- pre-marshalled BoundFmha on capacity-sized
    buffers, persistent grid of SMs - 1 CTAs, the forward's fused pad, keep bits materialised
    once per step by BoundDropoutMask, the backward's host LPT schedule -- gives bitwise the results of the plain calls that
    test_bf16_config2_full_batch_every_sequence checks against the fp64 oracle (config 2,
    p = 0.1); the padded copy equals ub_pad of O."""
    from paper_2208_08124_b200 import api
    H, S, p, seed = 16, 512, 0.1, 0x2208
    L = synth.gen_lengths("mlperf_like_v0", 56, 0)
    lengths, off, qkv, dout, o_ref, lse_ref, d_ref, scale = _run(ub, L, H, 64, torch.bfloat16, p=p, seed=seed,
                                                                   max_seqlen=S)
    T, cap = int(off[-1]), int(off[-1]) + 300            # capacity-sized buffers, as the bench's
    cu = torch.tensor(off.astype(np.int32)).cuda()
    q = torch.zeros((cap, 3, H, 64), dtype=torch.bfloat16, device="cuda"); q[:T] = qkv.cuda()
    g = torch.zeros((cap, H, 64), dtype=torch.bfloat16, device="cuda"); g[:T] = dout.cuda()
    out = torch.empty((cap, H, 64), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((H, cap), dtype=torch.float32, device="cuda")
    dq = torch.empty((cap, 3, H, 64), dtype=torch.bfloat16, device="cuda")
    padded = torch.full((len(L), S, H, 64), 7.0, dtype=torch.bfloat16, device="cuda")
    mask = torch.empty(api.dropout_mask_bytes(cap, H, S), dtype=torch.uint8, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    bm = api.BoundDropoutMask(cu, cap, H, S, p, mask)
    bf = api.BoundFmha(q, cu, S, out, lse, dout=g, dqkv=dq, p_dropout=p, num_ctas=sms - 1, padded=padded,
                       dropout_mask=mask)
    # the host LPT schedules the bench uploads with each exchange (ub_fmha_schedule)
    bf.set_schedules(None, torch.from_numpy(api.fmha_schedule(lengths, H, S, sms - 1, True)).cuda())
    bm(T, seed)
    bf.fwd(T, seed)
    bf.bwd(T, seed)
    torch.cuda.synchronize()
    lse_v = lse.flatten()[:H * T].view(H, T)               # the bound calls use lse as a dense [H, T]
    assert torch.equal(out[:T].cpu(), o_ref) and torch.equal(lse_v.cpu(), lse_ref)
    assert torch.equal(dq[:T].cpu(), d_ref)
    assert torch.equal(padded, ub.pad(out[:T], cu, len(L), S))


@pytest.mark.parametrize("case", ["config2", "edges"])
def test_host_schedule_same_results(ub, case):
    """ub_fmha_schedule (host LPT deal of the work items) passed as prm->schedule: forward and
    backward results bitwise those of the kernels' own snake deal, at p = 0 and 0.1 (with the
    materialised mask); a schedule built for another grid size falls back to the snake deal."""
    from paper_2208_08124_b200 import api
    S = 512
    if case == "config2":
        H = 16
        L = synth.gen_lengths("mlperf_like_v0", 56, 7)
        G = torch.cuda.get_device_properties(0).multi_processor_count - 4
    else:
        H, G = 2, 8
        L = np.array([1, 127, 128, 129, 300, 512, 64, 65, 449], np.int32)
    lengths, off, qkv, dout = make_batch(L, H, 64, seed=71)
    cu = torch.tensor(off.astype(np.int32)).cuda()
    T = int(off[-1])
    q, g = qkv.cuda(), dout.cuda()
    sf = torch.from_numpy(api.fmha_schedule(lengths, H, S, G, False)).cuda()
    sb = torch.from_numpy(api.fmha_schedule(lengths, H, S, G, True)).cuda()
    wrong = torch.from_numpy(api.fmha_schedule(lengths, H, S, G - 1, True)).cuda()
    for p in (0.0, 0.1):
        m = api.dropout_mask(cu, T, H, S, p, 3, 0) if p > 0 else None
        o1, l1 = ub.varlen_fmha_fwd(q, cu, S, None, p, 3, 0, num_ctas=G, dropout_mask=m)
        d1 = ub.varlen_fmha_bwd(q, o1, l1, g, cu, S, None, p, 3, 0, num_ctas=G, dropout_mask=m)
        o2, l2 = ub.varlen_fmha_fwd(q, cu, S, None, p, 3, 0, num_ctas=G, dropout_mask=m, schedule=sf)
        d2 = ub.varlen_fmha_bwd(q, o2, l2, g, cu, S, None, p, 3, 0, num_ctas=G, dropout_mask=m, schedule=sb)
        d3 = ub.varlen_fmha_bwd(q, o2, l2, g, cu, S, None, p, 3, 0, num_ctas=G, dropout_mask=m, schedule=wrong)
        torch.cuda.synchronize()
        assert torch.equal(o1, o2) and torch.equal(l1, l2), p
        assert torch.equal(d1, d2) and torch.equal(d1, d3), p
