"""Unpad / pad and the exchange copy kernels: bit-exact vs the oracle.  -m gpu."""
import numpy as np
import pytest
import torch

import synth
from oracle import balance as obal
from oracle import exchange as oex
from oracle import varlen as ovar

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ub():
    import paper_2208_08124_b200 as ub
    assert torch.cuda.is_available()
    return ub


@pytest.mark.parametrize("row_shape,dtype", [((1024,), torch.bfloat16), ((3, 16, 64), torch.bfloat16),
                                             ((4,), torch.int32), ((1,), torch.int32), ((3,), torch.uint8),
                                             ((5,), torch.float32)])
def test_unpad_pad_bit_exact(ub, row_shape, dtype):
    lengths = synth.gen_lengths("mlperf_like_v0", 56, 3)
    lengths[0], lengths[1] = 1, 512
    B, S = len(lengths), 512
    off = ovar.batch_offset(lengths)
    T = int(off[-1])
    g = torch.Generator().manual_seed(5)
    if dtype.is_floating_point:
        padded = torch.randn((B, S) + row_shape, generator=g).to(dtype)
    else:
        padded = torch.randint(0, 120, (B, S) + row_shape, generator=g).to(dtype)
    cu = torch.tensor(off.astype(np.int32)).cuda()
    packed = ub.unpad(padded.cuda(), cu, T)
    exp = ovar.unpad(padded.view(torch.uint8).numpy() if dtype != torch.uint8 else padded.numpy(), lengths)
    got = packed.cpu()
    got = got.view(torch.uint8).numpy() if dtype != torch.uint8 else got.numpy()
    assert np.array_equal(got, exp)
    # pad with zeros and with a pattern row
    back = ub.pad(packed, cu, B, S).cpu()
    ref = padded.clone()
    for b in range(B):
        ref[b, lengths[b]:] = 0
    assert torch.equal(back.view(torch.uint8), ref.view(torch.uint8))
    pad_row = torch.full(row_shape, 7, dtype=dtype)
    back2 = ub.pad(packed, cu, B, S, pad_row=pad_row.cuda()).cpu()
    exp2 = ovar.pad(packed.cpu().view(torch.uint8).numpy() if dtype != torch.uint8 else packed.cpu().numpy(), off, S,
                    pad_row.view(torch.uint8).numpy() if dtype != torch.uint8 else pad_row.numpy())
    got2 = back2.view(torch.uint8).numpy() if dtype != torch.uint8 else back2.numpy()
    assert np.array_equal(got2, exp2)


@pytest.mark.parametrize("words", [4, 12])
def test_span_bulk_chunks_cross_sequences(ub, words):
    # TMA bulk path (16-B rows): 32 KB chunks that hold many short sequences, chunk ends in
    # the middle of a row (48-B rows), empty sequences in both the packed and the zero space
    rng = np.random.default_rng(words)
    lengths = rng.integers(0, 40, 300).astype(np.int32)
    lengths[[0, 7, 8, 299]] = 0
    lengths[5] = 512
    B, S = len(lengths), 512
    off = np.concatenate([[0], np.cumsum(lengths)])      # (the oracle rejects L = 0, R8: sliced here)
    T = int(off[-1])
    padded = rng.integers(-2**31, 2**31 - 1, (B, S, words), dtype=np.int64).astype(np.int32)
    cu = torch.tensor(off.astype(np.int32)).cuda()
    packed = ub.unpad(torch.from_numpy(padded).cuda(), cu, T)
    exp = np.concatenate([padded[b, :lengths[b]] for b in range(B)])
    assert np.array_equal(packed.cpu().numpy(), exp)
    back = ub.pad(packed, cu, B, S).cpu().numpy()
    ref = np.zeros_like(padded)
    for b in range(B):
        ref[b, :lengths[b]] = exp[off[b]:off[b + 1]]
    assert np.array_equal(back, ref)


def test_span_vector_kernel_when_bulk_off():
    # UB_SPAN_BULK=0 selects the LDG/STG span kernel (read once per process): a subprocess
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, synth\n"
        "import paper_2208_08124_b200 as ub\n"
        "from oracle import varlen as ovar\n"
        "L = synth.gen_lengths('mlperf_like_v0', 56, 9); L[3] = 1\n"
        "off = ovar.batch_offset(L); T = int(off[-1])\n"
        "p = torch.randint(0, 255, (56, 512, 64), dtype=torch.uint8)\n"
        "cu = torch.tensor(off.astype(np.int32)).cuda()\n"
        "k = ub.unpad(p.cuda(), cu, T)\n"
        "assert np.array_equal(k.cpu().numpy(), ovar.unpad(p.numpy(), L))\n"
        "b = ub.pad(k, cu, 56, 512).cpu().numpy()\n"
        "assert np.array_equal(b, ovar.pad(k.cpu().numpy(), off, 512, np.zeros(64, np.uint8)))\n"
        "print('ok')\n")
    import os
    env = dict(os.environ, UB_SPAN_BULK="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


def test_unpad_unaligned_and_errors(ub):
    from paper_2208_08124_b200._lib import UbError
    lengths = np.array([3, 1, 4], np.int32)
    off = ovar.batch_offset(lengths)
    padded = torch.arange(3 * 5 * 3, dtype=torch.uint8).reshape(3, 5, 3)
    cu = torch.tensor(off.astype(np.int32)).cuda()
    big = torch.zeros(1 + 3 * 5 * 3, dtype=torch.uint8).cuda()
    view = big[1:].view(3, 5, 3)                          # 1-B misaligned base
    view.copy_(padded.cuda())
    packed = ub.unpad(view, cu, int(off[-1])).cpu().numpy()
    assert np.array_equal(packed, ovar.unpad(padded.numpy(), lengths))
    with pytest.raises(UbError) as e:
        ub.unpad(view, cu, 16)                            # T > B*S
    assert e.value.status == 3


@pytest.mark.parametrize("W,rec,srec,mode", [(2, 16, 4, "paper"), (4, 16, 4, "paper"), (8, 16, 4, "paper"),
                                              (3, 2048, 8, "paper"), (5, 6, 3, "paper"), (8, 16, 4, "lpt"),
                                              (3, 2048, 8, "lpt")])
def test_exchange_pack_transport_unpack_virtual_ranks(ub, W, rec, srec, mode):
    """W virtual ranks on one GPU: pack (kernel) -> transport (per-peer slices, as the
    grouped ncclSend/ncclRecv moves them) -> unpack (kernel); bytes equal the oracle
    (paper plan, and the LPT plan of reading R20)."""
    B = 56 if rec <= 16 else 9
    lens = synth.skewed_rank_lengths(W, B, 0, "sorted-block")
    toks = [synth.gen_bytes(int(lens[r].sum()) * rec, 70 + r).reshape(-1, rec) for r in range(W)]
    smps = [synth.gen_bytes(B * srec, 80 + r).reshape(B, srec) for r in range(W)]
    plan = ub.balance_plan(lens.reshape(-1), W, B, 512, mode)
    ref = (obal.balance_paper if mode == "paper" else obal.balance_lpt)(lens.reshape(-1), W, B)
    assert np.array_equal(np.asarray(plan["perm"], np.int64), np.asarray(ref["perm"], np.int64))
    exp = oex.exchange(lens, toks, smps, plan["perm"], W, B)
    send = []
    for r in range(W):
        tab, cnt, scnt, tot = ub.exchange_tables(lens.reshape(-1), plan["perm"], W, B, r, unpack=False)
        st = torch.empty((tot, rec), dtype=torch.uint8, device="cuda")
        ss = torch.empty((B, srec), dtype=torch.uint8, device="cuda")
        ub.exchange_copy(torch.from_numpy(toks[r]).cuda(), st, torch.from_numpy(smps[r]).cuda(), ss,
                         torch.from_numpy(tab).cuda(), B, rec, srec)
        send.append((st, ss, cnt, scnt))
    for d in range(W):
        ct, cs = [], []
        for s in range(W):
            st, ss, cnt, scnt = send[s]
            o, so = int(cnt[:d].sum()), int(scnt[:d].sum())
            ct.append(st[o:o + int(cnt[d])]); cs.append(ss[so:so + int(scnt[d])])
        rt, rs = torch.cat(ct), torch.cat(cs)
        tab, cnt, scnt, tot = ub.exchange_tables(lens.reshape(-1), plan["perm"], W, B, d, unpack=True)
        ot = torch.empty((tot, rec), dtype=torch.uint8, device="cuda")
        os_ = torch.empty((B, srec), dtype=torch.uint8, device="cuda")
        ub.exchange_copy(rt, ot, rs, os_, torch.from_numpy(tab).cuda(), B, rec, srec)
        torch.cuda.synchronize()
        assert np.array_equal(ot.cpu().numpy(), exp[d]["tokens"])
        assert np.array_equal(os_.cpu().numpy(), exp[d]["samples"])
        assert tot == plan["rank_tokens"][d]
        if B == 56:
            assert obal.imbalance(plan["rank_tokens"]) <= 0.05   # BASELINE gate (B = 56)


@pytest.mark.parametrize("force_nccl", [False, True])
def test_nccl_balance_exchange_single_rank(ub, force_nccl):
    """The full exchange (all-gather, plan, pack, grouped send/recv, unpack, cu H2D) at W=1
    on the one GPU this run has: the output is the paper's sorted order.  force_nccl routes
    the one-rank all-gather and the self chunk through ncclAllGather / ncclSend+ncclRecv
    (UB_COMM_FORCE_NCCL): the collective data plane itself moves the bytes."""
    B, rec, srec = 56, 16, 4
    lens = synth.gen_lengths("mlperf_like_v0", B, 5)
    toks = synth.gen_bytes(int(lens.sum()) * rec, 91).reshape(-1, rec)
    smps = synth.gen_bytes(B * srec, 92).reshape(B, srec)
    comm = ub.Comm(1, 0)
    comm.set_options(force_nccl=force_nccl)
    side = torch.cuda.Stream()
    ot, os_, ocu, T, perm = comm.balance_exchange(torch.from_numpy(lens).cuda(), torch.from_numpy(toks).cuda(),
                                                  torch.from_numpy(smps).cuda(), int(lens.sum()), 512, stream=side)
    side.synchronize()
    plan = obal.balance_paper(lens, 1, B)
    exp = oex.exchange(lens.reshape(1, B), [toks], [smps], plan["perm"], 1, B)[0]
    assert np.array_equal(perm, plan["perm"])
    assert T == int(lens.sum())
    assert np.array_equal(ot[:T].cpu().numpy(), exp["tokens"])
    assert np.array_equal(os_.cpu().numpy(), exp["samples"])
    assert np.array_equal(ocu.cpu().numpy(), exp["cu"])
    # all-gather + token send + token recv + sample send + sample recv when forced; none otherwise
    assert comm.nccl_ops() == (5 if force_nccl else 0)
    comm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("force_nccl", [False, True])
def test_nccl_exchange_two_phase_pipelined(ub, force_nccl):
    """ub_exchange_begin / ub_exchange_finish with several batches in flight (the bench's
    pipeline: begin n+2 before finish n+1) give what the oracle's exchange gives per batch,
    with the copies or (force_nccl) NCCL itself moving the data."""
    B, rec, srec = 56, 16, 4
    comm = ub.Comm(1, 0)
    comm.set_options(force_nccl=force_nccl, host_profile=True)
    side = torch.cuda.Stream()
    batches = []
    for k in range(6):
        lens = synth.gen_lengths(["mlperf_like_v0", "uniform", "bimodal"][k % 3], B, 40 + k)
        toks = synth.gen_bytes(int(lens.sum()) * rec, 140 + k).reshape(-1, rec)
        smps = synth.gen_bytes(B * srec, 240 + k).reshape(B, srec)
        batches.append((lens, toks, smps, torch.from_numpy(lens).cuda(), torch.from_numpy(toks).cuda(),
                        torch.from_numpy(smps).cuda()))
    cap = max(int(b[0].sum()) for b in batches)
    outs = [(torch.empty((cap, rec), dtype=torch.uint8, device="cuda"), torch.empty((B, srec), dtype=torch.uint8,
             device="cuda"), torch.empty(B + 1, dtype=torch.int32, device="cuda")) for _ in batches]
    comm.exchange_begin(0, batches[0][3], cap, rec, srec, stream=side)
    comm.exchange_begin(1, batches[1][3], cap, rec, srec, stream=side)
    res = []
    for k in range(len(batches)):
        ot, os_, ocu = outs[k]
        res.append(comm.exchange_finish(k % comm.SLOTS, B, batches[k][4], batches[k][5], cap, 512, "paper", ot, os_,
                                        ocu, stream=side))
        if k + 2 < len(batches):
            comm.exchange_begin((k + 2) % comm.SLOTS, batches[k + 2][3], cap, rec, srec, stream=side)
    side.synchronize()
    for k, (lens, toks, smps, *_) in enumerate(batches):
        T, perm = res[k]
        plan = obal.balance_paper(lens, 1, B)
        exp = oex.exchange(lens.reshape(1, B), [toks], [smps], plan["perm"], 1, B)[0]
        assert np.array_equal(perm, plan["perm"]) and T == int(lens.sum())
        ot, os_, ocu = outs[k]
        assert np.array_equal(ot[:T].cpu().numpy(), exp["tokens"])
        assert np.array_equal(os_.cpu().numpy(), exp["samples"])
        assert np.array_equal(ocu.cpu().numpy(), exp["cu"])
    assert comm.nccl_ops() == (5 * len(batches) if force_nccl else 0)
    prof = comm.host_profile()                      # UB_COMM_HOST_PROFILE: one sample per finish
    assert prof["finishes"] == len(batches)
    assert all(prof[k] >= 0.0 for k in comm.HOST_PHASES) and prof["plan"] > 0.0
    # misuse: finish without a begin, begin on a busy slot, slot out of range
    d = batches[0]
    with pytest.raises(ub.UbError):
        comm.exchange_finish(3, B, d[4], d[5], cap, 512, "paper", *outs[0], stream=side)
    comm.exchange_begin(3, d[3], cap, rec, srec, stream=side)
    with pytest.raises(ub.UbError):
        comm.exchange_begin(3, d[3], cap, rec, srec, stream=side)
    with pytest.raises(ub.UbError):
        comm.exchange_begin(comm.SLOTS, d[3], cap, rec, srec, stream=side)
    comm.exchange_finish(3, B, d[4], d[5], cap, 512, "paper", *outs[0], stream=side)
    side.synchronize()
    comm.close()


@pytest.mark.gpu
def test_exchange_emits_fmha_schedule(ub):
    """ub_exchange_slot_lengths / ub_exchange_fmha_schedule: after a finish, the slot's all-gathered
    lengths are the batch's, and the schedule the exchange emits (host copy and its upload) is
    ub_fmha_schedule of the delivered batch's lengths (perm order)."""
    from paper_2208_08124_b200 import api
    B, rec, srec, H, S, G = 56, 16, 4, 16, 512, 144
    lens = synth.gen_lengths("mlperf_like_v0", B, 77)
    comm = ub.Comm(1, 0)
    side = torch.cuda.Stream()
    cap = int(lens.sum())
    dl = torch.from_numpy(lens).cuda()
    toks = torch.zeros((cap, rec), dtype=torch.uint8, device="cuda")
    smps = torch.zeros((B, srec), dtype=torch.uint8, device="cuda")
    outs = (torch.empty((cap, rec), dtype=torch.uint8, device="cuda"), torch.empty((B, srec), dtype=torch.uint8,
            device="cuda"), torch.empty(B + 1, dtype=torch.int32, device="cuda"))
    comm.exchange_begin(2, dl, cap, rec, srec, stream=side)
    T, perm = comm.exchange_finish(2, B, toks, smps, cap, S, "paper", *outs, stream=side)
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    assert np.array_equal(comm.slot_lengths(2, B), lens)
    delivered = lens[perm[:B]]
    for is_bwd in (True, False):
        n = api.lib().ub_fmha_schedule_ints(B, H, S, G, 1 if is_bwd else 0)
        hs = torch.zeros(n, dtype=torch.int32).pin_memory()
        ds = torch.full((n,), -1, dtype=torch.int32, device="cuda")
        comm.bind_fmha_schedule(2, perm, B, H, S, G, is_bwd, hs, ds, stream=side)()
        side.synchronize()
        exp = api.fmha_schedule(delivered, H, S, G, is_bwd)
        assert np.array_equal(hs.numpy(), exp) and np.array_equal(ds.cpu().numpy(), exp)
    comm.close()
