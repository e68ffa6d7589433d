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


@pytest.mark.parametrize("W,rec,srec", [(2, 16, 4), (4, 16, 4), (8, 16, 4), (3, 2048, 8), (5, 6, 3)])
def test_exchange_pack_transport_unpack_virtual_ranks(ub, W, rec, srec):
    """W virtual ranks on one GPU: pack (kernel) -> transport (per-peer slices, as the
    grouped ncclSend/ncclRecv moves them) -> unpack (kernel); bytes equal the oracle."""
    B = 56 if rec <= 16 else 9
    lens = synth.skewed_rank_lengths(W, B, 0, "sorted-block")
    toks = [synth.gen_bytes(int(lens[r].sum()) * rec, 70 + r).reshape(-1, rec) for r in range(W)]
    smps = [synth.gen_bytes(B * srec, 80 + r).reshape(B, srec) for r in range(W)]
    plan = ub.balance_plan(lens.reshape(-1), W, B, 512, "paper")
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


def test_nccl_balance_exchange_single_rank(ub):
    """The full NCCL path (all-gather, plan, pack, grouped send/recv, unpack, cu H2D) at
    W=1 on the one GPU this run has: the output is the paper's sorted order."""
    B, rec, srec = 56, 16, 4
    lens = synth.gen_lengths("mlperf_like_v0", B, 5)
    toks = synth.gen_bytes(int(lens.sum()) * rec, 91).reshape(-1, rec)
    smps = synth.gen_bytes(B * srec, 92).reshape(B, srec)
    comm = ub.Comm(1, 0)
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
    comm.close()
