"""World-size-2 multi-process tests on CPU (gloo): the N>1 host logic of the exchange and
of bench.py's cross-rank reductions.  The device kernels are replaced by numpy copies that
follow the same library-built tables; the transport is gloo point-to-point in place of
the grouped ncclSend/ncclRecv (which needs GPUs)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2208_08124_b200 import api
        from oracle import balance as obal
        from oracle import exchange as oex
        import bench
        B, rec, srec = 56, 16, 4
        mine = synth.skewed_rank_lengths(world, B, 0, "sorted-block")[rank]
        # a1: all-gather of lengths
        parts = [torch.zeros(B, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(mine))
        all_l = torch.cat(parts).numpy()
        # a2-a3: every rank plans independently -> identical bytes
        plan = api.balance_plan(all_l, world, B, 512, "paper")
        perms = [torch.zeros(world * B, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(perms, torch.from_numpy(plan["perm"]))
        same = all(torch.equal(perms[0], p) for p in perms)
        ref = obal.balance_paper(all_l, world, B)
        # a4-a5: pack (tables), gloo p2p transport, unpack (tables)
        toks = synth.gen_bytes(int(mine.sum()) * rec, 40 + rank).reshape(-1, rec)
        smps = synth.gen_bytes(B * srec, 50 + rank).reshape(B, srec)
        tab, cnt, scnt, tot = api.exchange_tables(all_l, plan["perm"], world, B, rank, unpack=False)
        send_t = np.zeros((tot, rec), np.uint8); send_s = np.zeros((B, srec), np.uint8)
        for e in range(B):
            s0, n, d0, ss, ds = (int(tab[k * B + e]) for k in range(5))
            send_t[d0:d0 + n] = toks[s0:s0 + n]; send_s[ds] = smps[ss]
        utab, rcnt, rscnt, rtot = api.exchange_tables(all_l, plan["perm"], world, B, rank, unpack=True)
        recv_t = np.zeros((rtot, rec), np.uint8); recv_s = np.zeros((B, srec), np.uint8)
        # counts must agree pairwise: what r sends to d is what d receives from r
        cnts = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(cnts, torch.from_numpy(cnt))
        rc_ok = all(int(cnts[s][rank]) == int(rcnt[s]) for s in range(world))
        so = ro = sso = rso = 0
        for peer in range(world):
            st = torch.from_numpy(send_t[so:so + cnt[peer]].copy()); ss_ = torch.from_numpy(send_s[sso:sso + scnt[peer]].copy())
            rt = torch.zeros((int(rcnt[peer]), rec), dtype=torch.uint8); rs = torch.zeros((int(rscnt[peer]), srec), dtype=torch.uint8)
            if peer == rank:
                rt.copy_(st); rs.copy_(ss_)
            else:
                reqs = [dist.isend(st, peer), dist.isend(ss_, peer), dist.irecv(rt, peer), dist.irecv(rs, peer)]
                for r_ in reqs:
                    r_.wait()
            recv_t[ro:ro + rcnt[peer]] = rt.numpy(); recv_s[rso:rso + rscnt[peer]] = rs.numpy()
            so += cnt[peer]; ro += rcnt[peer]; sso += scnt[peer]; rso += rscnt[peer]
        out_t = np.zeros((rtot, rec), np.uint8); out_s = np.zeros((B, srec), np.uint8)
        for e in range(B):
            s0, n, d0, ss, ds = (int(utab[k * B + e]) for k in range(5))
            out_t[d0:d0 + n] = recv_t[s0:s0 + n]; out_s[ds] = recv_s[ss]
        # oracle on the full (gathered) data
        all_toks = [None] * world; all_smps = [None] * world
        lens2 = all_l.reshape(world, B)
        for r in range(world):
            all_toks[r] = synth.gen_bytes(int(lens2[r].sum()) * rec, 40 + r).reshape(-1, rec)
            all_smps[r] = synth.gen_bytes(B * srec, 50 + r).reshape(B, srec)
        exp = oex.exchange(lens2, all_toks, all_smps, ref["perm"], world, B)[rank]
        # bench.py reductions across ranks
        mx = bench.all_max(float(rank + 1), world)
        sm = bench.all_sum(float(rank + 1), world)
        gl = bench.all_gather_list(float(rank), world)
        q.put((rank, same, np.array_equal(plan["perm"], ref["perm"]), rc_ok,
               np.array_equal(out_t, exp["tokens"]), np.array_equal(out_s, exp["samples"]),
               obal.imbalance(plan["rank_tokens"]), mx, sm, gl))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_exchange_two_ranks_gloo(world):
    from paper_2208_08124_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2208_08124_b200 import build
        build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, plan_ok, rc_ok, tok_ok, smp_ok, imb, mx, sm, gl in res:
        assert same and plan_ok and rc_ok and tok_ok and smp_ok, rank
        assert imb <= 0.05
        assert mx == world and sm == world * (world + 1) / 2 and gl == [float(r) for r in range(world)]
