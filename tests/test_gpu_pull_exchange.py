"""NEXT-3 pull exchange on the GPU: two processes on one device (CUDA IPC maps a buffer of
another process on the same GPU exactly as it maps a peer GPU's over NVLink), host
coordination over gloo.  Every rank pulls its perm-ordered samples out of both ranks'
packed buffers with ub_exchange_pull; the bytes must equal the oracle exchange
(oracle/exchange.py) bit for bit."""
import os
import socket
import sys

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(W, B, rec, srec):
    sys.path.insert(0, ROOT)
    import synth
    lens = synth.gen_lengths("mlperf_like_v0", W * B, 21).reshape(W, B)
    toks = [synth.gen_bytes(int(lens[r].sum()) * rec, 90 + r).reshape(-1, rec) for r in range(W)]
    smps = [synth.gen_bytes(B * srec, 95 + r).reshape(B, srec) for r in range(W)]
    return lens, toks, smps


def _worker(rank, W, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=W)
    try:
        from paper_2208_08124_b200 import api
        from oracle import exchange as oex
        B, rec, srec = 9, 16, 4
        lens, toks, smps = _case(W, B, rec, srec)
        dev = torch.device("cuda", 0)
        my_t = torch.from_numpy(toks[rank]).to(dev)
        my_s = torch.from_numpy(smps[rank]).to(dev)
        torch.cuda.synchronize()
        handles = [None] * W
        dist.all_gather_object(handles, (api.ipc_export(my_t), api.ipc_export(my_s)))
        ptr_t, ptr_s, bases = [], [], []
        for r in range(W):
            if r == rank:
                ptr_t.append(my_t.data_ptr()); ptr_s.append(my_s.data_ptr())
            else:
                pt, bt = api.ipc_import(handles[r][0]); ps, bs = api.ipc_import(handles[r][1])
                ptr_t.append(pt); ptr_s.append(ps); bases += [bt, bs]
        plan = api.balance_plan(lens.reshape(-1), W, B, 512, "paper")
        tab, tot = api.exchange_pull_table(lens.reshape(-1), plan["perm"], W, B, rank)
        d_tab = torch.from_numpy(tab).to(dev)
        out_t = torch.zeros((tot, rec), dtype=torch.uint8, device=dev)
        out_s = torch.zeros((B, srec), dtype=torch.uint8, device=dev)
        api.exchange_pull(torch.tensor(ptr_t, dtype=torch.int64, device=dev),
                          torch.tensor(ptr_s, dtype=torch.int64, device=dev), d_tab, B, rec, srec, out_t, out_s)
        torch.cuda.synchronize()
        exp = oex.exchange(lens, toks, smps, plan["perm"], W, B)[rank]
        ok = bool(np.array_equal(out_t.cpu().numpy(), exp["tokens"]) and np.array_equal(out_s.cpu().numpy(), exp["samples"]))
        dist.barrier()                                   # every rank done reading the peers
        for b in bases:
            api.ipc_close(b)
        dist.barrier()                                   # mappings closed before buffers go
        q.put((rank, ok, None))
    except Exception as e:                               # reported to the parent
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def test_pull_exchange_two_processes_one_gpu():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    W, port = 2, _port()
    procs = [ctx.Process(target=_worker, args=(r, W, port, q)) for r in range(W)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(W)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in sorted(res):
        assert ok, f"rank {rank}: {err}"


def test_pull_exchange_one_rank_is_the_reorder():
    """W = 1: the pull is the a5 reorder of the rank's own batch."""
    from paper_2208_08124_b200 import api
    from oracle import exchange as oex
    B, rec, srec = 11, 16, 4
    lens, toks, smps = _case(1, B, rec, srec)
    plan = api.balance_plan(lens.reshape(-1), 1, B, 512, "paper")
    tab, tot = api.exchange_pull_table(lens.reshape(-1), plan["perm"], 1, B, 0)
    t = torch.from_numpy(toks[0]).cuda(); s = torch.from_numpy(smps[0]).cuda()
    out_t = torch.zeros((tot, rec), dtype=torch.uint8, device="cuda")
    out_s = torch.zeros((B, srec), dtype=torch.uint8, device="cuda")
    api.exchange_pull(torch.tensor([t.data_ptr()], dtype=torch.int64, device="cuda"),
                      torch.tensor([s.data_ptr()], dtype=torch.int64, device="cuda"),
                      torch.from_numpy(tab).cuda(), B, rec, srec, out_t, out_s)
    exp = oex.exchange(lens, toks, smps, plan["perm"], 1, B)[0]
    assert np.array_equal(out_t.cpu().numpy(), exp["tokens"]) and np.array_equal(out_s.cpu().numpy(), exp["samples"])


def _pipelined_worker(rank, W, port, q):
    """Several steps through a 2-slot ring with device-side flags only: no host barrier
    between a rank writing its buffer and the peers pulling from it."""
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=W)
    try:
        import synth
        from paper_2208_08124_b200 import api
        from oracle import exchange as oex
        B, rec, srec, S, N = 7, 16, 4, 2, 6
        dev = torch.device("cuda", 0)
        steps = []
        for n in range(N):
            lens = synth.gen_lengths("mlperf_like_v0", W * B, 100 + n).reshape(W, B)
            toks = [synth.gen_bytes(int(lens[r].sum()) * rec, 1000 + 10 * n + r).reshape(-1, rec) for r in range(W)]
            smps = [synth.gen_bytes(B * srec, 2000 + 10 * n + r).reshape(B, srec) for r in range(W)]
            plan = api.balance_plan(lens.reshape(-1), W, B, 512, "paper")
            steps.append((lens, toks, smps, plan))
        cap = max(int(l.sum()) for st in steps for l in st[0])
        tok = torch.zeros((S, cap, rec), dtype=torch.uint8, device=dev)
        smp = torch.zeros((S, B, srec), dtype=torch.uint8, device=dev)
        flags = torch.zeros(2 * S, dtype=torch.int32, device=dev)     # ready[S], done[S]
        torch.cuda.synchronize()
        handles = [None] * W
        dist.all_gather_object(handles, tuple(api.ipc_export(t) for t in (tok, smp, flags)))
        bases, base_ptr = [], []
        for r in range(W):
            if r == rank:
                base_ptr.append((tok.data_ptr(), smp.data_ptr(), flags.data_ptr()))
                continue
            ptrs = []
            for h in handles[r]:
                p, b = api.ipc_import(h)
                ptrs.append(p); bases.append(b)
            base_ptr.append(tuple(ptrs))
        dist.barrier()                                   # every mapping exists before any use
        i64 = lambda xs: torch.tensor(xs, dtype=torch.int64, device=dev)
        peer_tok = [i64([bp[0] + k * cap * rec for bp in base_ptr]) for k in range(S)]
        peer_smp = [i64([bp[1] + k * B * srec for bp in base_ptr]) for k in range(S)]
        ready = [i64([bp[2] + 4 * k for bp in base_ptr]) for k in range(S)]
        done = [i64([bp[2] + 4 * (S + k) for bp in base_ptr]) for k in range(S)]
        outs = []
        for n, (lens, toks, smps, plan) in enumerate(steps):
            k = n % S
            if n >= S:                                   # peers finished pulling step n - S
                api.wait_flags(done[k], n - S + 1)
            t = torch.from_numpy(toks[rank]).to(dev, non_blocking=False)
            tok[k, :t.shape[0]].copy_(t)
            smp[k].copy_(torch.from_numpy(smps[rank]).to(dev))
            api.signal(flags[k:k + 1], n + 1)            # publish this rank's buffer of step n
            tab, tot = api.exchange_pull_table(lens.reshape(-1), plan["perm"], W, B, rank)
            out_t = torch.zeros((tot, rec), dtype=torch.uint8, device=dev)
            out_s = torch.zeros((B, srec), dtype=torch.uint8, device=dev)
            api.exchange_pull(peer_tok[k], peer_smp[k], torch.from_numpy(tab).to(dev), B, rec, srec, out_t, out_s,
                              d_ready=ready[k], wait_value=n + 1)
            api.signal(flags[S + k:S + k + 1], n + 1)    # this rank is done reading slot k of step n
            outs.append((out_t, out_s))
        torch.cuda.synchronize()
        ok = True
        for n, (lens, toks, smps, plan) in enumerate(steps):
            exp = oex.exchange(lens, toks, smps, plan["perm"], W, B)[rank]
            ok = ok and np.array_equal(outs[n][0].cpu().numpy(), exp["tokens"]) and \
                np.array_equal(outs[n][1].cpu().numpy(), exp["samples"])
        dist.barrier()
        for b in bases:
            api.ipc_close(b)
        dist.barrier()
        q.put((rank, bool(ok), None))
    except Exception as e:
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def test_pull_exchange_pipelined_with_device_flags():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    W, port = 2, _port()
    procs = [ctx.Process(target=_pipelined_worker, args=(r, W, port, q)) for r in range(W)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(W)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in sorted(res):
        assert ok, f"rank {rank}: {err}"
