#!/usr/bin/env python
"""bench.py -- the unpadded-BERT hot path (arXiv 2208.08124) on B200, one JSON line.

A step is one pass of every row of SURVEY.md §8(a) over one 56-sequence BERT-large batch
per GPU (H=16, D=64, max_seqlen 512, MLPerf-like length mix, bf16):
  side stream (while step n computes, step n+1 is exchanged and the lengths of
  step n+2 are gathered, so the host never waits on work it has just enqueued):
    a1         exchange_begin: NCCL all-gather of lengths + D2H into a pinned slot
    a6 unpad   padded input records [56, 512, 16 B] -> packed [T, 16 B]
    a2-a5      exchange_finish: host plan (sort + interleave), pack, grouped
               ncclSend/ncclRecv, reorder, cu_seqlens H2D
  main stream:
    a7 varlen FMHA forward over the exchanged cu_seqlens
    a9 pad     attention output [T, 1024] -> [56, 512, 1024], fused into a7's
               epilogue (ub_varlen_fmha_fwd_pad; zeros past each length)
    a8 varlen FMHA backward (dO given)
Metric (BASELINE.json): unpadded FMHA fwd+bwd tokens/s, with the roofline fraction of the
dominant kernel and the 8-GPU token imbalance.

Usage: python bench.py --gpus N --steps K --warmup W [--impl reference]
       (N > 1: torchrun --nproc-per-node N ... bench.py --gpus N ...)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time


def _claim_stdout():
    """stdout carries exactly one JSON line: keep a private handle on it and point fd 1 at
    stderr, so that library banners written straight to fd 1 (NCCL prints its version there
    at communicator init) cannot land on it."""
    sys.stdout.flush()
    out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    return out

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

H, D, S, B = 16, 64, 512, 56
REC = 16      # per-token record: input_id, segment_id, masked_lm_label, position (int32 x 4)
SREC = 4      # per-sample record: next_sentence_label (int32)
N_SETS = 3    # rotating input sets: each step's working set (> 300 MB) and the 2 others exceed L2
PIPE = int(os.environ.get("UB_BENCH_PIPE", "3"))   # step n computes while step n+PIPE is exchanged and n+PIPE+1's lengths are gathered
N_EX = PIPE + 2   # exchange output buffers in flight: the side stream never waits on the step just enqueued
KERNELS_PER_STEP = 5    # ours at W = 1: unpad, exchange gather, fwd main (+ fused pad), bwd pre (Delta) + main,
                        # plus the dropout-mask kernel when p > 0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)   # 100 steps of ~0.23 ms: a stable mean
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dist", default="mlperf_like_v0", choices=list(synth.DISTRIBUTIONS))
    ap.add_argument("--p-dropout", type=float, default=0.1,
                    help="attention dropout of the headline step: 0.1, BERT-large's value, as SURVEY §8(d) "
                         "names the headline; the same step at p = 0 is reported beside it (p0_step)")
    ap.add_argument("--balance", default="paper",
                    choices=["paper", "snake", "lpt", "stay", "paper+locality", "snake+locality", "lpt+locality"])
    ap.add_argument("--skew", default="iid", choices=["iid", "sorted-block"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-encoder", action="store_true", help="skip the NEXT-1 encoder sub-layer measurement")
    ap.add_argument("--prof-every", type=int, default=0,
                    help="record the per-kernel events on every k-th step of the headline region; 0 (default): "
                         "the headline region runs uninstrumented (event records between kernels block their "
                         "programmatic-dependent-launch overlap, ~13 us per step) and the per-kernel times come "
                         "from a separate instrumented region of the same steps")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--mask-overlap", type=int, default=1,
                    help="launch step n+1's dropout mask right behind step n's backward (UB_MASK_OVERLAP_PREVIOUS)")
    ap.add_argument("--schedule", type=int, default=1,
                    help="host LPT schedule of the backward's work items (ub_fmha_schedule, from the "
                         "exchange's lengths, uploaded with the exchange; 2: the forward's too); 0: the "
                         "kernels' snake deal (same results)")
    ap.add_argument("--reserve-sms", type=int, default=1,
                    help="SMs the persistent FMHA grid leaves to the side-stream exchange (r02c: 0 left the "
                         "side-stream copies no SM while the FMHA kernels ran: 280 vs 214 us per step; with "
                         "the backward's LPT schedule 1 / 2 / 4: median step 219 / 222 / 222 us)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "nccl-forced"],
                    help="nccl-forced: the self chunk / one-rank all-gather also go through NCCL (UB_COMM_FORCE_NCCL)")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm": d["hbm_gbs"], "bf16": d["bf16_tflops"], "bf16_sust": d.get("bf16_tflops_sustained"),
                "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sust": 1400.0, "src": "fallback (B200_PROFILING.md)"}


def load_traffic():
    """dram bytes per launch from the committed ncu --set full summary, if present."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        return json.load(f).get("dram_bytes_per_launch", {})


def load_tensor_pipe():
    """ncu sm__pipe_tensor_cycles_active (% of peak, active cycles) per FMHA kernel from the
    newest round in the committed summary -- the TC-utilisation evidence BASELINE names."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        rounds = json.load(f).get("rounds", {})
    if not rounds:
        return {}
    tag = sorted(rounds)[-1]
    key = "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
    out = {"round": tag}
    for k in ("fmha_fwd", "fmha_bwd"):
        v = rounds[tag].get(k, {}).get(key)
        if v:
            out[k] = float(v["value"])
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc, self.path = index, None, None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [x for x in sm if x > 0.5 * (max(sm) if sm else 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_init(n):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={world} (launch N>1 with torchrun)")
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _red_dev():
    import torch.distributed as dist
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def all_max(x, world):
    """Max over ranks (timing: the job is as slow as its slowest rank)."""
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_red_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_sum(x, world):
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_red_dev())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def all_gather_list(x, world):
    if world == 1:
        return [x]
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_red_dev())
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [float(o.item()) for o in out]


def rank_lengths(args, world, rank, s):
    return synth.skewed_rank_lengths(world, B, s, args.skew, args.dist)[rank]


def rooflines(peaks, clk, ctas, lens_list, fwd_us, bwd_us, padded_fwd=True):
    """Per-kernel roofline: the kernel's time floor is the max of its tensor
    floor (strict algorithmic flops: fwd 4 H D sum L^2, bwd 8 H D sum L^2, at the measured
    BURST bf16 peak -- the timed region is milliseconds long at full clocks), its HBM floor
    (compulsory bytes: fwd 8256 B/token + the fused pad's padded rows B S H D 2, bwd 16448
    B/token) and its MUFU floor (H sum L^2 exp2, 16 per clock per SM on the SMs the kernel
    runs on, at the SM clock sampled during the run).  `bound` names the binding floor,
    `achieved` / `peak` are in that resource's unit, `frac` = floor / measured time; the
    tensor fraction is reported beside it whatever binds."""
    s2 = float(np.mean([float((np.asarray(L, np.float64) ** 2).sum()) for L in lens_list]))
    T = float(np.mean([float(np.sum(L)) for L in lens_list]))
    mhz = clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0
    mufu_rate = 16.0 * ctas * mhz * 1e6                       # exp2 / s
    tc_peak = peaks["bf16"] * 1e12
    bw = peaks["hbm"] * 1e9
    out = {}
    for name, us, fl, by in (("fwd", fwd_us, 4.0 * H * D * s2, 8256.0 * T + (B * S * H * D * 2 if padded_fwd else 0)),
                             ("bwd", bwd_us, 8.0 * H * D * s2, 16448.0 * T)):
        ex = H * s2
        floors = {"tensor": fl / tc_peak * 1e6, "hbm": by / bw * 1e6, "alu": ex / mufu_rate * 1e6}
        bound = max(floors, key=floors.get)
        t = us * 1e-6
        ach = {"tensor": (fl / t / 1e12, peaks["bf16"], "TFLOP/s"), "hbm": (by / t / 1e9, peaks["hbm"], "GB/s"),
               "alu": (ex / t / 1e9, mufu_rate / 1e9, "Gexp2/s")}[bound]
        out[name] = {"kernel": f"fmha_{name}_kernel", "bound": bound, "achieved": round(ach[0], 1),
                     "peak": round(ach[1], 1), "unit": ach[2], "frac": round(floors[bound] / us, 4),
                     "us": round(us, 2), "floors_us": {k: round(v, 2) for k, v in floors.items()},
                     "tensor_frac": round(fl / t / 1e12 / peaks["bf16"], 4),
                     "algorithmic": {"flops": fl, "bytes": by, "exp2": ex},
                     "peak_source": peaks["src"] + " (bf16: burst bf16_tflops; hbm: hbm_gbs; MUFU: 16 ex2/clk/SM "
                                                   f"(measured, scripts/ubench_ex2.cu) x {ctas} SMs x {mhz:.0f} MHz)"}
    return out


def flops_fwd(L):
    return 4.0 * H * D * float(np.sum(np.asarray(L, np.float64) ** 2))


def flops_bwd(L):
    return 8.0 * H * D * float(np.sum(np.asarray(L, np.float64) ** 2))


# ------------------------------------------------------------------ oracle legs
def oracle_sample(qkv_cpu, dout_cpu, L, seqs, scale):
    """fwd + bwd of the fp64 oracle on the listed sequences; returns tokens processed."""
    from oracle import attention as oatt
    from oracle import varlen as ovar
    off = ovar.batch_offset(L)
    q64 = qkv_cpu.double().numpy()
    g64 = dout_cpu.double().numpy()
    tok = 0
    for b in seqs:
        s, e = int(off[b]), int(off[b + 1])
        sub = np.array([0, e - s])
        oatt.varlen_fwd(q64[s:e], sub, e - s, scale)
        oatt.varlen_bwd(q64[s:e], g64[s:e], sub, e - s, scale)
        tok += e - s
    return tok


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((int(i.get("num_threads", 1)) for i in threadpool_info()), default=1)
    except Exception:
        return None


def cpu_baseline(args, seconds):
    """The oracle as it stands, timed on this host's cores on a bounded sample of the
    workload (sequences of batch 0 in order, fwd+bwd, until `seconds` elapse), and again
    with its BLAS limited to one thread on a shorter sample."""
    L = synth.gen_lengths(args.dist, B, 100)
    T = int(L.sum())
    qkv = synth.gen_normal((T, 3, H, D), 1000)
    dout = synth.gen_normal((T, H, D), 2000)
    cores = len(os.sched_getaffinity(0))

    def leg(secs):
        t0 = time.perf_counter()
        tok, n = 0, 0
        while n < B and time.perf_counter() - t0 < secs:
            tok += oracle_sample(qkv, dout, L, [n], 1 / math.sqrt(D))
            n += 1
        return tok, n, time.perf_counter() - t0

    tok, n, dt = leg(seconds)
    one = None
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            t1, n1, d1 = leg(max(2.0, seconds / 4))
        one = {"value": t1 / d1, "sample": f"first {n1} sequences ({t1} tokens), {d1:.1f} s, BLAS limited to 1 thread"}
    except Exception as e:  # threadpoolctl missing: report without the 1-thread leg
        one = {"unavailable": str(e)[:120]}
    return {"value": tok / dt, "unit": "tokens/s", "cores": cores, "blas_threads": _blas_threads(),
            "cpu_model": _cpu_model(), "kind": "oracle",
            "sample": f"fp64 numpy oracle fwd+bwd on the first {n} of 56 sequences ({tok} tokens) of one "
                      f"{args.dist} batch, H=16 D=64, {dt:.1f} s",
            "one_thread": one}


def run_reference(args, world, rank):
    """--impl reference: the oracle is this tier's reference arm (rank 0 only)."""
    if rank != 0:
        return None
    L = synth.gen_lengths(args.dist, B, 100)
    T = int(L.sum())
    qkv = synth.gen_normal((T, 3, H, D), 1000)
    dout = synth.gen_normal((T, H, D), 2000)
    order = list(np.argsort(L))
    per_step = 2
    for w in range(args.warmup):
        oracle_sample(qkv, dout, L, [order[(2 * w) % B]], 1 / math.sqrt(D))
    t0 = time.perf_counter()
    tok = 0
    for k in range(args.steps):
        seqs = [int(order[(k * per_step + j * 17) % B]) for j in range(per_step)]
        tok += oracle_sample(qkv, dout, L, seqs, 1 / math.sqrt(D))
    dt = time.perf_counter() - t0
    v = tok / dt
    cores = len(os.sched_getaffinity(0))
    return {"metric": "unpadded FMHA fwd+bwd tokens/s (BERT-large)", "impl": "reference", "value": v,
            "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"bert_large_fmha_{args.dist}", "batch_per_gpu": B, "heads": H, "head_dim": D,
                       "max_seqlen": S},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "blas_threads": _blas_threads(),
                             "cpu_model": _cpu_model(), "kind": "oracle",
                             "sample": f"{per_step} sequences per step of one {args.dist} batch, fwd+bwd fp64"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ------------------------------------------------------------------ our arm
class Workload:
    def __init__(self, args, world, rank, dev):
        import paper_2208_08124_b200 as ub
        self.ub, self.args, self.world, self.rank, self.dev = ub, args, world, rank, dev
        self.cap = B * S
        self.sets = []
        for s in range(N_SETS):
            L = rank_lengths(args, world, rank, s)
            recs = np.zeros((B, S, 4), np.int32)
            raw = synth.gen_bytes(B * S * 16, 500 + 10 * s + rank).view(np.int32).reshape(B, S, 4) & 0x7FFF
            for b in range(B):
                recs[b, :L[b]] = raw[b, :L[b]]
            smp = synth.gen_bytes(B * 4, 600 + s + rank).view(np.int32).reshape(B, 1) & 1
            off = ub.cu_seqlens(L, S)
            st = {"L": L, "T": int(off[-1]), "lengths": torch.from_numpy(L).to(dev),
                  "cu_local": torch.from_numpy(off).to(dev), "padded_recs": torch.from_numpy(recs).to(dev),
                  "samples": torch.from_numpy(smp).to(dev),
                  "qkv": synth.gen_normal_device((self.cap, 3, H, D), 1000 + 7 * s + 100 * rank, dev),
                  "dout": synth.gen_normal_device((self.cap, H, D), 2000 + 7 * s + 100 * rank, dev)}
            self.sets.append(st)
        self.packed_recs = torch.empty((self.cap, 4), dtype=torch.int32, device=dev)
        self.ex = [{"tokens": torch.empty((self.cap, 4), dtype=torch.int32, device=dev),
                    "samples": torch.empty((B, 1), dtype=torch.int32, device=dev),
                    "cu": torch.empty(B + 1, dtype=torch.int32, device=dev), "T": 0, "L": None} for _ in range(N_EX)]
        self.out = torch.empty((self.cap, H, D), dtype=torch.bfloat16, device=dev)
        self.lse = torch.empty((H, self.cap), dtype=torch.float32, device=dev)
        self.lse_buf = self.lse                               # the hot loop's [H, T] view of the same memory
        self._begin, self._finish, self._unpad, self._fmha, self._prof_on = {}, {}, {}, {}, False
        self._mask = {}
        self.p = args.p_dropout
        # R5's keep bits, materialised once per step (ub_dropout_mask) and read by both directions;
        # two buffers: step n+1's mask is launched right behind step n's backward as an
        # overlapping dependent (UB_MASK_OVERLAP_PREVIOUS) that fills the SMs the backward's
        # tail leaves idle, while that backward still reads step n's buffer
        self.mask_bufs = [torch.empty(ub.api.dropout_mask_bytes(self.cap, H, S), dtype=torch.uint8, device=dev)
                          for _ in range(2)]
        self.mask_buf = self.mask_bufs[0]
        self.mask_overlap = bool(args.mask_overlap)
        self._mask_issued = set()
        self.dqkv = torch.empty((self.cap, 3, H, D), dtype=torch.bfloat16, device=dev)
        self.padded_out = torch.empty((B, S, H, D), dtype=torch.bfloat16, device=dev)
        # the compute stream at the highest priority, the exchange at the lowest: when an SM
        # frees up between two persistent FMHA kernels the block scheduler hands it to the
        # compute stream, so side-stream copies never delay a persistent grid's start
        self.main = torch.cuda.Stream(priority=-5)
        torch.cuda.set_stream(self.main)
        self.side = torch.cuda.Stream(priority=0)
        self.ex_ready = [torch.cuda.Event() for _ in range(N_EX)]
        self.done = [torch.cuda.Event() for _ in range(N_EX)]
        self.comm = ub.Comm(world, rank)
        # leave SMs free for the side-stream exchange (NCCL + copy kernels) to run
        # concurrently with the persistent FMHA kernels (P:376-381 overlap)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        self.ctas = sms - args.reserve_sms
        # host LPT schedules of the FMHA work items, one pair per exchange slot: built in finish()
        # from the lengths the exchange delivered and uploaded on the side stream with it
        self.sched_on = args.schedule > 0
        self.sched_fwd = args.schedule > 1
        if self.sched_on:
            nf = ub.api.lib().ub_fmha_schedule_ints(B, H, S, self.ctas, 0)
            nb = ub.api.lib().ub_fmha_schedule_ints(B, H, S, self.ctas, 1)
            self.sched_host = [(torch.zeros(nf, dtype=torch.int32).pin_memory(),
                                torch.zeros(nb, dtype=torch.int32).pin_memory()) for _ in range(N_EX)]
            self.sched_dev = [(torch.zeros(nf, dtype=torch.int32, device=dev),
                               torch.zeros(nb, dtype=torch.int32, device=dev)) for _ in range(N_EX)]
        self.force_nccl = args.exchange == "nccl-forced"
        if self.force_nccl:
            self.comm.set_options(force_nccl=True)

    def _begin_fn(self, n):
        key = (n % self.comm.SLOTS, n % N_SETS)
        f = self._begin.get(key)
        if f is None:
            st = self.sets[n % N_SETS]
            f = self._begin[key] = self.comm.bind_begin(key[0], st["lengths"], self.cap, REC, SREC, stream=self.side)
        return f

    def prebind(self):
        """Every pre-marshalled call the pipeline cycles through -- (exchange slot, input set,
        exchange buffer, mask buffer) combinations recur with period lcm(SLOTS, N_SETS, N_EX, 2) --
        bound before any timed region: a first-time binding inside it (host allocations and
        driver queries, up to ~1 ms) drains the GPU queue."""
        period = int(np.lcm.reduce([self.comm.SLOTS, N_SETS, N_EX, 2]))
        p_was = self.p
        for s_ in range(N_SETS):
            st = self.sets[s_]
            if s_ not in self._unpad:
                self._unpad[s_] = self.ub.api.BoundUnpad(st["padded_recs"], st["cu_local"], self.packed_recs,
                                                         stream=self.side)
        for n in range(period):
            self._begin_fn(n)
            self._finish_fn(n)
            for p in {self.args.p_dropout, 0.0}:          # the headline's p and the p = 0 step
                self.p = p
                self.bound(n)
                if p > 0:
                    for ov in (False, True):
                        self.mask(n, overlap=ov)
        self.p = p_was

    def begin(self, n):
        """Side stream, two steps ahead: a1 all-gather of step n's lengths (no host wait)."""
        self._begin_fn(n)()

    def finish(self, n, marks=None):
        """Side stream, one step ahead: a6 unpad of step n's input records, a2-a5 plan and
        exchange.  Its one host wait is for the lengths begin(n) fetched a step earlier."""
        s, e = n % N_SETS, n % N_EX
        st, ex = self.sets[s], self.ex[e]
        self.side.wait_event(self.done[e])                # step n-N_EX finished with these buffers
        u = self._unpad.get(s)
        if u is None:
            u = self._unpad[s] = self.ub.api.BoundUnpad(st["padded_recs"], st["cu_local"], self.packed_recs,
                                                        stream=self.side)
        u(st["T"])
        if marks is not None:
            marks.append(time.perf_counter())
        key, f, fs = self._finish_fn(n)
        T, perm = f()
        ex["T"] = T
        ex["perm"] = perm.copy()
        ex["n"] = n
        if self.sched_on:
            # the FMHA schedule(s) of the batch the exchange delivered (the library reads the
            # slot's all-gathered lengths through this finish's perm), uploaded on the side stream
            # behind the exchange.  No host wait for the previous upload from these pinned
            # buffers (finish(n - N_EX)'s): the finish above waited for begin(n)'s lengths, queued
            # on the side stream behind it.
            for fn in fs:
                fn()
        self.ex_ready[e].record(self.side)
        if marks is not None:
            marks.append(time.perf_counter())

    def _finish_fn(self, n):
        """(key, bound exchange finish, bound schedule calls) of step n's slot / set / buffers."""
        s, e = n % N_SETS, n % N_EX
        st, ex = self.sets[s], self.ex[e]
        key = (n % self.comm.SLOTS, s, e)
        got = self._finish.get(key)
        if got is None:
            f = self.comm.bind_finish(key[0], B, self.packed_recs, st["samples"], self.cap, S, self.args.balance,
                                      ex["tokens"], ex["samples"], ex["cu"], stream=self.side)
            fs = []
            if self.sched_on:
                perm = f.perm
                hf, hb = self.sched_host[e]
                df, db = self.sched_dev[e]
                fs.append(self.comm.bind_fmha_schedule(key[0], perm, B, H, S, self.ctas, True, hb, db,
                                                       stream=self.side))
                if self.sched_fwd:
                    fs.append(self.comm.bind_fmha_schedule(key[0], perm, B, H, S, self.ctas, False, hf, df,
                                                           stream=self.side))
            got = self._finish[key] = (key, f, fs)
        return got

    def lens_of(self, n):
        """Lengths of this rank's post-exchange batch of step n (host bookkeeping, outside the
        timed enqueue)."""
        ex = self.ex[n % N_EX]
        allL = np.asarray(self.all_lengths_cache(n), np.int64)
        return allL[ex["perm"][self.rank * B:(self.rank + 1) * B]]

    def all_lengths_cache(self, n):
        s = n % N_SETS
        if not hasattr(self, "_all_l"):
            self._all_l = {}
        if s not in self._all_l:
            self._all_l[s] = synth.skewed_rank_lengths(self.world, B, s, self.args.skew, self.args.dist).reshape(-1)
        return self._all_l[s]

    def bound(self, n):
        """The pre-marshalled FMHA calls of step n's buffers (input set, exchange slot, dqkv)."""
        s, e = n % N_SETS, n % N_EX
        mb = n % 2
        key = (s, e, self.dqkv.data_ptr(), self.p, mb)
        b = self._fmha.get(key)
        if b is None:
            st = self.sets[s]
            b = self._fmha[key] = self.ub.api.BoundFmha(
                st["qkv"], self.ex[e]["cu"], S, self.out, self.lse_buf, dout=st["dout"], dqkv=self.dqkv,
                p_dropout=self.p, stream=self.main, num_ctas=self.ctas, padded=self.padded_out,
                dropout_mask=self.mask_bufs[mb] if self.p > 0 else None)
        return b

    def mask(self, n, overlap=False):
        """ub_dropout_mask of step n's exchanged batch (cu_seqlens of its exchange slot) into
        buffer n % 2; overlap: UB_MASK_OVERLAP_PREVIOUS (launched right behind step n-1's backward)."""
        e = n % N_EX
        key = (e, self.p, n % 2, overlap)
        m = self._mask.get(key)
        if m is None:
            m = self._mask[key] = self.ub.api.BoundDropoutMask(self.ex[e]["cu"], self.cap, H, S, self.p,
                                                               self.mask_bufs[n % 2], stream=self.main,
                                                               overlap_previous=overlap)
        return m

    def step(self, n, prof=None, marks=None):
        """Main stream: a7 fwd (+ fused a9 pad), a8 bwd for step n.  marks: host timestamps."""
        ex = self.ex[n % N_EX]
        T = ex["T"]
        self.main.wait_event(self.ex_ready[n % N_EX])
        # mask overlap: step n+1's exchange is waited for here, so that nothing separates step
        # n's backward from step n+1's mask on the stream
        nxt_ready = self.p > 0 and self.mask_overlap and self.ex[(n + 1) % N_EX].get("n") == n + 1
        if nxt_ready:
            self.main.wait_event(self.ex_ready[(n + 1) % N_EX])
        if prof is not None:
            for kid, pair in prof.items():
                self.ub.api.profile_events(kid, *pair)
            self._prof_on = True
        elif self._prof_on:                                 # unregister: this step runs uninstrumented
            for kid in (0, 1, 3):
                self.ub.api.profile_events(kid)
            self._prof_on = False
        if marks is not None:
            marks.append(time.perf_counter())
        b = self.bound(n)
        if self.sched_on:
            df, db = self.sched_dev[n % N_EX]
            b.set_schedules(df if self.sched_fwd else None, db)
        if self.p > 0 and n not in self._mask_issued:
            self.mask(n)(T, 0x2208 + n)                     # keep bits for both directions of this step
        self._mask_issued.discard(n)
        # a7 + a9: the forward's epilogue also writes the padded copy of O, zeros past
        # each length -- the separate pad pass is gone (ub_varlen_fmha_fwd_pad)
        b.fwd(T, 0x2208 + n)
        if marks is not None:
            marks.append(time.perf_counter())
        b.bwd(T, 0x2208 + n)
        if nxt_ready:                                       # step n+1's keep bits beside the backward's tail
            self.mask(n + 1, overlap=True)(self.ex[(n + 1) % N_EX]["T"], 0x2208 + n + 1)
            self._mask_issued.add(n + 1)
        if marks is not None:
            marks.append(time.perf_counter())
        self.done[n % N_EX].record(self.main)
        if marks is not None:
            marks.append(time.perf_counter())
        return T


def run_ours(args, world, rank, local):
    dev = torch.device("cuda", local)
    wl = Workload(args, world, rank, dev)
    wl.prebind()
    ub = wl.ub
    peaks = load_peaks()
    # warm-up.  Pipeline: step n computes (main) while n+PIPE is exchanged and the lengths of
    # n+PIPE+1 are gathered (side stream)
    for n in range(PIPE + 1):
        wl.begin(n)
    for n in range(PIPE):
        wl.finish(n)
    for n in range(args.warmup):
        wl.step(n)
        wl.finish(n + PIPE)
        wl.begin(n + PIPE + 1)
    torch.cuda.synchronize()
    barrier(world)
    # timed region
    kids = [ub.api.PROF_FWD, ub.api.PROF_BWD, ub.api.PROF_UNPAD]
    prof_events = [{k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in kids}
                   for _ in range(args.steps)]
    for d in prof_events:                 # create the cudaEvent_t handles outside the timed loop
        for a, b_ in d.values():
            a.record(wl.main)
            b_.record(wl.main)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tokens, lens_used = 0, []
    host_step, host_prep, marks = [], [], []
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    wl.comm.set_options(force_nccl=wl.force_nccl, host_profile=True)   # host-only phase clocks
    e0.record(wl.main)
    for k in range(args.steps):
        n = args.warmup + k
        step_ev[k].record(wl.main)
        h0 = time.perf_counter()
        m = []
        profiled = args.prof_every > 0 and k % args.prof_every == 0
        tokens += wl.step(n, prof_events[k] if profiled else None, m)
        lens_used.append((n, wl.ex[n % N_EX]["perm"]))      # a reference; lengths derived after the loop
        h1 = time.perf_counter()
        wl.finish(n + PIPE, m)
        wl.begin(n + PIPE + 1)
        m.append(time.perf_counter())
        marks.append(np.diff([h0] + m))
        host_step.append(h1 - h0)
        host_prep.append(time.perf_counter() - h1)
    step_ev[args.steps].record(wl.main)
    finish_prof = wl.comm.host_profile()
    wl.comm.set_options(force_nccl=wl.force_nccl, host_profile=False)
    wl.main.wait_stream(wl.side)      # steady state: the K steps plus the exchange of the next one
    e1.record(wl.main)
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    for kid in kids:
        ub.api.profile_events(kid)
    wl._prof_on = False
    lens_used = [np.asarray(wl.all_lengths_cache(nn), np.int64)[pp[rank * B:(rank + 1) * B]] for nn, pp in lens_used]
    last = args.warmup + args.steps + PIPE
    wl.finish(last)                   # drain the begin still in flight (untimed)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    step_us = [step_ev[k].elapsed_time(step_ev[k + 1]) * 1e3 for k in range(args.steps)]
    overlap = exchange_overlap(args, wl, world, last, ms / args.steps * 1e3)
    ms_max = all_max(ms, world)
    tok_all = all_sum(tokens, world)
    value = tok_all / (ms_max / 1e3)
    per_rank_tokens = all_gather_list(tokens / args.steps, world)
    imbalance = max(per_rank_tokens) / (sum(per_rank_tokens) / world) - 1.0

    # per-kernel device time (events the library records around its own launches, on the
    # launching stream): from the headline region (--prof-every k) or, by default, from a
    # separate region of the same pipelined steps with every step instrumented
    if args.prof_every > 0:
        prof_steps = [i for i in range(args.steps) if i % args.prof_every == 0]
        kt = {k: [prof_events[i][k][0].elapsed_time(prof_events[i][k][1]) for i in prof_steps] for k in kids}
        instr_ms = None
    else:
        rec = []
        instr_ms, _, _ = pipelined_region(wl, args, world, last + 1 + 20 * N_EX, args.p_dropout, prof=rec)
        prof_steps = list(range(len(rec)))
        kt = {k: [rec[i][2][k][0].elapsed_time(rec[i][2][k][1]) for i in prof_steps] for k in kids}
        lens_used = [np.asarray(wl.all_lengths_cache(nn), np.int64)[pp[rank * B:(rank + 1) * B]] for nn, pp, _ in rec]
        prof_events = [r[2] for r in rec]
    f_fwd = [flops_fwd(lens_used[i]) for i in prof_steps]
    f_bwd = [flops_bwd(lens_used[i]) for i in prof_steps]
    fwd_us, bwd_us = np.mean(kt[kids[0]]) * 1e3, np.mean(kt[kids[1]]) * 1e3
    unpad_us = np.mean(kt[kids[2]]) * 1e3
    fwd_tf = np.mean(f_fwd) / (fwd_us * 1e-6) / 1e12
    bwd_tf = np.mean(f_bwd) / (bwd_us * 1e-6) / 1e12
    mean_T = tokens / args.steps
    rl = rooflines(peaks, clk, wl.ctas, [lens_used[i] for i in prof_steps], fwd_us, bwd_us, padded_fwd=True)
    dom = "bwd" if bwd_us >= fwd_us else "fwd"
    roofline = dict(rl[dom])
    roofline["traffic"] = load_traffic().get("fmha_" + dom)
    roofline["other_kernel"] = rl["fwd" if dom == "bwd" else "bwd"]
    kernels = {"fmha_fwd": {"us": round(fwd_us, 2), "tflops": round(fwd_tf, 1)},
               "fmha_bwd": {"us": round(bwd_us, 2), "tflops": round(bwd_tf, 1)},
               "pad": "fused into fmha_fwd's epilogue (ub_varlen_fmha_fwd_pad); standalone ub_pad under gather",
               "unpad_records": {"us": round(unpad_us, 2)}}
    fmha_only = mean_T * world / ((fwd_us + bwd_us) * 1e-6)
    # TC utilisation (BASELINE metric), three ways: FA convention 14 H D sum L^2
    # per fwd+bwd (recompute credited), strict 12 H D sum L^2, and ncu's tensor-pipe activity
    s2 = float(np.mean([float((np.asarray(lens_used[i], np.int64) ** 2).sum()) for i in prof_steps]))
    fb_s = (fwd_us + bwd_us) * 1e-6
    tc_util = {"fa_convention_tflops": round(14 * H * D * s2 / fb_s / 1e12, 1),
               "strict_tflops": round(12 * H * D * s2 / fb_s / 1e12, 1),
               "fa_frac_of_burst_peak": round(14 * H * D * s2 / fb_s / 1e12 / peaks["bf16"], 4),
               "ncu_tensor_pipe_active_pct": load_tensor_pipe(),
               "note": "fwd (incl. its fused pad writes) + bwd main kernels, in-step device time"}
    # main-stream timeline from the same events: gap between a step's backward and the next
    # step's forward, and forward end -> backward main kernel (= the Delta prologue + gaps)
    P = prof_events
    F, Bk = kids[0], kids[1]
    f2b = float(np.mean([P[i][F][1].elapsed_time(P[i][Bk][0]) for i in prof_steps])) * 1e3
    step_ref = (instr_ms * 1e3) if instr_ms is not None else ms_max / args.steps * 1e3
    timeline = {"fwd_end_to_bwd_main_us": round(f2b, 2),
                "rest_of_step_us": round(step_ref - fwd_us - bwd_us - f2b, 2),
                "kernel_events_on": (f"every {args.prof_every} step(s) of the headline region" if args.prof_every
                                     else f"every step of a separate instrumented region "
                                          f"({round(step_ref, 2)} us per step there)")}

    # the same pipelined step without attention dropout (p = 0), beside the headline
    p0 = None
    if args.p_dropout > 0:
        ms0, tok0, _ = pipelined_region(wl, args, world, last + 1 + 10 * N_EX, 0.0)
        p0 = {"value": round(tok0 / (ms0 / 1e3), 1), "unit": "tokens/s", "ms_per_step": round(ms0, 4),
              "p_dropout": 0.0, "note": "the headline's pipelined step (exchange overlapped) at p = 0"}
        wl.p = args.p_dropout
    e2e = None if args.no_e2e else run_e2e(args, wl, world)
    gather = gather_bench(wl, peaks) if rank == 0 else None
    encoder = encoder_bench(wl, peaks) if rank == 0 and not args.no_encoder else None
    embedding = embedding_bench(wl, peaks) if rank == 0 and not args.no_encoder else None
    drop01 = dropout_bench(wl) if rank == 0 else None
    sweep = dist_sweep(wl, peaks) if rank == 0 and not args.no_encoder else None
    out = {"metric": "unpadded FMHA fwd+bwd tokens/s (BERT-large)", "value": round(value, 1), "unit": "tokens/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
           "data": "synthetic (seeded lengths + N(0,1) bf16 qkv/dO; no dataset)",
           "config": {"workload": f"bert_large_fmha_{args.dist}", "batch_per_gpu": B, "heads": H, "head_dim": D,
                      "max_seqlen": S, "p_dropout": args.p_dropout,
                      "p_dropout_applied": ub.api.dropout_effective_p(args.p_dropout) if args.p_dropout > 0 else 0.0,
                      "balance": args.balance, "skew": args.skew,
                      "parallelism": f"dp{world}", "fmha_ctas": wl.ctas,
                      "fmha_schedule": ("snake (in-kernel)", "bwd: host LPT (ub_fmha_schedule), fwd: snake",
                                        "host LPT (ub_fmha_schedule)")[min(args.schedule, 2)],
                      "exchange": args.exchange, "l2": "rotating 3 input sets; per-step working set > L2",
                      "step": "unpad records + exchange (side stream) | dropout keep bits (p > 0), fmha fwd with fused "
                   "pad, bwd (main stream)"},
           "roofline": roofline, "kernels": kernels, "fmha_only_tokens_per_s": round(fmha_only, 1),
           "p0_step": p0,
           "tc_util": tc_util,
           "imbalance": round(imbalance, 5), "planned_imbalance": planned_imbalance(args),
           "step_us_distribution": {"p10": round(float(np.percentile(step_us, 10)), 2),
                                    "median": round(float(np.median(step_us)), 2),
                                    "p90": round(float(np.percentile(step_us, 90)), 2),
                                    "mean": round(float(np.mean(step_us)), 2), "n": len(step_us),
                                    "max": round(float(np.max(step_us)), 2),
                                    "slowest": [[int(i), round(float(step_us[i]), 1)]
                                                for i in np.argsort(step_us)[::-1][:5]],
                                    "note": "main-stream step boundaries (events); the headline is the whole "
                                            "K-step region / K"},
           "exchange_overlap": overlap,
           "main_stream_timeline": timeline, "attn_dropout_0.1": drop01, "length_sweep": sweep, "gather": gather,
           "encoder_attn_sublayer": encoder, "embedding": embedding, "gpu_launches": (KERNELS_PER_STEP + (1 if args.p_dropout > 0 else 0)) * args.steps, "clocks": clk,
           "host_us_per_step": dict(zip(["step_setup", "fwd_call", "bwd_call", "pad_call", "unpad_call", "finish_call",
                                              "begin_call"],
                                        [round(1e6 * float(x), 1) for x in np.median(np.array(marks), axis=0)]),
                                    enqueue_compute=round(1e6 * float(np.median(host_step)), 1),
                                    exchange_calls=round(1e6 * float(np.median(host_prep)), 1)),
           "exchange_finish_host_us": {
               **{k: (round(v, 1) if isinstance(v, float) else v) for k, v in finish_prof.items()},
               "note": "mean host us per ub_exchange_finish in the timed steps: wait_lengths is the one host "
                       "wait (for this slot's all-gathered lengths: the GPU's pace, not host work); the rest is "
                       "host work (plan, tables, launches)"}}
    if e2e is not None:
        out["e2e"] = e2e
    return out, wl


def pipelined_region(wl, args, world, first, p, prof=None):
    """The headline's step loop (exchange pipelined on the side stream) at dropout p, started
    at step number `first` on an empty pipeline: returns (ms per step, max over ranks; tokens
    per step summed over ranks; next free step number).  prof: a list that receives, per
    timed step, (step number, perm reference, {kernel id: (start, stop) events}) with the
    library's per-kernel events recorded on every step."""
    wl.p = p
    for n in range(first, first + PIPE + 1):
        wl.begin(n)
    for n in range(first, first + PIPE):
        wl.finish(n)
    n = first
    for _ in range(args.warmup):
        wl.step(n)
        wl.finish(n + PIPE)
        wl.begin(n + PIPE + 1)
        n += 1
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(wl.main)
    tok = 0
    kids = (0, 1, 3)
    evs = [{k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in kids}
           for _ in range(args.steps)] if prof is not None else None
    if evs:
        for d in evs:
            for a, b_ in d.values():
                a.record(wl.main)
                b_.record(wl.main)
        e0.record(wl.main)
    for k in range(args.steps):
        tok += wl.step(n, evs[k] if evs else None)
        if prof is not None:
            prof.append((n, wl.ex[n % N_EX]["perm"], evs[k]))
        wl.finish(n + PIPE)
        wl.begin(n + PIPE + 1)
        n += 1
    wl.main.wait_stream(wl.side)
    e1.record(wl.main)
    if evs:
        for kid in kids:
            wl.ub.api.profile_events(kid)
        wl._prof_on = False
    torch.cuda.synchronize()
    barrier(world)
    wl.finish(n + PIPE)
    torch.cuda.synchronize()
    ms = all_max(e0.elapsed_time(e1), world) / args.steps
    return ms, all_sum(tok, world) / args.steps, n + PIPE + 1


def exchange_overlap(args, wl, world, last, step_us):
    """how much of the exchange the overlap hides.
    compute-only: the same K main-stream steps on batches whose exchange already finished
    (no side-stream work); isolated: the side stream's per-step work (unpad of the input
    records, a1-a5) alone, device time between events on that stream, the host plan between
    its phases included; exposed = overlapped step - compute-only step."""
    K = args.steps
    done = [last - i for i in range(N_EX)]              # exchanged batches whose buffers are intact
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k in range(3):
        wl.step(done[k % N_EX])
    e0.record(wl.main)
    for k in range(K):
        wl.step(done[k % N_EX])
    e1.record(wl.main)
    torch.cuda.synchronize()
    comp = all_max(e0.elapsed_time(e1), world) / K * 1e3
    # the exchange alone: begin + unpad + finish per step on the side stream, nothing else
    n0 = last + 1
    barrier(world)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wl.begin(n0)
    wl.side.synchronize()
    s0.record(wl.side)
    for k in range(K):
        wl.begin(n0 + k + 1)
        wl.finish(n0 + k)
    s1.record(wl.side)
    torch.cuda.synchronize()
    wl.finish(n0 + K)
    torch.cuda.synchronize()
    iso = all_max(s0.elapsed_time(s1), world) / K * 1e3
    return {"overlapped_step_us": round(step_us, 2), "compute_only_step_us": round(comp, 2),
            "exposed_exchange_us": round(step_us - comp, 2), "isolated_exchange_us": round(iso, 2),
            "exchange": "nccl" + (" (forced through NCCL at W=1)" if getattr(wl, "force_nccl", False) else ""),
            "note": "exposed = overlapped - compute-only (negative = within run-to-run noise); isolated = "
                    "side-stream events around K x (all-gather, unpad, plan, pack, send/recv, unpack)"}


def args_dist(wl):
    return getattr(wl.args, "dist", "mlperf_like_v0")


def gather_bench(wl, peaks, iters=20):
    """a6 / a9 on the config-2 hidden state (bf16 [56, 512, 1024] <-> [T, 1024]), HBM-bound:
    algorithmic bytes unpad = 2*T*row, pad = T*row + B*S*row; 3 rotating buffer sets."""
    ub = wl.ub
    st = wl.sets[0]
    T, cu = st["T"], st["cu_local"]
    row = H * D * 2
    bufs = [(torch.randn((B, S, H * D), device=wl.dev).to(torch.bfloat16),
             torch.empty((T, H * D), dtype=torch.bfloat16, device=wl.dev)) for _ in range(3)]
    out = {}
    from paper_2208_08124_b200 import api
    for name, kid, fn, nbytes in (("unpad", 3, lambda b: ub.unpad(b[0], cu, T, out=b[1]), 2 * T * row),
                                  ("pad", 2, lambda b: ub.pad(b[1], cu, B, S, out=b[0]), T * row + B * S * row)):
        for k in range(3):
            fn(bufs[k])
        torch.cuda.synchronize()
        # device time of the kernel alone: the library records these events right around its
        # launch (host-side call overhead excluded; the stream is kept busy ahead of the host)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
        torch.cuda._sleep(2_000_000)
        for k in range(iters):
            api.profile_events(kid, *ev[k])
            fn(bufs[k % 3])
        api.profile_events(kid)
        torch.cuda.synchronize()
        us_iso = float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3
        # back to back (how the step runs them): K launches between two events, per launch
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(iters):
            fn(bufs[k % 3])
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / iters * 1e3
        gbs = nbytes / (us * 1e-6) / 1e9
        out[name] = {"us": round(us, 2), "GBps": round(gbs, 1), "frac_hbm": round(gbs / peaks["hbm"], 3),
                     "bytes": int(nbytes), "us_isolated": round(us_iso, 2),
                     "frac_hbm_isolated": round(nbytes / (us_iso * 1e-6) / 1e9 / peaks["hbm"], 3),
                     "note": "us: back to back (K launches / K, rotating 3 buffer sets, > L2); us_isolated: "
                             "median of events recorded right around each launch (includes its ramp)"}
    # the size-matched ceiling: torch's own device copy of the packed tensor (same bytes as unpad;
    # at ~30 MB the launch ramp and drain keep any copy below the 2-GiB copy that measured the peak)
    cp = [torch.empty((T, H * D), dtype=torch.bfloat16, device=wl.dev) for _ in range(3)]
    for k in range(3):
        cp[k].copy_(bufs[k][1])
    torch.cuda.synchronize()
    torch.cuda._sleep(2_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(iters):
        cp[k % 3].copy_(bufs[k % 3][1])
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    out["torch_copy_same_bytes"] = {"us": round(us, 2), "GBps": round(2 * T * row / (us * 1e-6) / 1e9, 1),
                                    "frac_hbm": round(2 * T * row / (us * 1e-6) / 1e9 / peaks["hbm"], 3),
                                    "note": "torch copy_ of the packed tensor: the achievable copy rate at this size"}
    out["shape"] = f"hidden [{B}, {S}, {H * D}] bf16 <-> [T={T}, {H * D}]"
    # the qkv row (6 144 B) and a batch-size sweep of the hidden row (the launch
    # ramp / drain share shrinks as the copy grows); back to back, 2 rotating buffer sets
    sweep = {}
    for nb, rb in ((B, 3 * H * D * 2), (2 * B, H * D * 2), (4 * B, H * D * 2), (8 * B, H * D * 2)):
        Ls = synth.gen_lengths(args_dist(wl), nb, 7 + nb)
        offs = np.concatenate([[0], np.cumsum(Ls)]).astype(np.int32)
        Tn = int(offs[-1])
        cun = torch.from_numpy(offs).to(wl.dev)
        sets = [(torch.empty((nb, S, rb), dtype=torch.uint8, device=wl.dev),
                 torch.empty((Tn, rb), dtype=torch.uint8, device=wl.dev)) for _ in range(2)]
        res = {}
        for name, fn, nbytes in (("unpad", lambda b: ub.unpad(b[0], cun, Tn, out=b[1]), 2 * Tn * rb),
                                 ("pad", lambda b: ub.pad(b[1], cun, nb, S, out=b[0]), Tn * rb + nb * S * rb)):
            for k in range(2):
                fn(sets[k])
            torch.cuda.synchronize()
            torch.cuda._sleep(2_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for k in range(iters):
                fn(sets[k % 2])
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / iters * 1e3
            res[name] = {"us": round(us, 2), "frac_hbm": round(nbytes / (us * 1e-6) / 1e9 / peaks["hbm"], 3),
                         "bytes": int(nbytes)}
        sweep[f"B{nb}_row{rb}"] = res
        del sets
    out["sweep"] = sweep
    out["sweep_note"] = ("frac_hbm against the measured copy bandwidth (read + write); pad's zero fill is "
                         "write-only traffic, which can exceed that figure")
    # NEXT-3: the exchange's data movement at SURVEY §8(a) a4's stress record size (a bf16
    # hidden row, 2 kB per token), one rank: the pull gather (one pass) against the NCCL
    # path's pack + unpack copies (two passes; the transport between them is a third)
    rec = H * D * 2
    lens = np.asarray(st["L"], np.int32)
    perm = api.balance_plan(lens, 1, B, S, "paper")["perm"]
    d_pack = torch.from_numpy(api.exchange_tables(lens, perm, 1, B, 0, unpack=False)[0]).to(wl.dev)
    d_unpack = torch.from_numpy(api.exchange_tables(lens, perm, 1, B, 0, unpack=True)[0]).to(wl.dev)
    d_pull = torch.from_numpy(api.exchange_pull_table(lens, perm, 1, B, 0)[0]).to(wl.dev)
    src = [torch.randint(0, 255, (T, rec), dtype=torch.uint8, device=wl.dev) for _ in range(3)]
    mid = torch.empty((T, rec), dtype=torch.uint8, device=wl.dev)
    dst = torch.empty((T, rec), dtype=torch.uint8, device=wl.dev)
    peers = [torch.tensor([x.data_ptr()], dtype=torch.int64, device=wl.dev) for x in src]
    for name, fn, nbytes in (
            ("exchange_2kB_pull", lambda k: api.exchange_pull(peers[k], None, d_pull, B, rec, 0, dst), 2 * T * rec),
            ("exchange_2kB_pack_unpack", lambda k: (api.exchange_copy(src[k], mid, None, None, d_pack, B, rec, 0),
                                                    api.exchange_copy(mid, dst, None, None, d_unpack, B, rec, 0)),
             4 * T * rec)):
        for k in range(3):
            fn(k)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
        torch.cuda._sleep(2_000_000)
        for k in range(iters):
            ev[k][0].record()
            fn(k % 3)
            ev[k][1].record()
        torch.cuda.synchronize()
        us = float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3
        gbs = nbytes / (us * 1e-6) / 1e9
        out[name] = {"us": round(us, 2), "GBps": round(gbs, 1), "frac_hbm": round(gbs / peaks["hbm"], 3),
                     "bytes": int(nbytes), "rec_bytes": rec, "ranks": 1}
    # NEXT-1 piece: Dropout_Add_LayerNorm on the same packed hidden state, p = 0.1
    E = H * D
    hs = [tuple(torch.randn((T, E), device=wl.dev).to(torch.bfloat16) for _ in range(3)) for _ in range(3)]
    g = torch.ones(E, dtype=torch.bfloat16, device=wl.dev)
    bt = torch.zeros(E, dtype=torch.bfloat16, device=wl.dev)
    st = [ub.dal_fwd(h[0], h[1], g, bt, 0.1, 1e-12, 5) for h in hs]
    for name, kid, fn, nbytes in (
            ("dal_fwd", api.PROF_DAL_FWD, lambda k: ub.dal_fwd(hs[k][0], hs[k][1], g, bt, 0.1, 1e-12, 5), 3 * T * E * 2 + 8 * T),
            ("dal_bwd", api.PROF_DAL_BWD,
             lambda k: ub.dal_bwd(hs[k][2], hs[k][0], hs[k][1], g, st[k][1], st[k][2], 0.1, 5), 5 * T * E * 2 + 8 * T)):
        for k in range(3):
            fn(k)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
        torch.cuda._sleep(2_000_000)
        for k in range(iters):
            api.profile_events(kid, *ev[k])
            fn(k % 3)
        api.profile_events(kid)
        torch.cuda.synchronize()
        us = float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3
        gbs = nbytes / (us * 1e-6) / 1e9
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(iters):
            fn(k % 3)
        e1.record()
        torch.cuda.synchronize()
        us_b2b = e0.elapsed_time(e1) / iters * 1e3
        out[name] = {"us": round(us, 2), "GBps": round(gbs, 1), "frac_hbm": round(gbs / peaks["hbm"], 3),
                     "bytes": int(nbytes), "p_dropout": 0.1, "us_back_to_back": round(us_b2b, 2),
                     "frac_hbm_back_to_back": round(nbytes / (us_b2b * 1e-6) / 1e9 / peaks["hbm"], 3),
                     "note": "us: median of the library's events right around each launch (incl. its ramp); "
                             "back to back: K launches / K (the bwd's includes its small reduce kernel)"}
    return out


def dropout_bench(wl, iters=10):
    """Attention dropout p = 0.1 (BERT-large's training value) two ways on one
    batch: keep bits regenerated by Philox inside the FMHA kernels (no mask argument), and
    materialised once by ub_dropout_mask and read by both kernels (the headline step's way).
    Device time of each kernel from the library's events / CUDA events."""
    from paper_2208_08124_b200 import api
    ub = wl.ub
    st, ex = wl.sets[0], wl.ex[0]
    T = ex["T"]
    qkv, dout = st["qkv"][:T], st["dout"][:T]
    cu = ex["cu"]
    m = api.dropout_mask(cu, T, H, S, 0.1, 7, 0)
    o, lse = ub.varlen_fmha_fwd(qkv, cu, S, None, 0.1, 7, 0)
    res = {}

    def timed(kid, fn):
        fn()
        torch.cuda.synchronize()
        torch.cuda._sleep(2_000_000)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
        for k in range(iters):
            if kid is None:
                ev[k][0].record()
                fn()
                ev[k][1].record()
            else:
                api.profile_events(kid, *ev[k])
                fn()
        if kid is not None:
            api.profile_events(kid)
        torch.cuda.synchronize()
        return round(float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3, 2)
    for tag, mk in (("philox_in_kernel", None), ("mask", m)):
        r = {"fwd_us": timed(api.PROF_FWD, lambda: ub.varlen_fmha_fwd(qkv, cu, S, None, 0.1, 7, 0, out=o, lse=lse,
                                                                       dropout_mask=mk)),
             "bwd_us": timed(api.PROF_BWD, lambda: ub.varlen_fmha_bwd(qkv, o, lse, dout, cu, S, None, 0.1, 7, 0,
                                                                       dropout_mask=mk))}
        if mk is not None:
            r["mask_us"] = timed(None, lambda: api.dropout_mask(cu, T, H, S, 0.1, 7, 0, out=m))
        tot = r["fwd_us"] + r["bwd_us"] + r.get("mask_us", 0.0)
        r["fmha_only_tokens_per_s"] = round(T / (tot * 1e-6), 1)
        res[tag] = r
    res["note"] = "main kernels (and the mask kernel), L2-warm single batch, p = 0.1 (applied 25/256)"
    return res


def embedding_bench(wl, peaks, iters=10):
    """NEXT-4: unpadded BERT embedding fwd / bwd (fp32 gradients, 16-B vector reductions) on
    the config-2 packed batch, vocab 30 522, Zipf-like ids.  Algorithmic bytes: fwd the output
    plus each distinct table row once; bwd 1 row read + 2 fp32 row updates per token (word,
    position; the token-type rows are reduced per CTA)."""
    ub = wl.ub
    st = wl.sets[0]
    T, cu = st["T"], st["cu_local"]
    E, Vv, P = H * D, 30522, S        # noqa: N806
    rng = np.random.default_rng(0)
    off = cu.cpu().numpy().astype(np.int64)
    ids = torch.from_numpy(np.minimum(rng.zipf(1.2, T) - 1, Vv - 1).astype(np.int32)).to(wl.dev)
    pos = torch.from_numpy((np.arange(T) - np.repeat(off[:-1], np.diff(off))).astype(np.int32)).to(wl.dev)
    seg = torch.from_numpy((rng.random(T) < 0.5).astype(np.int32)).to(wl.dev)
    ww = (0.02 * torch.randn((Vv, E), device=wl.dev)).to(torch.bfloat16)
    wp = (0.02 * torch.randn((P, E), device=wl.dev)).to(torch.bfloat16)
    wt = (0.02 * torch.randn((2, E), device=wl.dev)).to(torch.bfloat16)
    dout = torch.randn((T, E), device=wl.dev).to(torch.bfloat16)
    out = torch.empty((T, E), dtype=torch.bfloat16, device=wl.dev)
    dws = [torch.zeros((n, E), dtype=torch.float32, device=wl.dev) for n in (Vv, P, 2)]
    res = {}
    uniq = int(torch.unique(ids).numel())
    # fwd compulsory HBM bytes: the output plus each distinct table row once (hot rows of the
    # Zipf ids, the position and type tables stay in L2)
    for name, fn, nb in (("fwd", lambda: ub.embedding_fwd(ids, pos, seg, ww, wp, wt, out=out),
                          (T + uniq + P + 2) * E * 2),
                         ("bwd", lambda: ub.embedding_bwd(dout, ids, pos, seg, *dws), T * E * 2 + 2 * T * E * 4)):
        fn()
        torch.cuda.synchronize()
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / iters * 1e3
        res[name] = {"us": round(us, 2), "GBps": round(nb / (us * 1e-6) / 1e9, 1),
                     "frac_hbm": round(nb / (us * 1e-6) / 1e9 / peaks["hbm"], 3)}
    res["config"] = f"T={T}, E={E}, vocab {Vv}, Zipf(1.2) ids, fp32 gradients"
    return res


def dist_sweep(wl, peaks, iters=10):
    """BASELINE config 5 on one GPU: the FMHA fwd + bwd main kernels on 56-sequence batches of
    each length distribution (uniform, MLPerf-like, bimodal 64/512), device time from the
    library's events, with the fwd+bwd TC utilisation (FA convention, burst peak)."""
    from paper_2208_08124_b200 import api
    ub = wl.ub
    out = {}
    for dist in ("uniform", "mlperf_like_v0", "bimodal"):
        L = synth.gen_lengths(dist, B, 0).astype(np.int64)
        T = int(L.sum())
        off = np.concatenate([[0], np.cumsum(L)]).astype(np.int32)
        cu = torch.from_numpy(off).to(wl.dev)
        qkv = synth.gen_normal_device((T, 3, H, D), 11, wl.dev)
        dout = synth.gen_normal_device((T, H, D), 12, wl.dev)
        o, lse = ub.varlen_fmha_fwd(qkv, cu, S)
        res = {}
        for name, kid, fn in (("fwd", api.PROF_FWD, lambda: ub.varlen_fmha_fwd(qkv, cu, S, out=o, lse=lse)),
                              ("bwd", api.PROF_BWD, lambda: ub.varlen_fmha_bwd(qkv, o, lse, dout, cu, S))):
            fn()
            torch.cuda.synchronize()
            torch.cuda._sleep(2_000_000)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
            for k in range(iters):
                api.profile_events(kid, *ev[k])
                fn()
            api.profile_events(kid)
            torch.cuda.synchronize()
            res[name + "_us"] = round(float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3, 2)
        s2 = float((L ** 2).sum())
        fb = (res["fwd_us"] + res["bwd_us"]) * 1e-6
        res["tokens_per_s"] = round(T / fb, 1)
        res["fa_convention_tflops"] = round(14 * H * D * s2 / fb / 1e12, 1)
        res["fa_frac_of_burst_peak"] = round(14 * H * D * s2 / fb / 1e12 / peaks["bf16"], 4)
        res["T"] = T
        out[dist] = res
    out["note"] = "main kernels only, one L2-warm batch each (seed 0), p = 0"
    return out


def encoder_bench(wl, peaks, iters=10):
    """NEXT-1 (BASELINE config 4 on one GPU): the unpadded encoder attention sub-layer
    (QKV Linear -> varlen FMHA -> out Linear -> Dropout_Add_LayerNorm) forward and backward
    on the config-2 batch, hidden 1024, p_attn = p_hidden = 0.1, random-init weights.
    Algorithmic flops: GEMMs 8*T*h^2 fwd / 16*T*h^2 bwd, attention 4 / 8 *H*D*sum(L^2)."""
    ub = wl.ub
    st = wl.sets[0]
    T, cu = st["T"], st["cu_local"]
    L = np.diff(cu.cpu().numpy().astype(np.int64))
    hid = H * D
    dev = wl.dev
    s = 1.0 / math.sqrt(hid)
    w = {k: (torch.randn(shape, device=dev) * sc).to(torch.bfloat16) for k, shape, sc in
         (("wq", (3 * hid, hid), s), ("bq", (3 * hid,), 0.1), ("wo", (hid, hid), s), ("bo", (hid,), 0.1),
          ("g", (hid,), 0.0), ("b", (hid,), 0.1))}
    w["g"] += 1.0
    xs = [torch.randn((T, hid), device=dev).to(torch.bfloat16) for _ in range(3)]
    dys = [torch.randn((T, hid), device=dev).to(torch.bfloat16) for _ in range(3)]
    saved = [None] * 3
    fwd = lambda k: ub.encoder_attn_fwd(xs[k], cu, S, w["wq"], w["bq"], w["wo"], w["bo"], w["g"], w["b"], H, 0.1, 0.1,
                                        1e-12, 0x2208 + k, 0, saved=saved[k])
    for k in range(3):
        saved[k] = fwd(k)[1]
    bwd = lambda k: ub.encoder_attn_bwd(dys[k], xs[k], cu, S, w["wq"], w["wo"], w["g"], saved[k], H, 0.1, 0.1, 1e-12,
                                        0x2208 + k, 0)
    out = {}
    s2 = float((L ** 2).sum())
    for name, fn, fl in (("fwd", fwd, 8 * T * hid * hid + 4 * H * D * s2),
                         ("bwd", bwd, 16 * T * hid * hid + 8 * H * D * s2)):
        for k in range(3):
            fn(k)
        torch.cuda.synchronize()
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(iters):
            fn(k % 3)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / iters * 1e3
        tf = fl / (us * 1e-6) / 1e12
        out[name] = {"us": round(us, 1), "tflops": round(tf, 1), "frac_bf16_peak": round(tf / peaks["bf16"], 3)}
    out["tokens_per_s_fwd_bwd"] = round(T / ((out["fwd"]["us"] + out["bwd"]["us"]) * 1e-6), 1)
    out["config"] = f"T={T} (config-2 batch), hidden {hid}, heads {H}, p_attn = p_hidden = 0.1, GEMMs via cuBLASLt"
    return out


def planned_imbalance(args, steps=20):
    """Token imbalance (max/mean - 1) that the library's planner (ub_balance_plan, the code
    the exchange runs) produces for W = 2, 4, 8 ranks of 56 sequences; 'before' = no
    exchange.  A pure function of the plan, so it is exact without 8 GPUs."""
    from paper_2208_08124_b200 import api
    out = {}
    for W in (2, 4, 8):
        rec = {"before": [], "paper": [], "snake": [], "lpt": [], "stay": []}
        moved = {m: [] for m in ("paper", "paper+locality", "lpt", "lpt+locality", "stay")}
        for skew in ("iid", "sorted-block"):
            for k in range(steps):
                a = synth.skewed_rank_lengths(W, B, 1000 + k, skew, args.dist)
                tok = a.sum(axis=1).astype(np.float64)
                rec["before"].append(tok.max() / tok.mean() - 1)
                for mode in ("paper", "snake", "lpt", "stay"):
                    rt = api.balance_plan(a.reshape(-1), W, B, S, mode)["rank_tokens"].astype(np.float64)
                    rec[mode].append(rt.max() / rt.mean() - 1)
                if skew == "iid":
                    flat = a.reshape(-1)
                    for mode in moved:
                        perm = api.balance_plan(flat, W, B, S, mode)["perm"]
                        kept = sum(int(flat[g]) for r in range(W) for g in perm[r * B:(r + 1) * B] if g // B == r)
                        moved[mode].append(1.0 - kept / float(flat.sum()))
        out[f"w{W}"] = {k: {"mean": round(float(np.mean(v)), 5), "max": round(float(np.max(v)), 5)}
                        for k, v in rec.items()}
        out[f"w{W}"]["moved_token_fraction"] = {k: round(float(np.mean(v)), 4) for k, v in moved.items()}
    out["note"] = (f"{steps} steps x (iid, sorted-block) skews, {args.dist}, B={B}/rank; moved_token_fraction: "
                   "share of tokens the all-to-all-v moves (iid skew), without / with the locality relabeling (R24)")
    return out


def _patch_lse(wl, n):
    """The ABI wants lse as a dense [H, T] array: view the front of the buffer per step."""
    T = wl.ex[n % N_EX]["T"]
    if not hasattr(wl, "lse_full"):
        wl.lse_full = wl.lse
    wl.lse = wl.lse_full.view(-1)[:H * max(T, 1)].view(H, max(T, 1))


def run_e2e(args, wl, world):
    """Same step through the public API with HOST inputs: per step the padded input
    records, lengths, sample records, qkv and dO are copied H2D from pinned memory and the
    step's result (dqkv) is read back D2H, all inside the timed region.  Copies run on their
    own streams (H2D of step n+1 and D2H of step n-1 overlap step n's kernels), so the
    number is bound by PCIe, as a data-loading pipeline would be."""
    host = []
    for s in range(N_SETS):
        st = wl.sets[s]
        host.append({"recs": st["padded_recs"].cpu().pin_memory(), "lengths": st["lengths"].cpu().pin_memory(),
                     "samples": st["samples"].cpu().pin_memory(),
                     "qkv": st["qkv"][:wl.cap].cpu().pin_memory(), "dout": st["dout"].cpu().pin_memory()})
    dq_host = [torch.empty((wl.cap, 3, H, D), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    dq_dev = [wl.dqkv, torch.empty_like(wl.dqkv)]
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    set_free = [torch.cuda.Event() for _ in range(N_SETS)]     # main stream finished with set s
    set_ready = [torch.cuda.Event() for _ in range(N_SETS)]    # qkv/dO of set s copied in
    dq_free = [torch.cuda.Event() for _ in range(2)]           # D2H of dq buffer i finished
    h2d = d2h = 0

    def load_records(n):
        """H2D of step n's input records, lengths and sample records (side stream), then the
        exchange's first phase (lengths all-gather)."""
        nonlocal h2d
        s = n % N_SETS
        st, hs = wl.sets[s], host[s]
        wl.side.wait_event(set_free[s])
        with torch.cuda.stream(wl.side):
            st["padded_recs"].copy_(hs["recs"], non_blocking=True)
            st["lengths"].copy_(hs["lengths"], non_blocking=True)
            st["samples"].copy_(hs["samples"], non_blocking=True)
        wl.begin(n)
        h2d += hs["recs"].numel() * 4 + B * 4 + B * 4

    def load(n):
        """Second phase of step n's exchange, then H2D of its qkv / dO (rows = this rank's
        post-exchange T) on h2d_s."""
        nonlocal h2d
        s = n % N_SETS
        st, hs = wl.sets[s], host[s]
        wl.finish(n)
        T = wl.ex[n % N_EX]["T"]
        h2d_s.wait_event(set_free[s])
        with torch.cuda.stream(h2d_s):
            st["qkv"][:T].copy_(hs["qkv"][:T], non_blocking=True)
            st["dout"][:T].copy_(hs["dout"][:T], non_blocking=True)
        set_ready[s].record(h2d_s)
        h2d += T * 3 * H * D * 2 + T * H * D * 2

    def one(n):
        nonlocal d2h
        s, i = n % N_SETS, n % 2
        T = wl.ex[n % N_EX]["T"]
        wl.main.wait_event(set_ready[s])
        wl.main.wait_event(dq_free[i])
        wl.dqkv = dq_dev[i]
        _patch_lse(wl, n)
        wl.step(n)
        set_free[s].record(wl.main)
        d2h_s.wait_event(set_free[s])
        with torch.cuda.stream(d2h_s):
            dq_host[i][:T].copy_(dq_dev[i][:T], non_blocking=True)
        dq_free[i].record(d2h_s)
        d2h += T * 3 * H * D * 2
        load(n + 1)
        load_records(n + 2)
        return T

    base = 10 ** 6
    load_records(base)
    load_records(base + 1)
    load(base)
    for n in range(min(args.warmup, 3)):
        one(base + n)
    torch.cuda.synchronize()
    barrier(world)
    n0 = base + min(args.warmup, 3)
    h2d = d2h = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(wl.main)
    tok = 0
    for k in range(args.steps):
        tok += one(n0 + k)
    # steady state: the K steps' kernels and D2H, and K H2D loads (qkv/dO of steps
    # n0+1 .. n0+K, records of n0+2 .. n0+K+1; the earlier ones were issued in the warm-up)
    wl.main.wait_stream(d2h_s)
    wl.main.wait_stream(h2d_s)
    wl.main.wait_stream(wl.side)
    e1.record(wl.main)
    torch.cuda.synchronize()
    barrier(world)
    wl.dqkv = dq_dev[0]
    wl.finish(n0 + args.steps + 1)              # drain the begin still in flight (untimed)
    torch.cuda.synchronize()
    ms = all_max(e0.elapsed_time(e1), world)
    tok_all = all_sum(tok, world)
    return {"value": round(tok_all / (ms / 1e3), 1), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d // args.steps),
            "d2h_bytes_per_step": int(d2h // args.steps)}


def main():
    args = parse()
    json_out = _claim_stdout()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        out = run_reference(args, world, rank)
        if out is not None:
            print(json.dumps(out), file=json_out, flush=True)
        return
    world, rank, local = dist_init(args.gpus)
    out, wl = run_ours(args, world, rank, local)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(out), file=json_out, flush=True)
    wl.comm.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
