"""Dev probe: host time of each pipelined-step call (step / finish / begin) per timed step, to
find the step whose host work drains the GPU queue.  Runs bench.py's headline region once."""
import sys, time, os
sys.argv = ["bench.py", "--no-e2e", "--no-cpu-baseline", "--no-encoder"]
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
log = []
for name in ("step", "finish", "begin"):
    orig = getattr(bench.Workload, name)
    def wrap(self, n, *a, _o=orig, _nm=name, **k):
        t = time.perf_counter()
        r = _o(self, n, *a, **k)
        log.append((_nm, n, (time.perf_counter() - t) * 1e6))
        return r
    setattr(bench.Workload, name, wrap)
args = bench.parse()
world, rank, local = bench.dist_init(args.gpus)
import torch
wl = bench.Workload(args, world, rank, torch.device("cuda", local))
for rep in range(2):
    log.clear()
    ms, tok, nxt = bench.pipelined_region(wl, args, world, 1000 * (rep + 1), 0.1)
    worst = sorted(log, key=lambda x: -x[2])[:8]
    print(f"rep {rep}: {ms * 1e3:.1f} us/step; slowest host calls:", [(a, b, round(c, 1)) for a, b, c in worst])
