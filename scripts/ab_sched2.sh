#!/bin/bash
# A/B (dev): snake vs host LPT schedule of the backward, with and without the mask overlapping the backward's tail
B() { timeout 300 python bench.py --steps 60 --warmup 5 --no-e2e --no-cpu-baseline --no-encoder "$@" 2>/tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); m=d['main_stream_timeline']; print(round(d['value']/1e6,2), d['step_us_distribution']['median'], 'p90', d['step_us_distribution']['p90'], 'bwd', d['kernels']['fmha_bwd']['us'], 'p0', round(d['p0_step']['value']/1e6,2), d['host_us_per_step'])" || tail -5 /tmp/err.txt; }
for r in 1 2; do
  echo "snake ov1: $(B --schedule 0)"; echo "lpt   ov1: $(B --schedule 1)"
  echo "snake ov0: $(B --schedule 0 --mask-overlap 0)"; echo "lpt   ov0: $(B --schedule 1 --mask-overlap 0)"
done
