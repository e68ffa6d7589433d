#!/bin/bash
# A/B (dev): probe_time kernels at p = 0.1 / 0 and the headline bench step for library variants.
# Usage: bash scripts/ab_step.sh tag1 tag2 ...   (tag "new" = libub.so, else libub_<tag>.so)
lib() { if [ "$1" = "new" ]; then echo $PWD/paper_2208_08124_b200/libub.so; else echo $PWD/paper_2208_08124_b200/libub_$1.so; fi; }
for r in 1 2; do for T in "$@"; do
  echo "$T: $(UB_LIB=$(lib $T) timeout 120 python scripts/probe_time.py mlperf_like_v0 0.1)"
  echo "$T: $(UB_LIB=$(lib $T) timeout 120 python scripts/probe_time.py mlperf_like_v0 0.0)"
done; done
for r in 1 2; do for T in "$@"; do
  echo "$T bench: $(UB_LIB=$(lib $T) timeout 300 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-encoder 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value']/1e6,2), d['step_us_distribution']['median'], d['kernels']['fmha_fwd']['us'], d['kernels']['fmha_bwd']['us'], 'p0', round(d['p0_step']['value']/1e6,2))")"
done; done
