#!/bin/bash
# A/B (dev): the headline bench step for library variants, interleaved, 3 runs each.
# Usage: bash scripts/ab_bench.sh tag1 tag2 ...   (tag "new" = libub.so, else libub_<tag>.so)
lib() { if [ "$1" = "new" ]; then echo $PWD/paper_2208_08124_b200/libub.so; else echo $PWD/paper_2208_08124_b200/libub_$1.so; fi; }
for r in 1 2 3; do for T in "$@"; do
  echo "$T bench: $(UB_LIB=$(lib $T) timeout 300 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-encoder 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); m=d['main_stream_timeline']; print(round(d['value']/1e6,2), d['step_us_distribution']['median'], 'fwd', d['kernels']['fmha_fwd']['us'], 'bwd', d['kernels']['fmha_bwd']['us'], 'f2b', m['fwd_end_to_bwd_main_us'], 'rest', m['rest_of_step_us'], 'p0', round(d['p0_step']['value']/1e6,2))")"
done; done
