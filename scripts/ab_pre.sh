#!/bin/bash
# A/B (dev): the backward's Delta prologue grid (one wave / two waves / one CTA per row block)
timeout 300 python -m pytest tests/test_gpu_fmha.py -q -x -k "config2 or edge" 2>&1 | tail -1
B() { timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-encoder 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); x=d['step_us_distribution']; print(round(d['value']/1e6,2), 'median', x['median'], 'mean', x['mean'], 'f2b', d['main_stream_timeline']['fwd_end_to_bwd_main_us'], 'p0', round(d['p0_step']['value']/1e6,2))"; }
for r in 1 2; do for T in pre0 new pre2; do
  if [ $T = new ]; then L=$PWD/paper_2208_08124_b200/libub.so; else L=$PWD/paper_2208_08124_b200/libub_$T.so; fi
  echo "$T: $(UB_LIB=$L B)"
done; done
