#!/bin/bash
# A/B (dev): the headline step's options on the prebound pipeline (100 steps each)
B() { timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-encoder "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); x=d['step_us_distribution']; print(round(d['value']/1e6,2), 'median', x['median'], 'mean', x['mean'], 'fwd', d['kernels']['fmha_fwd']['us'], 'bwd', d['kernels']['fmha_bwd']['us'], 'p0', round(d['p0_step']['value']/1e6,2))"; }
for r in 1 2; do
  echo "default:      $(B)"
  echo "mask-ov 0:    $(B --mask-overlap 0)"
  echo "schedule 2:   $(B --schedule 2)"
  echo "reserve 2:    $(B --reserve-sms 2)"
done
