#!/bin/bash
# A/B (dev): exchange pipeline depth of the bench step (UB_BENCH_PIPE)
for r in 1 2; do for P in 3 5; do echo "pipe $P: $(UB_BENCH_PIPE=$P timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-encoder 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); x=d['step_us_distribution']; print(round(d['value']/1e6,2), 'median', x['median'], 'mean', x['mean'], 'slowest', x['slowest'], 'p0', round(d['p0_step']['value']/1e6,2))")"; done; done
