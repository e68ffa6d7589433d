#!/bin/bash
# A/B (dev): SMs left free for the side-stream exchange by the persistent FMHA grids
B() { timeout 300 python bench.py --steps 60 --warmup 5 --no-e2e --no-cpu-baseline --no-encoder "$@" 2>/tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value']/1e6,2), d['step_us_distribution']['median'], 'p90', d['step_us_distribution']['p90'], 'fwd', d['kernels']['fmha_fwd']['us'], 'bwd', d['kernels']['fmha_bwd']['us'], 'p0', round(d['p0_step']['value']/1e6,2), 'exposed', d['exchange_overlap']['exposed_exchange_us'])" || tail -5 /tmp/err.txt; }
for r in 1 2; do for k in 4 2 1; do echo "reserve $k: $(B --reserve-sms $k)"; done; done
