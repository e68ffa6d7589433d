#!/bin/bash
for pk in 0 1; do for v in 0 1 2 3 4; do echo "poly=$v pack=$pk"; UB_FWD_PACK=$pk UB_FWD_POLY=$v timeout 120 python scripts/probe_time.py 2>&1 | tail -1; done; done
