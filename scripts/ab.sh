#!/bin/bash
# A/B timing of library variants: scripts/ab.sh libA.so libB.so ...  (probe_time, 3 runs each, interleaved)
for r in 1 2 3; do for L in "$@"; do echo -n "$L: "; UB_LIB=$PWD/paper_2208_08124_b200/$L timeout 120 python scripts/probe_time.py ${DIST:-mlperf_like_v0} ${P:-0.0}; done; done
