#!/bin/bash
# compute-sanitizer over the tiny-shape workload (scripts/sanitize.py), one log per tool.
# Usage (GPU box): bash scripts/sanitize.sh TAG   -> gpurun_out/sanitize_<tool>_TAG.log
TAG=${1:-r02}
mkdir -p gpurun_out
for TOOL in memcheck initcheck synccheck racecheck; do
  EXTRA=""
  [ "$TOOL" = "memcheck" ] && EXTRA="--leak-check full"
  ZERO=0
  [ "$TOOL" = "initcheck" ] && ZERO=1        # see scripts/sanitize.py:_zero_init_mode
  SANITIZE_ZERO=$ZERO timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL $EXTRA --print-limit 50 \
      python scripts/sanitize.py > gpurun_out/sanitize_${TOOL}_$TAG.log 2>&1
  echo "$TOOL rc=$?" >> gpurun_out/sanitize_$TAG.summary
  tail -3 gpurun_out/sanitize_${TOOL}_$TAG.log >> gpurun_out/sanitize_$TAG.summary
done
cat gpurun_out/sanitize_$TAG.summary
