#!/bin/bash
# Round profiling on the GPU box (1 GPU): GPU tests, smoke, bench line, ncu launch list,
# ncu --set full of the two FMHA main kernels, ncu DRAM bytes of the gather kernels, sanitizer.
# Outputs land in gpurun_out/ (summarised into profiles/ by scripts/ncu_summary.py TAG).
set -x
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt
timeout -k 10 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout -k 10 900 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout -k 10 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-encoder \
    > gpurun_out/launches_$TAG.log 2>&1
# the headline configuration: p = 0.1 with the step's materialised keep bits (probe_time.py
# passes the mask for p > 0); the p = 0 kernels as prof_{fwd,bwd}0_TAG
for K in fwd bwd; do
  timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:fmha_${K}_kernel -s 3 -c 1 \
      -o gpurun_out/prof_${K}_$TAG -f python scripts/probe_time.py mlperf_like_v0 0.1 > gpurun_out/ncu_${K}_$TAG.log 2>&1
  timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:fmha_${K}_kernel -s 3 -c 1 \
      -o gpurun_out/prof_${K}0_$TAG -f python scripts/probe_time.py mlperf_like_v0 0.0 > gpurun_out/ncu_${K}0_$TAG.log 2>&1
done
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:dropout_mask -s 3 -c 1 \
    -o gpurun_out/prof_mask_$TAG -f python scripts/probe_mask.py > gpurun_out/ncu_mask_$TAG.log 2>&1
timeout -k 10 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"span_copy|span_bulk|exchange_copy" -c 15 --csv --log-file gpurun_out/gather_$TAG.csv env PROBE_N=2 python scripts/probe_gather.py \
    > gpurun_out/gather_$TAG.log 2>&1
# (compute-sanitizer is closed on this pool since round 2: the r02 logs under profiles/sanitizer stand)
tail -2 gpurun_out/pytest_gpu_$TAG.log; tail -1 gpurun_out/smoke_$TAG.log
ls -la gpurun_out | tail -5
