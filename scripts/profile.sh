#!/bin/bash
# Round profiling on the GPU box (1 GPU): GPU tests, smoke, bench line, ncu launch list,
# ncu --set full of the two FMHA main kernels.  Outputs land in gpurun_out/ (summarised into
# profiles/ by scripts/ncu_summary.py TAG).
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
    > gpurun_out/launches_$TAG.log 2>&1
for K in fwd bwd; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fmha_${K}_kernel -s 3 -c 1 \
      -o gpurun_out/prof_${K}_$TAG -f python scripts/probe_time.py > gpurun_out/ncu_${K}_$TAG.log 2>&1
done
tail -2 gpurun_out/pytest_gpu_$TAG.log; tail -1 gpurun_out/smoke_$TAG.log
ls -la gpurun_out
