#!/bin/bash
# usage: prof_one.sh TAG KERNEL_REGEX [env...]  -> gpurun_out/prof_TAG.ncu-rep
TAG=$1; K=$2
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
   -o gpurun_out/prof_$TAG -f python scripts/probe_time.py > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
