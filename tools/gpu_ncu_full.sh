#!/bin/bash
# ncu --set full (with source counters) of one kernel of a decode step.
# usage: tools/gpu_ncu_full.sh <tag> <kernel-regex> <workload> [batch]
TAG=$1; K=$2; WL=${3:-cfg3}; B=${4:-0}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
    -o gpurun_out/prof_${TAG} python tools/prof_step.py --workload $WL --batch $B > gpurun_out/prof_${TAG}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/prof_${TAG}.log
