#!/bin/bash
# ncu --set full (source counters) of the hot kernels on one cfg-3 layer.
# usage: tools/gpu_ncu.sh <tag> [workload] [kernel-regex...]
TAG=${1:-r}
WL=${2:-cfg3}
shift 2
KS=${@:-k_attn k_score_tbl k_topk}
mkdir -p gpurun_out
for K in $KS; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
      -o gpurun_out/prof_${TAG}_${K} python tools/prof_step.py --workload $WL > gpurun_out/prof_${TAG}_${K}.log 2>&1
done
