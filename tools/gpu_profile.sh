#!/bin/bash
# Run on the GPU box: launch list of a short bench + one ncu --set full per hot kernel.
# usage: tools/gpu_profile.sh <tag> [workload]
set -x
TAG=${1:-r1}
WL=${2:-cfg3}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --workload $WL --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench_${TAG}.log 2>&1
for K in k_attn k_score_tbl k_topk k_merge; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
      -o gpurun_out/prof_${TAG}_${K} python tools/prof_step.py --workload $WL > gpurun_out/prof_${TAG}_${K}.log 2>&1
done
