#!/bin/bash
# Bench every BASELINE.json workload once (bounded steps) -> gpurun_out/allcfg_<tag>_<wl>.json
TAG=${1:-a}
mkdir -p gpurun_out
for WL in cfg1 cfg2 cfg3 cfg4u cfg4a cfg5; do
  timeout 400 python bench.py --workload $WL --steps 50 --warmup 5 --cpu-reps 2 > gpurun_out/allcfg_${TAG}_${WL}.json 2> gpurun_out/allcfg_${TAG}_${WL}.err
done
