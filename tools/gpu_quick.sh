#!/bin/bash
# Quick GPU iteration: parity tests, bench line, per-kernel launch times (ncu, warm caches).
# usage: tools/gpu_quick.sh <tag> [workload] [pytest-args...]
TAG=${1:-q}
WL=${2:-cfg3}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 240 > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
timeout 300 python bench.py --workload $WL --no-cpu-baseline > gpurun_out/bench_${TAG}.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 200 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --workload $WL --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_${TAG}.csv > gpurun_out/launches_${TAG}.txt 2>&1
