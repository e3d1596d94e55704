#!/bin/bash
# Round-end verification on the GPU box: the full GPU test suite, smoke(), the sanitizer
# set, then the measurement set (tools/gpu_final.sh). usage: tools/gpu_round_end.sh <tag>
TAG=${1:-end}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/smoke_${TAG}.log
timeout 1500 bash tools/gpu_sanitize.sh ${TAG}
timeout 2400 bash tools/gpu_final.sh ${TAG}
