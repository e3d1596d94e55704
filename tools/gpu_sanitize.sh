#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_step.py
# (every kernel-launching entry point on a cfg1-sized layer). usage: tools/gpu_sanitize.sh <tag>
TAG=${1:-san}
mkdir -p gpurun_out
for T in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $T --error-exitcode 99 --print-limit 50 \
      python tools/sanitize_step.py > gpurun_out/sanitize_${TAG}_${T}.log 2>&1
  echo "$T rc=$?"; tail -3 gpurun_out/sanitize_${TAG}_${T}.log
done
