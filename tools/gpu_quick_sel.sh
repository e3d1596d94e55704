#!/bin/bash
# Quick selection iteration: selection parity tests, step timelines (cfg3, its 8-GPU shard)
# and bench lines without the CPU baseline. usage: tools/gpu_quick_sel.sh <tag>
TAG=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullshape.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_${TAG}.log
for A in "cfg3" "cfg3 2"; do
  SEL_TRACE_WARM=1 timeout 300 python tools/select_trace.py $A 2>&1 | tail -12 | head -9 | sed "s/^/warm /"
  timeout 300 python tools/select_trace.py $A > gpurun_out/seltrace_${TAG}_$(echo $A | tr ' ' '_').txt 2>&1
  echo "== trace $A"; tail -17 gpurun_out/seltrace_${TAG}_$(echo $A | tr ' ' '_').txt
done
for A in "cfg3" "cfg3 --shard-of 8" "cfg5 --shard-of 8"; do
  N=$(echo $A | tr ' ' '_' | tr -d '-')
  timeout 400 python bench.py --workload $A --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_${N}.json 2> gpurun_out/bench_${TAG}_${N}.err
  python - "$N" gpurun_out/bench_${TAG}_${N}.json <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
    print(sys.argv[1], "value %.0f" % d["value"], {k: round(v, 1) for k, v in d["kernels_us"].items() if k != "select_bytes"},
          "attn_frac %.3f" % d["roofline"]["frac"], "verified", d["verified"])
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
