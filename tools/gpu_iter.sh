#!/bin/bash
# GPU iteration: parity tests, bench lines for the 1-GPU and per-GPU-shard shapes, and a
# launch list of the step kernels (ncu, device time per launch).
# usage: tools/gpu_iter.sh <tag> [skip-tests]
TAG=${1:-it}
mkdir -p gpurun_out
if [ -z "$2" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log; tail -3 gpurun_out/pytest_${TAG}.log
fi
for A in "cfg3" "cfg3 --shard-of 8" "cfg1" "cfg5 --shard-of 8"; do
  N=$(echo $A | tr ' ' '_' | tr -d '-')
  timeout 400 python bench.py --workload $A --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_${N}.json 2> gpurun_out/bench_${TAG}_${N}.err
  python - "$N" gpurun_out/bench_${TAG}_${N}.json <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
    print(sys.argv[1], "value %.0f" % d["value"], {k: round(v, 1) for k, v in d["kernels_us"].items() if k != "select_bytes"},
          "attn_frac %.3f" % d["roofline"]["frac"], "verified", d["verified"], "proj", (d.get("projected") or {}).get("aggregate_tokens_per_s"))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
for A in "cfg3" "cfg3 --shard-of 8"; do
  N=$(echo $A | tr ' ' '_' | tr -d '-')
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_select|k_attn|k_score|k_topk" -c 48 --csv \
    --log-file gpurun_out/launches_${TAG}_${N}.csv python bench.py --workload $A --steps 4 --warmup 3 --no-cpu-baseline --no-verify > /dev/null 2>&1
  echo "== launches $N"; python tools/launches.py gpurun_out/launches_${TAG}_${N}.csv
done
