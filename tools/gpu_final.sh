#!/bin/bash
# Round measurement set (GPU box): bench lines for every BASELINE.json workload at its
# per-GPU shape, the reference arm, the launch list and ncu captures of the two step
# kernels at cfg3. usage: tools/gpu_final.sh <tag>
TAG=${1:-final}
mkdir -p gpurun_out
run() {  # name, args...
  local N=$1; shift
  timeout 400 python bench.py "$@" > gpurun_out/bench_${TAG}_${N}.json 2> gpurun_out/bench_${TAG}_${N}.err
  python - "$N" gpurun_out/bench_${TAG}_${N}.json <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
    print(sys.argv[1], "value %.0f" % d["value"], "e2e %.0f" % d["e2e"]["value"],
          {k: round(v, 1) for k, v in d["kernels_us"].items() if k != "select_bytes"},
          "attn_frac %.3f" % d["roofline"]["frac"], "step_frac %.3f" % d["step_roofline"]["frac"],
          "verified", d["verified"], "proj", (d.get("projected") or {}).get("aggregate_tokens_per_s"))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
}
run cfg3 --workload cfg3 --steps 100 --warmup 10
run cfg3_s2 --workload cfg3 --shard-of 2 --steps 100 --warmup 10 --no-cpu-baseline
run cfg3_s4 --workload cfg3 --shard-of 4 --steps 100 --warmup 10 --no-cpu-baseline
run cfg3_s8 --workload cfg3 --shard-of 8 --steps 100 --warmup 10 --no-cpu-baseline
run cfg1 --workload cfg1 --steps 100 --warmup 10 --cpu-reps 3
run cfg1_s8 --workload cfg1 --shard-of 8 --steps 100 --warmup 10 --no-cpu-baseline
run cfg2 --workload cfg2 --steps 20 --warmup 5 --cpu-reps 2
run cfg4u_s8 --workload cfg4u --shard-of 8 --steps 100 --warmup 10 --no-cpu-baseline
run cfg4a_s8 --workload cfg4a --shard-of 8 --steps 100 --warmup 10 --no-cpu-baseline
run cfg5_s8 --workload cfg5 --shard-of 8 --steps 100 --warmup 10 --no-cpu-baseline
run cfg5 --workload cfg5 --steps 20 --warmup 5 --cpu-reps 2
timeout 300 python bench.py --impl reference --workload cfg3 --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_ref_cfg3.json 2>/dev/null
echo "ref"; cat gpurun_out/bench_${TAG}_ref_cfg3.json
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_select|k_attn" -c 40 --csv \
    --log-file gpurun_out/launches_${TAG}_cfg3.csv python bench.py --workload cfg3 --steps 4 --warmup 3 --no-cpu-baseline --no-verify > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_${TAG}_cfg3.csv
for K in k_attn k_select; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
      -o gpurun_out/prof_${TAG}_${K} python tools/prof_step.py --workload cfg3 > gpurun_out/prof_${TAG}_${K}.log 2>&1
  echo "ncu $K rc=$?"
done
