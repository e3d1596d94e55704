#!/bin/bash
# A/B of prebuilt library variants on the same box: bench lines (no CPU baseline) for each
# workload, variants alternated twice. usage: tools/gpu_ab.sh <tag> <lib_a.so> <lib_b.so> ...
# (libraries under paper_2605_12110_b200/lib/, selected per run through ABSP_LIB;
# AB_WORKLOADS="cfg3,cfg5 --shard-of 8" overrides the workload list)
TAG=$1; shift
mkdir -p gpurun_out
IFS=',' read -ra WLS <<< "${AB_WORKLOADS:-cfg3,cfg3 --shard-of 8,cfg3 --shard-of 2,cfg5 --shard-of 8,cfg1}"
for A in "${WLS[@]}"; do
  N=$(echo $A | tr ' ' '_' | tr -d '-')
  for rep in 1 2; do
    for LIBV in "$@"; do
      OUT=gpurun_out/ab_${TAG}_${N}_${LIBV%.so}_${rep}.json
      ABSP_LIB=$LIBV timeout 400 python bench.py --workload $A --steps 50 --warmup 5 --no-cpu-baseline > $OUT 2> ${OUT%.json}.err
      python - "$N $LIBV $rep" $OUT <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
    print(sys.argv[1], "value %.0f" % d["value"], {k: round(v, 1) for k, v in d["kernels_us"].items() if k != "select_bytes"},
          "attn_frac %.3f" % d["roofline"]["frac"], "verified", d["verified"])
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
    done
  done
done
