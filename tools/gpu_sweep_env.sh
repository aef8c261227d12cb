#!/bin/bash
# bench one config under several values of an environment knob
# usage: gpurun -- 'bash tools/gpu_sweep_env.sh TAG CFG VAR "v1 v2 ..." [extra bench args]'
TAG=$1; CFG=$2; VAR=$3; VALS=$4; shift 4
OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --config $CFG --no-cpu-baseline --e2e-steps 0 --steps 5 "$@" > $OUT/bench_${CFG}_${VAR}_$v.json 2> $OUT/bench_${CFG}_${VAR}_$v.err
  python - "$OUT/bench_${CFG}_${VAR}_$v.json" "$CFG $VAR=$v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(sys.argv[2], f"value {d['value']:.4g} step {d['ms_per_step']:.2f} rows {d['stages_ms']['rows']:.2f} table {d['stages_ms']['table_build']:.2f} search {r.get('search_ms', 0):.2f} eval {r.get('eval_ms', 0):.2f}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
