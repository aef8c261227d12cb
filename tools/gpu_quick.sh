#!/bin/bash
# quick iteration: selected GPU tests (-k EXPR) then c118/c56 bench lines
TAG=$1; K=${2:-large_bucket}; OUT=gpurun_out/$TAG; mkdir -p $OUT
make -s -C paper_2408_07625_b200/csrc > $OUT/make.log 2>&1 || { echo 'build failed'; tail $OUT/make.log; exit 1; }  # never measure a stale .so
timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > $OUT/pytest_sel.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_sel.log
tail -n 15 $OUT/pytest_sel.log
for cfg in c118 c56; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline --e2e-steps 1 > $OUT/bench_$cfg.json 2> $OUT/bench_$cfg.err
  python - "$OUT/bench_$cfg.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(sys.argv[1].split("/")[-1], f"value {d['value']:.4g} step {d['ms_per_step']:.2f} rows {d['stages_ms']['rows']:.2f} table {d['stages_ms']['table_build']:.2f} search {r.get('search_ms', 0):.2f} eval {r.get('eval_ms', 0):.2f} cand {d['path_stats']['candidates_per_sample']:.0f}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
  tail -n 3 $OUT/bench_$cfg.err
done
