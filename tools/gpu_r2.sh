#!/bin/bash
# Round-2 quick check: GPU tests, smoke, bench c118/c56 (default split path, and QVMC_FUSED=1).
TAG=${1:-r2a}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
for cfg in c118 c56; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline > $OUT/bench_$cfg.json 2> $OUT/bench_$cfg.err
  QVMC_FUSED=1 timeout 600 python bench.py --config $cfg --no-cpu-baseline --e2e-steps 0 > $OUT/bench_${cfg}_fused.json 2> $OUT/bench_${cfg}_fused.err
done
tail -n 3 $OUT/pytest_gpu.log $OUT/smoke.log
for f in $OUT/bench_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(sys.argv[1].split("/")[-1], f"value {d['value']:.4g} step {d['ms_per_step']:.2f} rows {d['stages_ms']['rows']:.2f} table {d['stages_ms']['table_build']:.2f} search {r.get('search_ms', 0):.2f} eval {r.get('eval_ms', 0):.2f} cand {d['path_stats']['candidates_per_sample']:.0f}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
