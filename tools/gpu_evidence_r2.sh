#!/bin/bash
# Round-2 evidence in one call: compute-sanitizer over every device path, BASELINE config 2 (c20, 1e5)
# and the config-5 sweep (c56, 1e3..1e7) with the CPU reference per size.
TAG=${1:-r2ev}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_driver.py > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/sanitize_$tool.log
  tail -3 $OUT/sanitize_$tool.log
done
timeout 900 python bench.py --config c20 > $OUT/bench_c20.json 2> $OUT/bench_c20.err
tail -c 600 $OUT/bench_c20.json
for n in 1000 10000 100000 1000000 10000000; do
  timeout 900 python bench.py --config c56 --n-unq $n --steps 5 --warmup 3 --e2e-steps 2 \
      > $OUT/sweep_c56_$n.json 2> $OUT/sweep_c56_$n.err
  python - $OUT/sweep_c56_$n.json $n <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    cb = d.get("cpu_baseline") or {}
    print(f"n_unq {sys.argv[2]:>9}  value {d['value']:.4g}/s  step {d['ms_per_step']:.3f} ms  rows {d['stages_ms']['rows']:.3f}  table {d['stages_ms']['table_build']:.3f}  e2e {d['e2e']['value']:.4g}/s  cpu {cb.get('value', 0):.4g}/s  frac {d['roofline']['frac']:.3f} {d['roofline']['bound']}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
