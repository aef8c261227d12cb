#!/bin/bash
# BASELINE config 5: unique-sample sweep at 56 qubits (1 GPU). usage: bash tools/gpu_sweep.sh TAG
TAG=$1; mkdir -p gpurun_out/$TAG
for n in 1000 10000 100000 1000000 10000000; do
  timeout 900 python bench.py --config c56 --n-unq $n --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 \
      > gpurun_out/$TAG/sweep_$n.json 2> gpurun_out/$TAG/sweep_$n.err
  python - gpurun_out/$TAG/sweep_$n.json $n <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"n_unq {sys.argv[2]:>9}  value {d['value']:.4g}/s  step {d['ms_per_step']:.3f} ms  rows {d['stages_ms']['rows']:.3f}  table {d['stages_ms']['table_build']:.3f}  e2e {d['e2e']['value']:.4g}/s")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
