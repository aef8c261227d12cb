#!/bin/bash
# c56 small-size sweep: normal vs speculative + CUDA graph steps
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
for n in 1000 10000 100000 1000000; do
  for mode in plain graph; do
    extra=""; [ $mode = graph ] && extra="--graph"
    timeout 600 python bench.py --config c56 --n-unq $n --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 $extra \
      > $OUT/c56_${n}_$mode.json 2> $OUT/c56_${n}_$mode.err
    python - $OUT/c56_${n}_$mode.json $n $mode <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"n {sys.argv[2]:>8} {sys.argv[3]:6} value {d['value']:.4g}/s step {d['ms_per_step']:.4f} ms launches {d['gpu_launches']}")
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e)
PY
  done
done
