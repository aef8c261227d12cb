#!/bin/bash
# One gpurun call: GPU parity tests with the main library, then a short bench per tuning variant.
# usage: gpurun -- 'bash tools/gpu_variants.sh TAG "c118 c56" v1 v2 ...'
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -n 3 $OUT/pytest_gpu.log
for cfg in $CFGS; do
  for v in main "$@"; do
    lib=paper_2408_07625_b200/lib/libqvmc_cuda.so
    [ "$v" != main ] && lib=paper_2408_07625_b200/lib/variants/libqvmc_cuda_$v.so
    QVMC_CUDA_LIB=$lib timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 \
      > $OUT/bench_${cfg}_$v.json 2> $OUT/bench_${cfg}_$v.err
    python - "$OUT/bench_${cfg}_$v.json" "$cfg" "$v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:5} {sys.argv[3]:8} value {d['value']:.4g}  rows {d['stages_ms']['rows']:.2f} ms  table {d['stages_ms']['table_build']:.2f} ms  cand/s {d['path_stats']['candidates_per_sample']:.0f} pairs/s {d['path_stats']['pairs_per_sample']:.1f}")
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e)
PY
  done
done
