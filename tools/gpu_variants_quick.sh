#!/bin/bash
# short bench per tuning variant (no tests): usage gpurun -- 'bash tools/gpu_variants_quick.sh TAG "c118 c56" v1 v2 ...'
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
for cfg in $CFGS; do
  for v in main "$@"; do
    lib=paper_2408_07625_b200/lib/libqvmc_cuda.so
    [ "$v" != main ] && lib=paper_2408_07625_b200/lib/variants/libqvmc_cuda_$v.so
    QVMC_CUDA_LIB=$lib timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 0 \
      > $OUT/bench_${cfg}_$v.json 2> $OUT/bench_${cfg}_$v.err
    python - "$OUT/bench_${cfg}_$v.json" "$cfg" "$v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(f"{sys.argv[2]:5} {sys.argv[3]:8} value {d['value']:.4g}  rows {d['stages_ms']['rows']:.2f} ms  table {d['stages_ms']['table_build']:.2f} ms search {r.get('search_ms', 0):.2f} eval {r.get('eval_ms', 0):.2f}")
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e)
PY
  done
done
