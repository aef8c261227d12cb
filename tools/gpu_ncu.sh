#!/bin/bash
# one ncu --set full capture each of the search and the evaluation kernel for one config
# usage: gpurun -- 'bash tools/gpu_ncu.sh TAG CONFIG'
TAG=$1; CFG=${2:-c118}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows_join -s 3 -c 1 \
    -o $OUT/search_$CFG python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval_chunks -s 3 -c 1 \
    -o $OUT/eval_$CFG python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ls -la $OUT
