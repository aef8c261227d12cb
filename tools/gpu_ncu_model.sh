#!/bin/bash
# one ncu --set full capture of k_log_psi (amplitude evaluation) for one config
# usage: gpurun -- 'bash tools/gpu_ncu_model.sh TAG CONFIG [N_UNQ]'
TAG=$1; CFG=${2:-c118}; N=${3:-200000}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_log_psi_part -s 2 -c 1 \
    -o $OUT/logpsi_$CFG python tools/bench_model.py --config $CFG --n-unq $N --steps 1 --warmup 2 --cpu-sample 10 \
    > /dev/null 2>&1
ls -la $OUT
