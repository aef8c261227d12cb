#!/bin/bash
# One gpurun call: launch list + one ncu --set full capture of the row kernel for each config.
# usage: gpurun -- 'bash tools/gpu_profile.sh TAG "c118 c56" [kernel-regex]'
TAG=$1; CFGS=$2; KRE=${3:-k_rows}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for cfg in $CFGS; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$cfg.csv \
      python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $OUT/launches_$cfg.log 2>&1
  python tools/launch_summary.py $OUT/launches_$cfg.csv > $OUT/launches_$cfg.txt
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 \
      -o $OUT/rows_$cfg python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_$cfg.log 2>&1
done
