#!/bin/bash
# launch lists (ncu gpu__time_duration) for the given configs: bash tools/gpu_launches.sh TAG "c118 c56"
TAG=$1; CFGS=$2
mkdir -p gpurun_out/$TAG
for cfg in $CFGS; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$TAG/l_$cfg.csv \
      python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/$TAG/l_$cfg.csv > gpurun_out/$TAG/l_$cfg.txt
done
