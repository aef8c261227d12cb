#!/bin/bash
# Measurement pass: integer/issue peaks, per-kernel instruction + DRAM counts of one
# bench step (c118, c56), launch list, and ncu --set full of the top kernels.
# usage: gpurun --timeout 3000 -- 'bash tools/gpu_profile_r2.sh TAG [full]'
TAG=${1:-prof}; FULL=${2:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
make -s -C paper_2408_07625_b200/csrc > $OUT/make.log 2>&1 || { echo build failed; exit 1; }
( cd tools/micro && nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o int_rates int_rates.cu ) > $OUT/int_rates_build.log 2>&1
./tools/micro/int_rates > $OUT/int_rates_b200.json 2> $OUT/int_rates.err
cat $OUT/int_rates_b200.json
for CFG in c118 c56; do
  timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --profile-from-start off --csv --log-file $OUT/step_$CFG.csv \
      python bench.py --config $CFG --steps 1 --warmup 2 --no-cpu-baseline --e2e-steps 0 --profile-step > $OUT/step_$CFG.log 2>&1
  python tools/ncu_step_metrics.py $CFG $OUT/step_$CFG.csv > $OUT/step_$CFG.json 2>&1
  cp profiles/ncu_step_$CFG.json $OUT/ 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > $OUT/launches_bench.log 2>&1
python tools/launch_summary.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1
if [ -n "$FULL" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows_join -s 3 -c 1 \
      -o $OUT/search_c118 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval_chunks -s 3 -c 1 \
      -o $OUT/eval_c118 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
fi
cat $OUT/launches_summary.txt | head -20
ls -la $OUT
