#!/bin/bash
# Round-end evidence in one gpurun call: GPU tests, smoke, bench lines (ours + reference arm),
# launch lists, and one ncu --set full capture each of the search and evaluation kernels.
TAG=${1:-final}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c118.json 2> $OUT/bench_c118.err
timeout 600 python bench.py --config c56 > $OUT/bench_c56.json 2> $OUT/bench_c56.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_c118.json 2> $OUT/bench_ref_c118.err
for cfg in c118 c56; do
  timeout 300 python tools/bench_model.py --config $cfg > $OUT/bench_model_$cfg.json 2> $OUT/bench_model_$cfg.err
done
# (gpurun brings back <= 64 MiB: the ncu captures go in separate calls, tools/gpu_ncu.sh)
for cfg in c118 c56; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$cfg.csv \
      python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  python tools/launch_summary.py $OUT/launches_$cfg.csv > $OUT/launches_$cfg.txt
  rm -f $OUT/launches_$cfg.csv
done
tail -n 2 $OUT/pytest_gpu.log $OUT/smoke.log
