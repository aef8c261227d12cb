#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench lines, launch list, ncu capture of the hot kernel.
# usage (from this container): gpurun --timeout 2400 -- 'bash tools/gpu_check.sh [tag]'
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c118.json 2> $OUT/bench_c118.err
timeout 600 python bench.py --config c56 --no-cpu-baseline > $OUT/bench_c56.json 2> $OUT/bench_c56.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $OUT/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows -s 2 -c 1 \
    -o $OUT/rows python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_full.log 2>&1
tail -3 $OUT/*.log
cat $OUT/bench_c118.json $OUT/bench_c56.json
