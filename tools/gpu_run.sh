#!/bin/bash
# Generic gpurun step: GPU tests (optionally a subset), smoke, bench line.
# usage: gpurun --timeout 2400 -- 'bash tools/gpu_run.sh TAG "PYTEST_ARGS" [bench args...]'
TAG=${1:-r2}
PYARGS=${2:-"tests -m gpu"}
shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt
timeout 1500 python -m pytest $PYARGS -x -q -rs --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
if [ "$#" -gt 0 ]; then
  timeout 900 python bench.py "$@" > $OUT/bench.json 2> $OUT/bench.err
  cat $OUT/bench.json
fi
tail -25 $OUT/pytest_gpu.log
tail -2 $OUT/smoke.log
