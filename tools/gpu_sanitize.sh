#!/bin/bash
# compute-sanitizer over tools/sanitize_driver.py (every device path, small sizes).
# usage: gpurun --timeout 3000 -- 'bash tools/gpu_sanitize.sh TAG'
TAG=${1:-san}
OUT=gpurun_out/$TAG
make -s -C paper_2408_07625_b200/csrc > /dev/null 2>&1 || { echo build failed; exit 1; }
mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_driver.py > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/sanitize_$tool.log
  tail -4 $OUT/sanitize_$tool.log
done
