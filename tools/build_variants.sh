#!/bin/bash
# Build tuning variants of libqvmc_cuda.so into paper_2408_07625_b200/lib/variants/
# (bench with QVMC_CUDA_LIB=<variant> to compare). Usage: tools/build_variants.sh name:"-DFLAG=.." ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2408_07625_b200/csrc
OUT=$ROOT/paper_2408_07625_b200/lib/variants
mkdir -p "$OUT"
for spec in "$@"; do
  name=${spec%%:*}
  flags=${spec#*:}
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++20 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
    -I"$ROOT/include" -I"$SRC" --expt-relaxed-constexpr $flags -shared -o "$OUT/libqvmc_cuda_$name.so" \
    "$SRC/qvmc_cuda.cu" "$SRC/host_index.cpp" -lcudart -lcublas -lcusolver -ldl -Xptxas -v 2>&1 |
    grep -A2 "properties for _ZN9qvmc_b20011k_rows_joinILi2ELi0" | tail -1 | sed "s/^/$name: /" &
done
wait
