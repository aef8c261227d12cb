for v in main g12 g8; do
  lib=paper_2408_07625_b200/lib/libqvmc_cuda.so
  [ "$v" != main ] && lib=paper_2408_07625_b200/lib/variants/libqvmc_cuda_$v.so
  for cfg in c118 c56; do
    echo "$v $cfg $(QVMC_CUDA_LIB=$lib timeout 600 python tools/bench_vmc.py --config $cfg --iterations 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["stages_ms"]["energy_gradient"],2), round(d["ms_per_iteration"],1))')"
  done
done
