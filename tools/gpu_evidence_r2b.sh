#!/bin/bash
# Round-2 evidence on the current tree: GPU tests, smoke, bench lines (ours + reference arm), configs 2 and 5,
# amplitude model, sampler / VMC iteration, launch list.
TAG=${1:-r2fin}; OUT=gpurun_out/$TAG; mkdir -p $OUT
make -s -C paper_2408_07625_b200/csrc > $OUT/make.log 2>&1 || { echo 'build failed'; tail $OUT/make.log; exit 1; }  # never measure a stale .so
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
tail -n 2 $OUT/pytest_gpu.log $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c118.json 2> $OUT/bench_c118.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_c118.json 2> $OUT/bench_ref_c118.err
timeout 600 python bench.py --config c56 > $OUT/bench_c56.json 2> $OUT/bench_c56.err
timeout 600 python bench.py --config c20 > $OUT/bench_c20.json 2> $OUT/bench_c20.err
timeout 600 python bench.py --config c40h > $OUT/bench_c40h.json 2> $OUT/bench_c40h.err
for n in 1000 10000 100000 1000000 10000000; do
  timeout 900 python bench.py --config c56 --n-unq $n --steps 5 --warmup 3 --e2e-steps 2 > $OUT/sweep_c56_$n.json 2> $OUT/sweep_c56_$n.err
done
for cfg in c118 c56; do
  timeout 300 python tools/bench_model.py --config $cfg > $OUT/bench_model_$cfg.json 2> $OUT/bench_model_$cfg.err
  timeout 900 python tools/bench_vmc.py --config $cfg --iterations 6 > $OUT/bench_vmc_$cfg.json 2> $OUT/bench_vmc_$cfg.err
done
for f in $OUT/bench_c118.json $OUT/bench_ref_c118.json $OUT/bench_c56.json $OUT/bench_c20.json $OUT/bench_c40h.json $OUT/sweep_*.json; do
  python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d.get("roofline", {})
    print(sys.argv[1].split("/")[-1], f"value {d['value']:.4g} step {d['ms_per_step']:.3f} e2e {d['e2e']['value']:.4g} frac {r.get('frac', 0):.3f} {r.get('bound', '')} cpu {(d.get('cpu_baseline') or {}).get('value', 0):.4g}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
