import sys, time, ctypes as C, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
import numpy as np, torch
import paper_2408_07625_b200 as q
from paper_2408_07625_b200 import _lib
from bench_model import params_for
M = q.AnqsModel(q.QuditLayout.make(118, 6), q.SectorConstraint(110, False)); M.set_params(params_for(118, 6, 64))
K = 1_000_000
kd = torch.empty((K, 2), dtype=torch.int64, device='cuda'); lp = torch.empty(K, dtype=torch.float64, device='cuda')
n = C.c_int64()
for it in [100, 200, 200, 200, 101]:
    t0 = time.perf_counter()
    _lib.check(_lib.lib().qvmc_cuda_sample(M._h, K, 2024, 0, it, _lib.MEM_DEVICE, C.c_void_p(kd.data_ptr()), C.c_void_p(lp.data_ptr()), C.byref(n)))
    print(f"=== iteration {it}: {1e3*(time.perf_counter()-t0):.1f} ms", file=sys.stderr, flush=True)
