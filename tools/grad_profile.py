"""One energy_gradient call at a BASELINE layout (for ncu launch lists)."""
import sys, ctypes as C
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
import numpy as np, torch
import paper_2408_07625_b200 as q
from paper_2408_07625_b200 import _lib, synthetic
from bench_model import params_for
cfg = sys.argv[1] if len(sys.argv) > 1 else "c118"
n_q, bits, ne, spin = {"c118": (118, 6, 110, False), "c56": (56, 6, 14, True)}[cfg]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
M = q.AnqsModel(q.QuditLayout.make(n_q, bits), q.SectorConstraint(ne, spin)); M.set_params(params_for(n_q, bits, 64))
keys = synthetic.near_hf_keys(n_q, ne, N, seed=2)
w = np.full(N, 1.0 / N); loc = np.random.default_rng(0).normal(size=N) + 0j
kd = torch.from_numpy(keys.view(np.int64)).cuda(); wd = torch.from_numpy(w).cuda(); ld = torch.from_numpy(loc).cuda()
g = torch.empty(M.n_params(), dtype=torch.float64, device='cuda')
L = _lib.lib()
for it in range(3):
    if it == 2: torch.cuda.profiler.start()
    _lib.check(L.qvmc_cuda_energy_gradient(M._h, N, C.c_void_p(kd.data_ptr()), C.c_void_p(wd.data_ptr()), C.c_void_p(ld.data_ptr()), _lib.MEM_DEVICE, C.c_void_p(g.data_ptr())))
torch.cuda.profiler.stop()
print("done")
