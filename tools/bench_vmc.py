"""run_optimisation's iteration (proj/src/optimizer.cpp:73-160) entirely on one B200:
sample -> fill_amplitudes -> surrogate E_loc + moments -> energy gradient ->
SR direction -> Adam + parameter re-layout. Keys, amplitudes, local energies,
gradient and parameters stay in HBM; the host sees only the per-iteration
scalars (sample count, log-norm, moments) the reference also reads.

    python tools/bench_vmc.py [--config c118|c56] [--k 1000000] [--iterations 6] [--warmup 2] [--n-sr 100]

One JSON line: per-stage medians (CUDA events on one stream; the sampler, SR
and Adam entry points synchronise internally) and the variational energy of
every iteration (it should fall: Adam on the SR direction, lr 1e-3).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

MODEL = {"c118": (6, 110, False), "c56": (6, 14, True), "c20": (5, 10, False)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c118", choices=sorted(MODEL))
    ap.add_argument("--k", type=int, default=1_000_000)
    ap.add_argument("--iterations", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--n-sr", type=int, default=100)
    ap.add_argument("--lr", type=float, default=1e-3)
    args = ap.parse_args()

    import torch
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import _lib, synthetic
    from paper_2408_07625_b200.distributed import device_evaluate
    from bench_model import params_for

    cfg = synthetic.CONFIGS[args.config]
    n_q = cfg.n_qubits
    bits, ne, spin = MODEL[args.config]
    K = args.k
    M = q.AnqsModel(q.QuditLayout.make(n_q, bits), q.SectorConstraint(ne, spin))
    M.set_params(params_for(n_q, bits, 64))
    c, x, y, z = synthetic.jw_terms(n_q, cfg.n_terms, seed=1)
    H = q.HamiltonianIndex.from_masks(n_q, c, x, y, z)
    L = _lib.lib()
    dev = torch.device("cuda:0")
    W, P = M.W, M.n_params()
    kd = torch.empty((K, W), dtype=torch.int64, device=dev)
    lpd = torch.empty(K, dtype=torch.float64, device=dev)
    la = torch.empty(K, dtype=torch.float64, device=dev)
    ph = torch.empty_like(la)
    loc = torch.empty(K, dtype=torch.complex128, device=dev)
    mom = torch.empty(5, dtype=torch.float64, device=dev)
    grad = torch.empty(P, dtype=torch.float64, device=dev)
    dirn = torch.empty(P, dtype=torch.float64, device=dev)
    nout = C.c_int64()
    norm2 = np.zeros(2)
    lam = C.c_double()
    s = torch.cuda.Stream(dev)
    M.set_stream(s.cuda_stream)
    evaluate = device_evaluate(H, 0)
    P_ = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    names = ["sample", "fill_amplitudes", "eloc_and_moments", "energy_gradient", "sr_direction", "adam_update"]
    rec, energies = [], []
    with torch.cuda.stream(s):
        for it in range(-args.warmup, args.iterations):
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
            t0 = time.perf_counter()
            ev[0].record(s)
            _lib.check(L.qvmc_cuda_sample(M._h, K, 2024, 0x53414d50, max(it, 0), _lib.MEM_DEVICE, P_(kd), P_(lpd),
                                          C.byref(nout)))
            n = nout.value
            ev[1].record(s)
            _lib.check(L.qvmc_cuda_fill_amplitudes(M._h, n, P_(kd), P_(lpd), _lib.MEM_DEVICE, P_(la), P_(ph),
                                                   C.c_void_p(norm2.ctypes.data)))
            ev[2].record(s)
            evaluate(kd[:n], la[:n], ph[:n], lpd[:n], float(norm2[1]), 0, n, loc, mom)
            ev[3].record(s)
            wts = torch.exp(lpd[:n] - float(norm2[1]))  # variational_energy weights (energy.cpp:59-66)
            _lib.check(L.qvmc_cuda_energy_gradient(M._h, n, P_(kd), P_(wts), P_(loc), _lib.MEM_DEVICE, P_(grad)))
            ev[4].record(s)
            _lib.check(L.qvmc_cuda_sr_direction(M._h, n, P_(kd), P_(lpd), P_(loc), args.n_sr, 0.0, P_(grad),
                                                _lib.MEM_DEVICE, P_(dirn), C.byref(lam)))
            ev[5].record(s)
            _lib.check(L.qvmc_cuda_model_adam_step(M._h, P_(dirn), args.lr, 0.9, 0.999, 1e-8, _lib.MEM_DEVICE))
            ev[6].record(s)
            ev[6].synchronize()
            wall = time.perf_counter() - t0
            m = mom.cpu().numpy()
            st = [ev[i].elapsed_time(ev[i + 1]) for i in range(6)]
            print(f"iteration {it}: n {n} e_var {m[0] / m[3]:.6f} stages ms {[round(v, 2) for v in st]}",
                  file=sys.stderr, flush=True)
            if it >= 0:
                rec.append(st + [wall * 1e3])
                energies.append(float(m[0] / m[3]))
    med = np.median(np.array(rec), axis=0)
    print(json.dumps({
        "metric": f"VMC iterations/s on one B200 ({n_q} qubits, K = {K:.0e}, n_sr = {args.n_sr})",
        "value": 1e3 / float(med[-1]), "unit": "iterations/s", "ms_per_iteration": float(med[-1]),
        "samples_per_s": n / (float(med[-1]) * 1e-3),
        "stages_ms": {k: float(v) for k, v in zip(names, med[:6])},
        "e_var_per_iteration": energies, "iterations": args.iterations, "warmup": args.warmup,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {n_q} qubits, {ne} electrons, {cfg.n_terms} JW strings, ANQS "
                               f"qudits of {bits} bits hidden 64 ({P} parameters), Adam lr {args.lr}"}}))


if __name__ == "__main__":
    main()
