"""Device Gumbel top-K sampler (qvmc_cuda_sample = sample_without_replacement,
sampler.cpp:37-102) and one full VMC iteration chained on the device:
sample -> fill_amplitudes -> surrogate E_loc + moments -> energy gradient, keys
never leaving HBM (run_optimisation's steps, optimizer.cpp:80-140, minus SR/Adam).

    python tools/bench_sampler.py [--config c118|c56] [--k 1000000] [--steps 3] [--warmup 1]

One JSON line: sampler samples/s (median wall time of the call, which
synchronises once per qudit level to size the candidate sort), the chained
iteration's samples/s with its stage split (CUDA events, medians over the
timed iterations after warm-up ones), and the unmodified reference
sampler (oracle/_ref) at a bounded K on all host threads.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

MODEL = {"c118": (6, 110, False), "c56": (6, 14, True)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c118", choices=sorted(MODEL))
    ap.add_argument("--k", type=int, default=1_000_000)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--cpu-k", type=int, default=20_000)
    ap.add_argument("--cpu-grad", type=int, default=2000)
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
    p = params_for(n_q, bits, 64)
    M = q.AnqsModel(q.QuditLayout.make(n_q, bits), q.SectorConstraint(ne, spin))
    M.set_params(p)
    c, x, y, z = synthetic.jw_terms(n_q, cfg.n_terms, seed=1)
    H = q.HamiltonianIndex.from_masks(n_q, c, x, y, z)
    L = _lib.lib()
    dev = torch.device("cuda:0")
    W = M.W
    kd = torch.empty((K, W), dtype=torch.int64, device=dev)
    lpd = torch.empty(K, dtype=torch.float64, device=dev)
    la = torch.empty(K, dtype=torch.float64, device=dev)
    ph = torch.empty_like(la)
    loc = torch.empty(K, dtype=torch.complex128, device=dev)
    mom = torch.empty(5, dtype=torch.float64, device=dev)
    grad = torch.empty(M.n_params(), dtype=torch.float64, device=dev)
    nout = C.c_int64()
    norm2 = np.zeros(2)
    s = torch.cuda.Stream(dev)
    M.set_stream(s.cuda_stream)
    evaluate = device_evaluate(H, 0)

    def sample(it):
        _lib.check(L.qvmc_cuda_sample(M._h, K, 2024, 0, it, _lib.MEM_DEVICE, C.c_void_p(kd.data_ptr()),
                                      C.c_void_p(lpd.data_ptr()), C.byref(nout)))
        return nout.value

    with torch.cuda.stream(s):
        for it in range(args.warmup):
            sample(it)
        torch.cuda.synchronize()
        t_samp = []
        for it in range(args.steps):
            t0 = time.perf_counter()
            n = sample(100 + it)
            t_samp.append(time.perf_counter() - t0)
            print(f"sample call {it}: {t_samp[-1] * 1e3:.2f} ms", file=sys.stderr)
        # the chained iteration: sample -> fill_amplitudes -> E_loc + moments, one stream
        tot, parts = [], []
        launches0 = q.launch_count()
        for it in range(-args.warmup, args.steps):  # warm-up iterations first (buffer growth), then timed
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0, e1, e2, e3, e4 = (torch.cuda.Event(enable_timing=True) for _ in range(5))
            e0.record(s)
            n = sample(200 + it)
            e1.record(s)
            _lib.check(L.qvmc_cuda_fill_amplitudes(M._h, n, C.c_void_p(kd.data_ptr()), C.c_void_p(lpd.data_ptr()),
                                                   _lib.MEM_DEVICE, C.c_void_p(la.data_ptr()),
                                                   C.c_void_p(ph.data_ptr()), C.c_void_p(norm2.ctypes.data)))
            e2.record(s)
            evaluate(kd[:n], la[:n], ph[:n], lpd[:n], float(norm2[1]), 0, n, loc, mom)
            e3.record(s)
            wts = torch.exp(lpd[:n] - float(norm2[1]))  # variational_energy weights (energy.cpp:59-66)
            _lib.check(L.qvmc_cuda_energy_gradient(M._h, n, C.c_void_p(kd.data_ptr()), C.c_void_p(wts.data_ptr()),
                                                   C.c_void_p(loc.data_ptr()), _lib.MEM_DEVICE,
                                                   C.c_void_p(grad.data_ptr())))
            e4.record(s)
            e4.synchronize()
            st_ms = (e0.elapsed_time(e1), e1.elapsed_time(e2), e2.elapsed_time(e3), e3.elapsed_time(e4))
            print(f"iteration {it}: stages ms {[round(v, 2) for v in st_ms]}", file=sys.stderr)
            if it < 0:
                launches0 = q.launch_count()
                continue
            tot.append(time.perf_counter() - t0)
            parts.append(st_ms)
        launches = q.launch_count() - launches0
    st = q.last_stats(H)
    ms_s = float(np.median(t_samp)) * 1e3  # medians: a rare host stall inside one call is not the kernel's cost
    pm = np.median(np.array(parts), axis=0)
    ms_it = float(np.median(tot)) * 1e3
    m = mom.cpu().numpy()

    cpu = None
    import oracle
    if oracle.ref_available():
        threads = os.cpu_count() or 1
        R = oracle.RefModel(n_q, bits, ne, spin, 64)
        R.set_params(p)
        t0 = time.perf_counter()
        keys_r, _ = R.sample(args.cpu_k, 2024, 0, 100, threads=threads)
        secs = time.perf_counter() - t0
        kg = min(len(keys_r), args.cpu_grad)
        t0 = time.perf_counter()
        R.energy_gradient(keys_r[:kg], np.full(kg, 1.0 / kg), np.ones(kg, dtype=np.complex128) * (1 + 0.1j),
                          threads=threads)
        gsecs = time.perf_counter() - t0
        cpu = {"value": len(keys_r) / secs, "unit": "samples/s", "cores": threads, "kind": "reference",
               "sample": f"sample_without_replacement with K = {args.cpu_k} ({secs:.2f} s)",
               "energy_gradient": {"value": kg / gsecs, "unit": "samples/s",
                                   "sample": f"energy_gradient over batched_grad_log_psi of {kg} samples "
                                             f"({gsecs:.2f} s)"}}
    print(json.dumps({
        "metric": f"device sampler samples/s ({n_q} qubits, K = {K:.0e})", "value": n / (ms_s * 1e-3),
        "unit": "samples/s", "ms_per_call": ms_s, "n_sampled": n, "steps": args.steps, "dtype": "f64",
        "config": {"workload": f"{args.config}: {n_q} qubits, {ne} electrons, qudits of {bits} bits, hidden 64, "
                               f"seeded random parameters; E_loc over {cfg.n_terms} JW strings"},
        "iteration": {"value": n / (ms_it * 1e-3), "unit": "samples/s", "ms": ms_it,
                      "stages_ms": {"sample": float(pm[0]), "fill_amplitudes": float(pm[1]),
                                    "eloc_and_moments": float(pm[2]), "energy_gradient": float(pm[3])},
                      "pairs_per_sample": st["pairs"] / max(n, 1), "e_var": float(m[0] / m[3]),
                      "gpu_launches": int(launches)},
        "cpu_baseline": cpu}))


if __name__ == "__main__":
    main()
