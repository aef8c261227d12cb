"""One VMC iteration's evaluation on one B200, chained on the device: amplitudes of
the sampled set (fill_amplitudes, sampler.cpp:104-120) then the surrogate local
energies + energy moments (optimizer.cpp:87-93), keys resident in HBM.

    python tools/bench_iteration.py [--config c118|c56] [--n-unq 1000000] [--steps 5] [--warmup 3]

Prints one JSON line: samples/s of the chained evaluation (CUDA events on one
stream, L2 flushed between steps), the two stages' share, and the unmodified
reference (oracle/_ref: fill_amplitudes with the compiled model.cpp, then
find_coupled_pairs(auto) -> local_energies -> variational_energy) on a bounded
sample with all host threads. log_probs (the sampler's output, an input here)
are 2·log|ψ| of the same model, computed before the timed region.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
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
    ap.add_argument("--n-unq", type=int, default=None)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-sample", type=int, default=10000)
    args = ap.parse_args()

    import torch
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import _lib, synthetic
    from paper_2408_07625_b200.distributed import device_evaluate
    from bench_model import params_for

    cfg = synthetic.CONFIGS[args.config]
    n_q = cfg.n_qubits
    bits, ne, spin = MODEL[args.config]
    n = args.n_unq or cfg.n_unq
    c, x, y, z = synthetic.jw_terms(n_q, cfg.n_terms, seed=1)
    H = q.HamiltonianIndex.from_masks(n_q, c, x, y, z)
    keys = synthetic.near_hf_keys(n_q, ne, n, seed=2)
    p = params_for(n_q, bits, 64)
    M = q.AnqsModel(q.QuditLayout.make(n_q, bits), q.SectorConstraint(ne, spin))
    M.set_params(p)
    la0, _ = M.log_psi(keys)
    lp_host = 2.0 * la0  # the sampler's log_probs for these samples

    dev = torch.device("cuda:0")
    s = torch.cuda.Stream(dev)
    M.set_stream(s.cuda_stream)
    evaluate = device_evaluate(H, 0)
    kd = torch.from_numpy(keys.view(np.int64)).to(dev)
    lp = torch.from_numpy(lp_host).to(dev)
    la = torch.empty(n, dtype=torch.float64, device=dev)
    ph = torch.empty_like(la)
    loc = torch.empty(n, dtype=torch.complex128, device=dev)
    mom = torch.empty(5, dtype=torch.float64, device=dev)
    norm2 = np.zeros(2)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    L = _lib.lib()

    def step(ev=None):
        _lib.check(L.qvmc_cuda_fill_amplitudes(M._h, n, C.c_void_p(kd.data_ptr()), C.c_void_p(lp.data_ptr()),
                                               _lib.MEM_DEVICE, C.c_void_p(la.data_ptr()), C.c_void_p(ph.data_ptr()),
                                               _ptr(norm2)))
        if ev is not None:
            ev.record(s)
        evaluate(kd, la, ph, lp, float(norm2[1]), 0, n, loc, mom)

    def _ptr(a):
        return C.c_void_p(a.ctypes.data)

    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        launches0 = q.launch_count()
        tot, amp = [], []
        for _ in range(args.steps):
            flush.fill_(1)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(s)
            step(e1)
            e2.record(s)
            e2.synchronize()
            tot.append(e0.elapsed_time(e2))
            amp.append(e0.elapsed_time(e1))
        launches = q.launch_count() - launches0
    ms, ms_amp = float(np.mean(tot)), float(np.mean(amp))
    m = mom.cpu().numpy()
    e_var = m[0] / m[3]

    cpu = None
    import oracle
    if oracle.ref_available():
        from bench import masks_to_strings
        threads = os.cpu_count() or 1
        k = min(args.cpu_sample, n)
        R = oracle.RefModel(n_q, bits, ne, spin, 64)
        R.set_params(p)
        RI = oracle.RefIndex.from_strings(n_q, c, masks_to_strings(n_q, x, y, z))
        t0 = time.perf_counter()
        la_r, ph_r, norm_r, log_norm_r = R.fill_amplitudes(keys[:k], lp_host[:k], threads=threads)
        t_amp = time.perf_counter() - t0
        _, out5, t3, _ = RI.run_path(keys[:k], la_r, ph_r, lp_host[:k], norm_r, log_norm_r, backend=3,
                                     threshold=4096, threads=threads, want_locals=False)
        secs = t_amp + float(t3.sum())
        cpu = {"value": k / secs, "unit": "samples/s", "cores": threads, "kind": "reference",
               "sample": f"first {k} samples as their own sample set: fill_amplitudes {t_amp:.2f} s + "
                         f"find_coupled_pairs/local_energies/variational_energy {float(t3.sum()):.2f} s"}

    print(json.dumps({
        "metric": f"VMC iteration evaluation samples/s ({n_q} qubits, {n:.0e} samples): fill_amplitudes + "
                  f"surrogate E_loc + moments",
        "value": n / (ms * 1e-3), "unit": "samples/s", "ms_per_step": ms, "steps": args.steps,
        "warmup": args.warmup, "dtype": "f64", "data": "synthetic",
        "stages_ms": {"fill_amplitudes": ms_amp, "eloc_and_moments": ms - ms_amp},
        "config": {"workload": f"{args.config}: {n_q} qubits, {ne} electrons, {cfg.n_terms} JW strings, "
                               f"ANQS qudits of {bits} bits hidden 64, near-HF samples", "l2": "flushed between steps"},
        "e_var": e_var, "gpu_launches": int(launches), "cpu_baseline": cpu}))


if __name__ == "__main__":
    main()
