"""Amplitude-evaluation benchmark: AnqsModel::log_psi over a
batch of unique samples on one B200, beside the reference CPU path.

    python tools/bench_model.py [--config c118|c56] [--n-unq 1000000] [--steps 10] [--warmup 3]

Prints one JSON line: samples/s with keys resident in HBM (CUDA events around
k_log_psi on the model's stream), the end-to-end rate through the C ABI with
host buffers, the fp64 FLOP rate against a DGEMM measured in the same run
(torch.matmul float64 8192^3, cuBLAS) and the unmodified reference
(oracle/_ref: model.cpp log_psi, all host threads) on a bounded sample.
Parameters: seeded uniform(±1/sqrt(fan_in)) like init_params (model.cpp:105-127).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CONFIGS = {"c118": (118, 6, 110, False), "c56": (56, 6, 14, True)}


def params_for(n, bits, hidden, seed=7):
    rng = np.random.default_rng(seed)
    out = []
    for o in range(0, n, bits):
        k = min(bits, n - o)
        for hd in range(2):
            s1, s2 = 1 / np.sqrt(n), 1 / np.sqrt(hidden)
            bs = 0.0 if hd == 0 else 0.1
            out += [rng.uniform(-s1, s1, hidden * n), rng.uniform(-bs * s1, bs * s1, hidden) if bs else np.zeros(hidden),
                    rng.uniform(-s2, s2, hidden * hidden), rng.uniform(-bs * s2, bs * s2, hidden) if bs else np.zeros(hidden),
                    rng.uniform(-s2, s2, (1 << k) * hidden), rng.uniform(-bs * s2, bs * s2, 1 << k) if bs else np.zeros(1 << k)]
    return np.concatenate(out)


def flops_per_sample(n, bits, keys, hidden=64):
    """(executed, reference-equivalent) fp64 flops per sample: the device's sparse layer 1
    (one add per hidden unit per prefix-minority orbital), 64x64 layer-2 GEMM rows for both
    heads, the 2^k-output amplitude layer 3 and the phase head's single output; the reference
    evaluates every layer densely (model.cpp:160-175)."""
    from paper_2408_07625_b200 import basis
    bits_rows = basis.to_bool_rows(keys[:2000], n)
    ex = ref = 0.0
    for o in range(0, n, bits):
        k = min(bits, n - o)
        ones = bits_rows[:, :o].sum(1)
        m = np.minimum(ones, o - ones).mean()
        ex += 2 * (hidden * m + 2 * hidden * hidden) + 2 * hidden * (1 << k) + 2 * hidden
        ref += 2 * 2 * (hidden * n + hidden * hidden + hidden * (1 << k))
    return ex, ref


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c118", choices=sorted(CONFIGS))
    ap.add_argument("--n-unq", type=int, default=1_000_000)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-sample", type=int, default=4000)
    args = ap.parse_args()

    import torch
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import synthetic

    n, bits, ne, spin = CONFIGS[args.config]
    keys = synthetic.near_hf_keys(n, ne, args.n_unq, seed=2)
    p = params_for(n, bits, 64)
    M = q.AnqsModel(q.QuditLayout.make(n, bits), q.SectorConstraint(ne, spin))
    M.set_params(p)
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream(dev)  # a real stream handle (0 would select the model's own stream)
    M.set_stream(stream.cuda_stream)
    kd = torch.from_numpy(keys.view(np.int64)).to(dev)
    la = torch.empty(args.n_unq, dtype=torch.float64, device=dev)
    ph = torch.empty_like(la)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    run = lambda: M.log_psi_device(kd.data_ptr(), args.n_unq, la.data_ptr(), ph.data_ptr())  # noqa: E731
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    launches0 = q.launch_count()
    ts = []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    launches = q.launch_count() - launches0
    ms = float(np.mean(ts))

    # end to end through the C ABI with host buffers (keys in, log|psi| and phase out)
    pin_k = torch.from_numpy(keys.view(np.int64)).pin_memory().numpy().view(np.uint64)
    M.set_stream(None)
    M.log_psi(pin_k)
    t0 = time.perf_counter()
    for _ in range(3):
        M.log_psi(pin_k)
    e2e_s = (time.perf_counter() - t0) / 3

    # fp64 peak measured in this run: cuBLAS DGEMM 8192^3
    a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    b = torch.randn_like(a)
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    dgemm_tf = 2 * 8192 ** 3 / (best * 1e-3) / 1e12

    ex, ref_eq = flops_per_sample(n, bits, keys)
    achieved = ex * args.n_unq / (ms * 1e-3) / 1e12

    # parity spot check against the restatement
    import oracle
    from oracle.model_oracle import ModelOracle
    O = ModelOracle(n, bits, ne, spin, 64, p)
    rows = np.arange(0, args.n_unq, max(1, args.n_unq // 200))
    lo, po = O.log_psi(keys[rows])
    lg, pg = la.cpu().numpy()[rows], ph.cpu().numpy()[rows]
    max_dev = float(max(np.abs(lg - lo).max(), np.abs(pg - po).max()))

    cpu = None
    if oracle.ref_available():
        R = oracle.RefModel(n, bits, ne, spin, 64)
        R.set_params(p)
        threads = os.cpu_count() or 1
        sample = keys[:args.cpu_sample]
        t0 = time.perf_counter()
        lr, pr = R.log_psi(sample, threads=threads)
        dt = time.perf_counter() - t0
        max_dev = max(max_dev, float(np.abs(la.cpu().numpy()[:args.cpu_sample] - lr).max()))
        cpu = {"value": args.cpu_sample / dt, "unit": "samples/s", "cores": threads, "kind": "reference",
               "sample": f"first {args.cpu_sample} samples, model.cpp log_psi via parallel_for; {dt:.2f} s"}

    print(json.dumps({
        "metric": f"AnqsModel log_psi samples/s ({n} qubits, {args.n_unq:.0e} samples)",
        "value": args.n_unq / (ms * 1e-3), "unit": "samples/s", "ms_per_step": ms, "steps": args.steps,
        "warmup": args.warmup, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {n} qubits, {ne} electrons, qudits of {bits} bits, hidden 64, "
                               f"near-HF samples (seed 2), seeded parameters", "l2": "flushed between steps"},
        "e2e": {"value": args.n_unq / e2e_s, "unit": "samples/s", "h2d_bytes_per_step": int(keys.nbytes),
                "d2h_bytes_per_step": 16 * args.n_unq, "path": "qvmc_cuda_log_psi(QVMC_MEM_HOST)"},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": dgemm_tf, "unit": "TFLOP/s",
                     "frac": achieved / dgemm_tf, "peak_source": "cuBLAS DGEMM 8192^3 measured in this run",
                     "flops_per_sample_executed": ex, "flops_per_sample_reference_dense": ref_eq},
        "gpu_launches": int(launches), "max_abs_dev_vs_oracle_and_reference": max_dev, "cpu_baseline": cpu}))


if __name__ == "__main__":
    main()
