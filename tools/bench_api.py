"""Time the reference-shaped API path (what the C++ drop-in runs inside run_optimisation):
find_coupled_pairs -> local_energies -> variational_energy, host arrays in and out.

usage: python tools/bench_api.py [--config c118] [--n-unq N] [--steps K]
"""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c118")
    ap.add_argument("--n-unq", type=int, default=None)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import synthetic
    H, b = synthetic.config_inputs(args.config, n_unq=args.n_unq) if hasattr(synthetic, "config_inputs") else (None, None)
    cfg = synthetic.CONFIGS[args.config]
    if H is None:
        H = synthetic.jw_hamiltonian(cfg.n_qubits, cfg.n_terms, seed=1)
        keys = synthetic.near_hf_keys(cfg.n_qubits, cfg.n_electrons, args.n_unq or cfg.n_unq, seed=2)
        b = synthetic.sample_batch(keys, seed=3)
    q.surrogate_energy(H, b)  # warm-up: device handle + workspaces
    t = {"find_coupled_pairs": [], "local_energies": [], "variational_energy": [], "fused": []}
    for _ in range(args.steps):
        t0 = time.perf_counter()
        pairs = q.find_coupled_pairs(b.vectors, H)
        t1 = time.perf_counter()
        loc = q.local_energies(pairs, b, H)
        t2 = time.perf_counter()
        q.variational_energy(b, loc, index=H)
        t3 = time.perf_counter()
        q.surrogate_energy(H, b)
        t4 = time.perf_counter()
        for k, v in zip(t, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
            t[k].append(v)
    n = b.size()
    out = {k: statistics.median(v) for k, v in t.items()}
    api = out["find_coupled_pairs"] + out["local_energies"] + out["variational_energy"]
    print(json.dumps({"config": args.config, "n_unq": n, "pairs": int(len(pairs.entries)),
                      "seconds": out, "api_samples_per_s": n / api, "fused_samples_per_s": n / out["fused"]}))


if __name__ == "__main__":
    main()
