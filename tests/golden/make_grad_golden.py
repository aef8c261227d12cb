"""Regenerate tests/golden/grad.npz from the UNMODIFIED reference (oracle/_ref).

    python tests/golden/make_grad_golden.py

Per configuration: AnqsModel parameters from make_model_golden.model_params
(stored seed), seeded in-sector keys, weights and local energies; the
reference's energy_gradient (proj/src/energy.cpp:93-107) over its
batched_grad_log_psi rows (proj/src/model.cpp:273-336), and sampled columns
of those Jacobian rows. Small models store the whole gradient; the 56/118
qubit ones a fixed sample of its entries plus its norm. Needs
/root/reference at generation time only.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

import oracle  # noqa: E402
from make_model_golden import model_params  # noqa: E402
from paper_2408_07625_b200 import synthetic  # noqa: E402

OUT = Path(__file__).resolve().parent / "grad.npz"

# name: (n_qubits, bits, n_e, spin, param seed, keys kind, count, full gradient stored)
CASES = {
    "s8": (8, 3, 3, False, 401, "random", 40, True),
    "s12": (12, 6, 6, True, 402, "sector", 0, True),
    "r20": (20, 6, 10, False, 403, "random", 300, True),
    "h56": (56, 6, 14, True, 404, "near_hf", 200, False),
    "h118": (118, 6, 110, False, 405, "near_hf", 100, False),
}


def main():
    arrays = {}
    for name, (n, bits, ne, spin, pseed, kind, count, full) in CASES.items():
        R = oracle.RefModel(n, bits, ne, spin, 64)
        R.set_params(model_params((n, bits, 64), seed=pseed))
        if kind == "sector":
            keys = synthetic.sector_keys(n, ne, spin_balanced=spin)
        elif kind == "near_hf":
            keys = synthetic.near_hf_keys(n, ne, count, seed=pseed)
        else:
            keys = synthetic.random_sector_keys(n, ne, count, seed=pseed)
        rng = np.random.default_rng(pseed)
        w = rng.uniform(0.1, 1.0, len(keys))
        w /= w.sum()
        loc = rng.normal(size=len(keys)) - 3.0 + 0.2j * rng.normal(size=len(keys))
        g = R.energy_gradient(keys, w, loc, threads=8)
        J = R.grad_log_psi(keys[:8], threads=8)
        cols = np.sort(rng.choice(R.n_params, 2048, replace=False))
        arrays[f"{name}_cfg"] = np.array([n, bits, ne, int(spin), 64, pseed])
        arrays[f"{name}_keys"] = keys
        arrays[f"{name}_w"] = w
        arrays[f"{name}_loc"] = loc
        arrays[f"{name}_jcols"] = cols
        arrays[f"{name}_jac"] = J[:, cols]
        arrays[f"{name}_jnorm"] = np.linalg.norm(J, axis=1)
        arrays[f"{name}_gnorm"] = np.array([np.linalg.norm(g)])
        if full:
            arrays[f"{name}_grad"] = g
        else:
            arrays[f"{name}_gcols"] = cols
            arrays[f"{name}_grad_at"] = g[cols]
        print(name, keys.shape, R.n_params, np.linalg.norm(g))
    np.savez_compressed(OUT, **arrays)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
