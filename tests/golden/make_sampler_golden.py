"""Regenerate tests/golden/sampler.npz from the UNMODIFIED reference sampler (oracle/_ref).

    python tests/golden/make_sampler_golden.py

sample_without_replacement (proj/src/sampler.cpp:37-102) on reference
AnqsModels (hidden 64, parameters from make_model_golden.model_params with a
stored seed, or the reference's four-state model of checks.cpp:94-106), with
CounterRng(seed, stream) and an iteration index per case. Stores the sampled
keys and log-probabilities in the reference's ChildLess order. Needs
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

OUT = Path(__file__).resolve().parent / "sampler.npz"

# name: (n_qubits, bits, n_e, spin, param seed, [(K, rng seed, stream, iteration), ...])
CASES = {
    "t8": (8, 3, 3, False, 301, [(1, 31, 0, 1), (3, 31, 0, 3), (17, 62, 0, 17), (56, 93, 0, 56), (200, 124, 0, 200)]),
    "x6": (6, 3, 2, False, 302, [(100, 5, 0, 0)]),  # exhaustion: the whole C(6,2) = 15 sector
    "s12": (12, 6, 6, True, 303, [(50, 7, 1, 3), (400, 7, 1, 4)]),
    "r20": (20, 6, 10, False, 304, [(300, 9, 0, 1), (4096, 9, 0, 2)]),
    "r70": (70, 4, 20, False, 305, [(2000, 11, 2, 5)]),
    "h56": (56, 6, 14, True, 306, [(3000, 13, 0, 7)]),
    "h118": (118, 6, 110, False, 307, [(2000, 17, 0, 9)]),
    "r130": (130, 5, 64, True, 308, [(500, 19, 3, 11)]),
}


def four_state_params(n_params, probs):
    """checks.cpp:94-106: zero parameters except the amplitude b3 of the one-hot codes."""
    p = np.zeros(n_params)
    b3 = n_params // 2 - 16  # block 0 amplitude head: W1 4*64, b1 64, W2 64*64, b2 64, W3 16*64, b3 16
    for code, pr in zip((8, 4, 2, 1), probs):
        p[b3 + code] = 0.5 * np.log(pr)
    return p


def main():
    arrays = {}
    for name, (n, bits, ne, spin, pseed, runs) in CASES.items():
        R = oracle.RefModel(n, bits, ne, spin, 64)
        R.set_params(model_params((n, bits, 64), seed=pseed))
        arrays[f"{name}_cfg"] = np.array([n, bits, ne, int(spin), 64, pseed])
        arrays[f"{name}_runs"] = np.array(runs, dtype=np.int64)
        for i, (K, seed, stream, it) in enumerate(runs):
            keys, lp = R.sample(K, seed, stream, it, threads=8)
            arrays[f"{name}_{i}_keys"] = keys
            arrays[f"{name}_{i}_lp"] = lp
            print(name, K, keys.shape)
    # four-state model (checks.cpp:94-106), K = 2 over the first 64 iterations of CounterRng(4242, 1)
    probs = (0.7, 0.2, 0.08, 0.02)
    R = oracle.RefModel(4, 4, 1, False, 64)
    p = four_state_params(R.n_params, probs)
    R.set_params(p)
    keys = []
    for t in range(64):
        k, _ = R.sample(2, 4242, 1, t)
        keys.append(k[:, 0])
    # Philox/Gumbel and condition_max known answers from the compiled reference (rng.hpp, sampler.cpp:15-23)
    rng = np.random.default_rng(5)
    kat = []
    for _ in range(64):
        seed = int(rng.integers(0, 2**63))
        st, c = int(rng.integers(0, 2**32)), [int(v) for v in rng.integers(0, 2**32, 4)]
        kat.append([seed, st, *c])
    arrays["gumbel_args"] = np.array(kat, dtype=np.uint64)
    arrays["gumbel_vals"] = np.array([oracle.ref_gumbel(*[int(v) for v in r]) for r in kat])
    cm = [(-1.37, 2.5, 2.5), (0.0, 0.0, -1.0), (-700.0, 800.0, -750.0)]
    for _ in range(61):
        parent = 4.0 * (rng.uniform() - 0.5)
        a, b = parent - 8.0 * rng.uniform(), parent - 8.0 * rng.uniform()
        cm.append((parent, max(a, b), a))
    arrays["cmax_args"] = np.array(cm)
    arrays["cmax_vals"] = np.array([oracle.ref_condition_max(*r) for r in cm])
    arrays["four_probs"] = np.array(probs)
    arrays["four_first64"] = np.array(keys, dtype=np.uint64)
    np.savez_compressed(OUT, **arrays)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
