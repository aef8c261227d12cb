"""Regenerate tests/golden/model.npz from the UNMODIFIED reference AnqsModel (oracle/_ref).

    python tests/golden/make_model_golden.py

For each configuration: parameters drawn with numpy (seeded, so only the seed
is stored) are set on the reference model (model.cpp:99-103), and the
reference's log_psi (model.cpp:262-271) and fill_amplitudes
(sampler.cpp:104-120) outputs are stored with the keys. One configuration
also stores the reference's own init_params (model.cpp:105-127) draw. Needs
/root/reference at generation time only.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2408_07625_b200 import synthetic  # noqa: E402

OUT = Path(__file__).resolve().parent / "model.npz"

# name: (n_qubits, bits_per_qudit, n_electrons, spin_constraint, keys kind, count)
CONFIGS = {
    "s8": (8, 3, 4, True, "sector", 0),
    "s12": (12, 6, 6, True, "sector", 0),
    "r20": (20, 6, 10, False, "random", 500),
    "h56": (56, 6, 14, True, "near_hf", 300),
    "r70": (70, 4, 20, False, "random", 200),
    "h118": (118, 6, 110, False, "near_hf", 300),
    "r130": (130, 5, 64, True, "random_spin", 100),
}


def model_params(n_params_layout, seed):
    """Seeded parameters in the reference's flat layout (model.cpp:65-80)."""
    n, bits, hidden = n_params_layout
    rng = np.random.default_rng(seed)
    out = []
    for o in range(0, n, bits):
        k = min(bits, n - o)
        for _ in range(2):
            s1, s2 = 1 / np.sqrt(n), 1 / np.sqrt(hidden)
            out += [rng.uniform(-s1, s1, hidden * n), rng.uniform(-0.1 * s1, 0.1 * s1, hidden),
                    rng.uniform(-s2, s2, hidden * hidden), rng.uniform(-0.1 * s2, 0.1 * s2, hidden),
                    rng.uniform(-s2, s2, (1 << k) * hidden), rng.uniform(-0.1 * s2, 0.1 * s2, 1 << k)]
    return np.concatenate(out)


def make_keys(n, ne, spin, kind, count, seed):
    if kind == "sector":
        keys = synthetic.sector_keys(n, ne, spin_balanced=spin)
    elif kind == "near_hf":
        keys = synthetic.near_hf_keys(n, ne, count, seed=seed)
    elif kind == "random":
        keys = synthetic.random_sector_keys(n, ne, count, seed=seed)
    else:  # random spin-balanced: ne/2 on even and ne/2 on odd orbitals
        rng = np.random.default_rng(seed)
        bits = np.zeros((count, n), dtype=bool)
        ev, od = np.arange(0, n, 2), np.arange(1, n, 2)
        for r in range(count):
            bits[r, rng.choice(ev, ne // 2, replace=False)] = True
            bits[r, rng.choice(od, ne // 2, replace=False)] = True
        from paper_2408_07625_b200 import basis
        keys = basis.from_bool_rows(bits)
    # plus out-of-sector keys (masked: log_psi = (-inf, 0), model.cpp:263)
    W = keys.shape[1]
    bad = keys[:3].copy()
    bad[:, 0] ^= np.uint64(1)
    return np.concatenate([keys, bad]).reshape(-1, W)


def main():
    arrays = {}
    for i, (name, (n, bits, ne, spin, kind, count)) in enumerate(CONFIGS.items()):
        R = oracle.RefModel(n, bits, ne, spin, 64)
        p = model_params((n, bits, 64), seed=100 + i)
        assert p.size == R.n_params
        R.set_params(p)
        keys = make_keys(n, ne, spin, kind, count, seed=200 + i)
        la, ph = R.log_psi(keys, threads=8)
        lp = 2.0 * np.where(np.isfinite(la), la, -50.0)
        la2, ph2, norm, log_norm = R.fill_amplitudes(keys, lp, threads=8)
        assert np.array_equal(la, la2) and np.array_equal(ph, ph2)
        arrays.update({f"{name}_cfg": np.array([n, bits, ne, int(spin), 64, 100 + i]), f"{name}_keys": keys,
                       f"{name}_la": la, f"{name}_ph": ph, f"{name}_lp": lp,
                       f"{name}_norm": np.array([norm, log_norm])})
        print(name, keys.shape, R.n_params)
    # the reference's own init_params draw (SequentialRng(seed, "INIT"), model.cpp:105-127)
    R = oracle.RefModel(12, 6, 6, True, 64)
    R.init_params(42)
    keys = synthetic.sector_keys(12, 6, spin_balanced=True)
    la, ph = R.log_psi(keys)
    arrays.update({"init_cfg": np.array([12, 6, 6, 1, 64, 42]), "init_keys": keys, "init_la": la, "init_ph": ph,
                   "init_params_head": R.params[:64], "init_params_sum": np.array([R.params.sum()])})
    np.savez_compressed(OUT, **arrays)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
