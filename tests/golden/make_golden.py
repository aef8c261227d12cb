"""Regenerate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference to have built
oracle/_ref/libqvmc_ref_hot.so):

    python tests/golden/make_golden.py

Writes tests/golden/*.npz. Every array here is an output of the reference's
own code: HamiltonianIndex::parse/from_terms groupings, loop_over_{terms,
batch,trie} pair lists and ops, group_element per pair, local_energies and
variational_energy. The GPU tests and the oracle tests compare against these
files, so nothing at test time needs /root/reference.

Families (seeds and streams exactly as the reference tests draw them):
  * fixtures toy/h2/h4/h6 (proj/fixtures/*.ham) + full particle sectors
  * coupling  : proj/tests/test_coupling.cpp:138-168 (SequentialRng(seed, 1234), seeds 1..40)
  * accept3   : proj/tests/acceptance_main.cpp:131-160 (SequentialRng(seed, 0xAC3), seeds 1..200)
  * checks    : proj/src/checks.cpp:156-188 (SequentialRng(seed, 0xBAC0), seeds 1..25)
  * opscale   : proj/tests/test_coupling.cpp:170-190 (n=24, 128 vectors seed 9, H seeds 2 with 40/400 terms)
"""
from __future__ import annotations

import itertools
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent
FIXTURES = Path("/root/reference/proj/fixtures")


def index_arrays(R: "oracle.RefIndex", prefix: str) -> dict:
    return {f"{prefix}n_qubits": np.int64(R.n_qubits), f"{prefix}xy": R.xy, f"{prefix}offsets": R.offsets,
            f"{prefix}coeff": R.coeff, f"{prefix}x": R.x, f"{prefix}y": R.y, f"{prefix}z": R.z,
            f"{prefix}yz": R.yz, f"{prefix}y_weight": R.y_weight, f"{prefix}diag": np.int64(R.diag)}


def amplitudes(n: int, seed: int):
    rng = np.random.default_rng(seed)
    la = rng.normal(0.0, 0.4, n)
    ph = rng.uniform(0.0, 2 * math.pi, n)
    lp = 2.0 * la
    mx = lp.max()
    log_norm = float(mx + np.log(np.exp(lp - mx).sum()))
    return la, ph, lp, math.exp(log_norm), log_norm


def path_arrays(R, keys, prefix: str, seed: int) -> dict:
    d = {f"{prefix}keys": keys}
    for be, name in ((0, "terms"), (1, "batch"), (2, "trie")):
        e, ops, _ = R.pairs(keys, backend=be)
        d[f"{prefix}ops_{name}"] = np.uint64(ops)
        if be == 0:
            d[f"{prefix}pairs"] = e
        else:
            assert np.array_equal(e, d[f"{prefix}pairs"]), "reference backends disagree"
    e = d[f"{prefix}pairs"]
    h = np.array([R.group_element(keys[j], g) for (_, j, g) in e], dtype=np.complex128)
    d[f"{prefix}pair_h"] = h
    la, ph, lp, norm, log_norm = amplitudes(keys.shape[0], seed)
    d.update({f"{prefix}la": la, f"{prefix}ph": ph, f"{prefix}lp": lp, f"{prefix}norm": np.float64(norm),
              f"{prefix}log_norm": np.float64(log_norm)})
    loc = R.local_energies(keys, la, ph, e)
    d[f"{prefix}eloc"] = loc
    out5, w = oracle.ref_variational_energy(lp, norm, log_norm, loc)
    d[f"{prefix}evar"] = out5  # e_var, im_residual, ipr, norm, log_norm
    return d


def sector(n_qubits, n_e, spin=False):
    rows = []
    for occ in itertools.combinations(range(n_qubits), n_e):
        if spin and sum(1 for o in occ if o % 2 == 0) != n_e // 2:
            continue
        w = 0
        for o in occ:
            w |= 1 << o
        rows.append([w])
    return np.array(rows, dtype=np.uint64)


def fixtures():
    d = {}
    for name, n_e in (("toy", 2), ("h2", 2), ("h4", 4), ("h6", 6)):
        R = oracle.RefIndex.parse((FIXTURES / f"{name}.ham").read_text())
        d.update(index_arrays(R, f"{name}_"))
        keys = sector(R.n_qubits, n_e, spin=(name != "toy"))
        d.update(path_arrays(R, keys, f"{name}_sector_", seed=7))
    # the paper's toy batch {1100, 1001, 0110}, psi = (2, 1, -1) (checks.cpp:55-69)
    R = oracle.RefIndex.parse((FIXTURES / "toy.ham").read_text())
    keys = np.array([[0b0011], [0b1001], [0b0110]], dtype=np.uint64)  # qubit i = bit i
    e, ops, _ = R.pairs(keys, backend=1)
    d["toybatch_pairs"] = e
    la = np.array([math.log(2.0), 0.0, 0.0])
    ph = np.array([0.0, 0.0, math.pi])
    d["toybatch_eloc"] = R.local_energies(keys, la, ph, e)
    np.savez_compressed(OUT / "fixtures.npz", **d)
    print("fixtures.npz", len(d), "arrays")


def family(name, stream, seeds, draw):
    d = {"seeds": np.array(list(seeds), dtype=np.int64)}
    for seed in seeds:
        rng = oracle.RefRng(seed, stream)
        n, n_terms, n_unq, vec_seed = draw(rng, seed)
        R = oracle.RefIndex.random(n, n_terms, seed, min(4, n))
        keys = oracle.ref_random_vectors(n, n_unq, vec_seed)
        p = f"s{seed}_"
        d.update(index_arrays(R, p))
        d.update(path_arrays(R, keys, p, seed=seed))
    np.savez_compressed(OUT / f"{name}.npz", **d)
    print(f"{name}.npz", len(seeds), "instances")


def draw_coupling(rng, seed):
    n = 4 + rng.uniform_int(67)
    n_terms = 1 + rng.uniform_int(80)
    cap = (1 << n) if n < 12 else 4096
    n_unq = 1 + rng.uniform_int(min(cap, 256))
    return n, n_terms, n_unq, seed + 1


def draw_accept3(rng, seed):
    n = 4 + rng.uniform_int(37)
    n_terms = 1 + rng.uniform_int(120)
    cap = (1 << n) if n < 12 else 100000
    n_unq = 1 + rng.uniform_int(min(cap, 512))
    return n, n_terms, n_unq, seed + 1000


def draw_checks(rng, seed):
    n = 4 + rng.uniform_int(37)
    n_terms = 1 + rng.uniform_int(60)
    n_unq = 1 + rng.uniform_int(100)
    return n, n_terms, min(n_unq, 1 << min(n, 20)), seed


def opscale():
    d = {}
    keys = oracle.ref_random_vectors(24, 128, 9)
    for tag, nt in (("small", 40), ("large", 400)):
        R = oracle.RefIndex.random(24, nt, 2)
        d.update(index_arrays(R, f"{tag}_"))
        d.update(path_arrays(R, keys, f"{tag}_", seed=5))
    np.savez_compressed(OUT / "opscale.npz", **d)
    print("opscale.npz")


if __name__ == "__main__":
    if not oracle.ref_available():
        oracle.build(ref=True)
    fixtures()
    family("coupling", 1234, range(1, 41), draw_coupling)
    family("accept3", 0xAC3, range(1, 201), draw_accept3)
    family("checks", 0xBAC0, range(1, 26), draw_checks)
    opscale()
