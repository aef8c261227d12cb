"""Seeded synthetic inputs for the BASELINE.json configurations.

The generators run in C++ in ``lib/libqvmc_synth.so`` (``qvmc_synth_*``,
include/qvmc_synth.h; g++ only, separate from the kernels' libqvmc_cuda.so so
that bench.py's reference arm never loads the product library) so 3e6-term
Hamiltonians and 1e6-sample sets take seconds. The reference ships no
molecule fixtures beyond toy/h2/h4/h6 and its own ``random_hamiltonian``
produces no off-diagonal couplings at these sizes, so the
throughput inputs are JW-structured Pauli strings plus near-HF determinants.
"""
from __future__ import annotations

import ctypes as C
import itertools
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .basis import from_bool_rows, n_words
from .energy import SampleBatch, normalise
from .hamiltonian import HamiltonianIndex, _ptr

SYNTH_PATH = Path(__file__).resolve().parent / "lib" / "libqvmc_synth.so"
_synth = None


def _slib() -> C.CDLL:
    global _synth
    if _synth is None:
        if not SYNTH_PATH.exists():
            raise ImportError(f"{SYNTH_PATH} is missing: run __graft_entry__.build()")
        L = C.CDLL(str(SYNTH_PATH))
        L.qvmc_synth_jw_hamiltonian.restype = C.c_int
        L.qvmc_synth_jw_hamiltonian.argtypes = [C.c_int, C.c_int64, C.c_uint64] + [C.c_void_p] * 4 + [
            C.POINTER(C.c_int64)]
        L.qvmc_synth_near_hf_samples.restype = C.c_int
        L.qvmc_synth_near_hf_samples.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_uint64, C.c_void_p]
        L.qvmc_synth_last_error.restype = C.c_char_p
        _synth = L
    return _synth


def _scheck(status: int) -> None:
    if status != 0:
        raise ValueError(_slib().qvmc_synth_last_error().decode())


@dataclass(frozen=True)
class Config:
    name: str
    n_qubits: int
    n_electrons: int
    n_terms: int
    n_unq: int


# BASELINE.json configs (see DESIGN.md for the substitutions SURVEY.md §0 forces)
CONFIGS = {
    "c56": Config("synthetic 56q (N2 cc-pVDZ-sized), 1e6 samples", 56, 14, 300_000, 1_000_000),
    "c118": Config("synthetic 118q (BeI2 STO-3G-sized), 1e6 samples", 118, 110, 3_000_000, 1_000_000),
    "c20": Config("synthetic 20q (N2 STO-3G-sized), 1e5 samples", 20, 10, 12_000, 100_000),
    # not a BASELINE config: half filling, 20 orbitals in the minority set (190 deletion buckets per row,
    # the join's tables sized per call; QVMC_JOIN=0 measures the sector candidate lists instead)
    "c40h": Config("synthetic 40q half-filled (20 e-), 1e5 samples", 40, 20, 100_000, 100_000),
}


def jw_terms(n_qubits: int, n_terms: int, seed: int = 1):
    """Raw JW-structured strings as (coeff, x, y, z) mask arrays."""
    W = n_words(n_qubits)
    coeff = np.zeros(n_terms, dtype=np.float64)
    x = np.zeros((n_terms, W), dtype=np.uint64)
    y = np.zeros((n_terms, W), dtype=np.uint64)
    z = np.zeros((n_terms, W), dtype=np.uint64)
    got = C.c_int64()
    _scheck(_slib().qvmc_synth_jw_hamiltonian(n_qubits, n_terms, seed, _ptr(coeff), _ptr(x), _ptr(y), _ptr(z),
                                              C.byref(got)))
    k = int(got.value)
    return coeff[:k], x[:k], y[:k], z[:k]


def jw_hamiltonian(n_qubits: int, n_terms: int, seed: int = 1) -> HamiltonianIndex:
    return HamiltonianIndex.from_masks(n_qubits, *jw_terms(n_qubits, n_terms, seed))


def near_hf_keys(n_qubits: int, n_electrons: int, n_unq: int, seed: int = 2) -> np.ndarray:
    keys = np.zeros((n_unq, n_words(n_qubits)), dtype=np.uint64)
    _scheck(_slib().qvmc_synth_near_hf_samples(n_qubits, n_electrons, n_unq, seed, _ptr(keys)))
    return keys


def sector_keys(n_qubits: int, n_electrons: int, spin_balanced: bool = False) -> np.ndarray:
    """Every determinant of the sector (optionally n_e/2 on even 'up' sites)."""
    rows = []
    for occ in itertools.combinations(range(n_qubits), n_electrons):
        if spin_balanced and sum(1 for o in occ if o % 2 == 0) != (n_electrons + 1) // 2:
            continue
        b = np.zeros(n_qubits, dtype=np.uint8)
        b[list(occ)] = 1
        rows.append(b)
    return from_bool_rows(np.stack(rows))


def random_sector_keys(n_qubits: int, n_electrons: int, n_unq: int, seed: int = 2) -> np.ndarray:
    """n_unq distinct uniformly random determinants with n_electrons particles."""
    if n_unq > math.comb(n_qubits, n_electrons):
        raise ValueError("requested more distinct determinants than the sector holds")
    rng = np.random.default_rng(seed)
    seen, out = set(), []
    while len(out) < n_unq:
        batch = rng.random((2 * (n_unq - len(out)) + 16, n_qubits)).argsort(axis=1)[:, :n_electrons]
        for occ in batch:
            key = tuple(sorted(occ.tolist()))
            if key in seen:
                continue
            seen.add(key)
            out.append(key)
            if len(out) == n_unq:
                break
    bits = np.zeros((n_unq, n_qubits), dtype=np.uint8)
    for i, occ in enumerate(out):
        bits[i, list(occ)] = 1
    return from_bool_rows(bits)


def amplitudes(n_unq: int, seed: int = 3, noise: float = 0.1):
    """log|psi_i| = -0.5 i/n + N(0, noise), phase in {0, pi}; log p = 2 log|psi|."""
    rng = np.random.default_rng(seed)
    la = -0.5 * np.arange(n_unq, dtype=np.float64) / max(n_unq, 1)
    if noise:
        la = la + rng.normal(0.0, noise, n_unq)
    ph = np.where(rng.random(n_unq) < 0.5, 0.0, math.pi)
    return la, ph


def sample_batch(keys: np.ndarray, seed: int = 3) -> SampleBatch:
    la, ph = amplitudes(keys.shape[0], seed)
    lp, norm, log_norm = normalise(la)
    return SampleBatch(np.ascontiguousarray(keys), lp, la, ph, norm, log_norm)


def make_config(name: str, n_unq: int = None, n_terms: int = None):
    """(HamiltonianIndex, SampleBatch) for a named BASELINE config."""
    cfg = CONFIGS[name]
    h = jw_hamiltonian(cfg.n_qubits, n_terms or cfg.n_terms, seed=1)
    if name == "c20":  # 1e5 distinct exceeds the spin-balanced sector (C(10,5)^2 = 63,504)
        keys = random_sector_keys(cfg.n_qubits, cfg.n_electrons, n_unq or cfg.n_unq, seed=2)
    else:
        keys = near_hf_keys(cfg.n_qubits, cfg.n_electrons, n_unq or cfg.n_unq, seed=2)
    return h, sample_batch(keys, seed=3)
