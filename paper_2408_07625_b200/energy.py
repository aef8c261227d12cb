"""Local energies and the variational energy (reference: proj/include/qvmc/energy.hpp).

``local_energies`` / ``variational_energy`` keep the reference signatures
(energy.hpp:23-24, :39) and run on the device through the C ABI.
``surrogate_energy`` is the throughput path: the fused kernel computes the
surrogate E_loc of every sampled x without materialising the pair list, and
the energy moments, in one call.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .coupling import CoupledPairs
from .hamiltonian import HamiltonianIndex, _ptr


@dataclass
class SampleBatch:
    """SampleBatch (sampler.hpp:37-46): distinct vectors + per-vector log p, log|psi|, phase."""
    vectors: np.ndarray                      # uint64 [n, n_words]
    log_probs: np.ndarray                    # float64 [n]
    log_amps: np.ndarray                     # float64 [n]
    phases: np.ndarray                       # float64 [n]
    norm: float = 0.0
    log_norm: float = 0.0

    def size(self) -> int:
        return int(self.vectors.shape[0])


@dataclass
class EnergyReport:
    """EnergyReport (energy.hpp:27-35), plus the weighted variance of E_loc."""
    e_var: float = 0.0
    im_residual: float = 0.0
    locals: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.complex128))
    weights: np.ndarray = field(default_factory=lambda: np.zeros(0))
    norm: float = 0.0
    log_norm: float = 0.0
    ipr: float = 0.0
    sum_weights: float = 0.0
    variance: float = 0.0   # sum_x w_x |E_loc(x) - E|^2 with E = sum_x w_x E_loc(x)


def _f64(a, n: int, name: str) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.shape != (n,):
        raise ValueError(f"{name}: expected {n} values, got shape {a.shape}")
    return a


def local_energies(pairs: CoupledPairs, batch: SampleBatch, index: HamiltonianIndex, threads: int = 1,
                   device: int = 0) -> np.ndarray:
    """energy.cpp:13-48: E_loc(x) = sum over the run of x of H_{xx'} psi(x')/psi(x)."""
    n = batch.size()
    keys = np.ascontiguousarray(batch.vectors, dtype=np.uint64).reshape(n, index.n_words)
    la = _f64(batch.log_amps, n, "log_amps")
    ph = _f64(batch.phases, n, "phases")
    entries = np.ascontiguousarray(pairs.entries, dtype=np.uint32).reshape(-1, 3)
    out = np.zeros(n, dtype=np.complex128)
    _lib.check(_lib.lib().qvmc_cuda_local_energies(index.device_handle(device), n, _ptr(keys), _ptr(la), _ptr(ph),
                                                   entries.shape[0], _ptr(entries), _ptr(out), _lib.MEM_HOST))
    return out


def _report_from_moments(m: np.ndarray, norm: float, log_norm: float, locals_: np.ndarray,
                         weights: np.ndarray) -> EnergyReport:
    r = EnergyReport(locals=locals_, weights=weights, norm=norm, log_norm=log_norm)
    r.e_var, r.im_residual, r.ipr, r.sum_weights = float(m[0]), float(m[1]), float(m[2]), float(m[3])
    # sum w|E - E0|^2 = sum w|E|^2 - 2 Re(conj(E0) sum w E) + |E0|^2 sum w, E0 = sum w E
    e0 = complex(m[0], m[1])
    r.variance = float(m[4] - 2.0 * (e0.conjugate() * e0).real + abs(e0) ** 2 * m[3])
    return r


def _check_residual(r: EnergyReport) -> None:
    """energy.cpp:74-76."""
    if abs(r.im_residual) > 1e-6 * max(1.0, abs(r.e_var)):
        raise RuntimeError(f"variational_energy: imaginary residual {r.im_residual:f}")


def variational_energy(batch: SampleBatch, locals_: np.ndarray, device: int = 0,
                       index: Optional[HamiltonianIndex] = None) -> EnergyReport:
    """energy.cpp:50-78: E = Re sum_x w_x E_loc(x), w = p/N; moments reduced on the device."""
    n = batch.size()
    locals_ = np.ascontiguousarray(locals_, dtype=np.complex128)
    if locals_.shape != (n,):
        raise ValueError("variational_energy: locals/batch size mismatch")
    if not (batch.norm > 0.0):
        raise RuntimeError("variational_energy: sampled norm is zero")
    lp = _f64(batch.log_probs, n, "log_probs")
    m = np.zeros(5, dtype=np.float64)
    w = np.zeros(n, dtype=np.float64)
    h = _moments_handle(index, device)
    _lib.check(_lib.lib().qvmc_cuda_energy_moments(h, n, _ptr(lp), float(batch.log_norm), _ptr(locals_), _ptr(m),
                                                   _ptr(w), _lib.MEM_HOST))
    r = _report_from_moments(m, batch.norm, batch.log_norm, locals_, w)
    _check_residual(r)
    return r


_scratch_index = {}


def _moments_handle(index: Optional[HamiltonianIndex], device: int):
    # the moment reduction needs a handle only for its stream and workspace
    if index is not None:
        return index.device_handle(device)
    if device not in _scratch_index:
        _scratch_index[device] = HamiltonianIndex.from_terms(1, [(1.0, "I")])
    return _scratch_index[device].device_handle(device)


def surrogate_energy(index: HamiltonianIndex, batch: SampleBatch, row_begin: int = 0, row_end: Optional[int] = None,
                     want_locals: bool = True, device: int = 0, check: bool = True) -> EnergyReport:
    """find_coupled_pairs + local_energies + variational_energy fused on the device
    for rows [row_begin, row_end) against the whole sample set (optimizer.cpp:87-93)."""
    n = batch.size()
    row_end = n if row_end is None else row_end
    if check and not (batch.norm > 0.0):
        raise RuntimeError("variational_energy: sampled norm is zero")
    keys = np.ascontiguousarray(batch.vectors, dtype=np.uint64).reshape(n, index.n_words)
    la = _f64(batch.log_amps, n, "log_amps")
    ph = _f64(batch.phases, n, "phases")
    lp = _f64(batch.log_probs, n, "log_probs")
    rows = row_end - row_begin
    out = np.zeros(max(rows, 0), dtype=np.complex128)
    m = np.zeros(5, dtype=np.float64)
    _lib.check(_lib.lib().qvmc_cuda_eloc_fused(index.device_handle(device), n, _ptr(keys), _ptr(la), _ptr(ph),
                                               _ptr(lp), float(batch.log_norm), row_begin, row_end,
                                               _ptr(out) if want_locals else None, _ptr(m), _lib.MEM_HOST))
    r = _report_from_moments(m, batch.norm, batch.log_norm, out, np.zeros(0))
    if check and row_begin == 0 and row_end == n:
        _check_residual(r)
    return r


def last_stats(index: HamiltonianIndex, device: int = 0) -> dict:
    st = _lib.QvmcStats()
    _lib.check(_lib.lib().qvmc_cuda_last_stats(index.device_handle(device), C.byref(st)))
    return {k: (float if k.endswith("_ms") else int)(getattr(st, k)) for k, _ in _lib.QvmcStats._fields_
            if not k.startswith("reserved")}


def normalise(log_amps: np.ndarray) -> tuple:
    """log_probs = 2 log|psi|, norm = sum p, log_norm = log norm (as fill_amplitudes, sampler.cpp:104-120)."""
    lp = 2.0 * np.asarray(log_amps, dtype=np.float64)
    mx = lp.max()
    log_norm = float(mx + math.log(np.exp(lp - mx).sum()))
    return lp, math.exp(log_norm), log_norm
