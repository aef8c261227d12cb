"""Coupled-pair search (reference: proj/include/qvmc/coupling.hpp).

All backends return the identical canonical pair list (by x, then x'),
computed by the device kernel through ``qvmc_cuda_pairs``; the backend only
selects the ``ops`` semantics the reference reports (coupling.hpp:22-26):
terms = n_unq*|XY| (coupling.cpp:75), batch = n_unq^2 (coupling.cpp:93),
trie = candidates the device actually probed (bounded like the reference's
trie visit count, test_coupling.cpp:189, :202).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from .hamiltonian import HamiltonianIndex, _ptr


class CouplingBackend(enum.IntEnum):
    kTerms = _lib.BACKEND_TERMS
    kBatch = _lib.BACKEND_BATCH
    kTrie = _lib.BACKEND_TRIE
    kAuto = _lib.BACKEND_AUTO


_NAMES = {"terms": CouplingBackend.kTerms, "batch": CouplingBackend.kBatch, "trie": CouplingBackend.kTrie,
          "auto": CouplingBackend.kAuto}


def parse_backend(name: str) -> CouplingBackend:
    """coupling.cpp:17-23."""
    try:
        return _NAMES[name]
    except KeyError:
        raise ValueError(f"unknown coupling backend: {name}") from None


def backend_name(b: CouplingBackend) -> str:
    return {v: k for k, v in _NAMES.items()}[CouplingBackend(b)]


@dataclass
class CoupledPairs:
    """CoupledPairs (coupling.hpp:29-38): entries[:, 0] = x, [:, 1] = x', [:, 2] = xy."""
    entries: np.ndarray
    ops: int
    backend: CouplingBackend


@dataclass
class CouplingOptions:
    backend: CouplingBackend = CouplingBackend.kAuto
    auto_batch_threshold: int = 4096
    threads: int = 1  # accepted for interface parity; the device ignores it


def _as_keys(batch, index: HamiltonianIndex) -> np.ndarray:
    keys = np.ascontiguousarray(batch, dtype=np.uint64)
    if keys.ndim == 1:
        keys = keys.reshape(-1, index.n_words)
    if keys.shape[1:] != (index.n_words,):
        raise ValueError("BasisVector: length mismatch")
    return keys


def _pairs(batch, index: HamiltonianIndex, backend: int, threshold: int = 4096, device: int = 0) -> CoupledPairs:
    keys = _as_keys(batch, index)
    L = _lib.lib()
    h = index.device_handle(device)
    n_pairs, ops, used = C.c_uint64(), C.c_uint64(), C.c_int()
    _lib.check(L.qvmc_cuda_pairs(h, keys.shape[0], _ptr(keys), _lib.MEM_HOST, int(backend), int(threshold),
                                 C.byref(n_pairs), C.byref(ops), C.byref(used)))
    entries = np.zeros((int(n_pairs.value), 3), dtype=np.uint32)
    if entries.size:
        _lib.check(L.qvmc_cuda_pairs_fetch(h, _ptr(entries), _lib.MEM_HOST))
    return CoupledPairs(entries, int(ops.value), CouplingBackend(used.value))


def loop_over_terms(batch, index: HamiltonianIndex, threads: int = 1) -> CoupledPairs:
    return _pairs(batch, index, CouplingBackend.kTerms)


def loop_over_batch(batch, index: HamiltonianIndex, threads: int = 1) -> CoupledPairs:
    return _pairs(batch, index, CouplingBackend.kBatch)


def loop_over_trie(batch, index: HamiltonianIndex, threads: int = 1) -> CoupledPairs:
    return _pairs(batch, index, CouplingBackend.kTrie)


def find_coupled_pairs(batch, index: HamiltonianIndex, options: CouplingOptions = CouplingOptions()) -> CoupledPairs:
    """coupling.cpp:153-169: auto = batch below the threshold, trie above."""
    return _pairs(batch, index, options.backend, options.auto_batch_threshold)
