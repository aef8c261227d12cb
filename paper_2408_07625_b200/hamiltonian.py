"""HamiltonianIndex: Pauli-string Hamiltonian grouped by flip mask.

Mirrors proj/include/qvmc/hamiltonian.hpp:41-107. The grouping itself
(merge duplicate strings, drop |c| < 1e-12, group by xy = x|y in
first-occurrence order; hamiltonian.cpp:63-117) runs in C++ inside
libqvmc_cuda (``qvmc_index_build``); this module parses text and encodes
strings into the (x, y, z) masks that function takes. The device copy used
by the kernels is created lazily per CUDA device (``device_handle``).
"""
from __future__ import annotations

import ctypes as C
import math
import re
from typing import Iterable, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .basis import n_words as _n_words

_LETTERS = np.frombuffer(b"IXYZ", dtype=np.uint8)


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data) if a.size else C.c_void_p(0)


def encode_strings(n_qubits: int, strings: Sequence[str]) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """encode_term (hamiltonian.cpp:38-61) for many strings: -> x, y, z masks [n, W]."""
    W = _n_words(n_qubits)
    n = len(strings)
    if n == 0:
        z = np.zeros((0, W), dtype=np.uint64)
        return z, z.copy(), z.copy()
    for s in strings:
        if len(s) != n_qubits:
            raise ValueError(f"HamiltonianIndex: pauli string length {len(s)} != qubits {n_qubits}")
    raw = np.frombuffer("".join(strings).encode("ascii", errors="replace"), dtype=np.uint8).reshape(n, n_qubits)
    bad = ~np.isin(raw, _LETTERS)
    if bad.any():
        r, c = np.argwhere(bad)[0]
        raise ValueError(f"encode_term: illegal Pauli character '{strings[r][c]}'")
    out = []
    for letter in b"XYZ":
        bits = np.zeros((n, 64 * W), dtype=np.uint8)
        bits[:, :n_qubits] = raw == letter
        out.append(np.ascontiguousarray(np.packbits(bits, axis=1, bitorder="little").view("<u8").astype(np.uint64)))
    return out[0], out[1], out[2]


class HamiltonianIndex:
    """Immutable grouped Hamiltonian (hamiltonian.hpp:41-107)."""

    def __init__(self, handle: C.c_void_p, n_qubits: int):
        L = _lib.lib()
        self._handle = handle
        self._n_qubits = n_qubits
        self._W = _n_words(n_qubits)
        nq, nt, nxy, dg = C.c_int(), C.c_uint64(), C.c_uint32(), C.c_int64()
        _lib.check(L.qvmc_index_info(handle, C.byref(nq), C.byref(nt), C.byref(nxy), C.byref(dg)))
        self._n_terms, self._n_xy, self._diag = int(nt.value), int(nxy.value), int(dg.value)
        W, T, G = self._W, self._n_terms, self._n_xy
        self.xy = np.zeros((G, W), dtype=np.uint64)
        self.group_offsets = np.zeros(G + 1, dtype=np.uint64)
        self.coeff = np.zeros(T, dtype=np.float64)
        self.yz = np.zeros((T, W), dtype=np.uint64)
        self.y_weight = np.zeros(T, dtype=np.uint8)
        self.x_masks = np.zeros((T, W), dtype=np.uint64)
        self.y_masks = np.zeros((T, W), dtype=np.uint64)
        self.z_masks = np.zeros((T, W), dtype=np.uint64)
        _lib.check(L.qvmc_index_export(handle, _ptr(self.xy), _ptr(self.group_offsets), _ptr(self.coeff),
                                       _ptr(self.yz), _ptr(self.y_weight), _ptr(self.x_masks),
                                       _ptr(self.y_masks), _ptr(self.z_masks)))
        self._xy_lookup = {self.xy[g].tobytes(): g for g in range(G)}
        self._device = {}

    def plan_summary(self) -> dict:
        """The device-layout plan of this index, computed on the host
        (``qvmc_index_plan_summary``): join drain-record kinds, bitmap bits."""
        out = _lib.QvmcPlanSummary()
        _lib.check(_lib.lib().qvmc_index_plan_summary(self._handle, C.byref(out)))
        return {k: int(getattr(out, k)) for k, _ in _lib.QvmcPlanSummary._fields_}

    # ------------------------------------------------------------ builders
    @staticmethod
    def from_masks(n_qubits: int, coeff, x, y, z) -> "HamiltonianIndex":
        W = _n_words(n_qubits)
        coeff = np.ascontiguousarray(coeff, dtype=np.float64)
        x, y, z = (np.ascontiguousarray(a, dtype=np.uint64).reshape(-1, W) for a in (x, y, z))
        if not (len(coeff) == len(x) == len(y) == len(z)):
            raise ValueError("HamiltonianIndex: mask/coefficient length mismatch")
        h = C.c_void_p()
        _lib.check(_lib.lib().qvmc_index_build(n_qubits, W, len(coeff), _ptr(coeff), _ptr(x), _ptr(y), _ptr(z),
                                               C.byref(h)))
        return HamiltonianIndex(h, n_qubits)

    @staticmethod
    def from_terms(n_qubits: int, terms: Iterable[Tuple[float, str]]) -> "HamiltonianIndex":
        """HamiltonianIndex::from_terms (hamiltonian.cpp:63-117)."""
        if n_qubits < 1 or n_qubits > 256:
            raise ValueError("HamiltonianIndex: qubit count out of range")
        terms = list(terms)
        coeff = np.array([float(c) for c, _ in terms], dtype=np.float64)
        x, y, z = encode_strings(n_qubits, [s for _, s in terms])
        return HamiltonianIndex.from_masks(n_qubits, coeff, x, y, z)

    @staticmethod
    def parse(text) -> "HamiltonianIndex":
        """HamiltonianIndex::parse (hamiltonian.cpp:119-170): errors carry line numbers."""
        if not isinstance(text, str):
            text = text.read()
        n_qubits = -1
        coeffs, strings = [], []
        for line_no, line in enumerate(text.splitlines(), start=1):
            def fail(msg):
                raise RuntimeError(f"hamiltonian line {line_no}: {msg}")
            body = line.split("#", 1)[0].strip(" \t\r")
            if not body:
                continue
            tok = body.split()
            if n_qubits < 0:
                m = re.match(r"[+-]?\d+", tok[1]) if len(tok) >= 2 else None
                n = int(m.group(0)) if m else -1
                if tok[0] != "qubits:" or m is None or n < 1 or n > 256:
                    fail("expected header 'qubits: <N>'")
                n_qubits = n
                continue
            if len(tok) < 2:
                fail("expected '<coeff> <pauli_string>'")
            if len(tok) > 2:
                fail(f"trailing content '{tok[2]}'")
            cs, paulis = tok
            try:
                c = float(cs)
            except ValueError:
                try:  # strtod also accepts hexadecimal floating constants
                    if not re.fullmatch(r"[+-]?0[xX][0-9a-fA-F.]+([pP][+-]?\d+)?", cs):
                        raise ValueError(cs)
                    c = float.fromhex(cs)
                except ValueError:
                    fail(f"cannot parse coefficient '{cs}' as a real number")
            if not math.isfinite(c):
                fail("non-finite coefficient")
            if len(paulis) != n_qubits:
                fail(f"pauli string has length {len(paulis)}, expected {n_qubits}")
            for ch in paulis:
                if ch not in "IXYZ":
                    fail(f"illegal Pauli character '{ch}'")
            coeffs.append(c)
            strings.append(paulis)
        if n_qubits < 0:
            raise RuntimeError("hamiltonian: missing 'qubits:' header")
        return HamiltonianIndex.from_terms(n_qubits, zip(coeffs, strings))

    @staticmethod
    def load(path: str) -> "HamiltonianIndex":
        try:
            with open(path) as f:
                text = f.read()
        except OSError:
            raise RuntimeError(f"cannot open hamiltonian file: {path}") from None
        return HamiltonianIndex.parse(text)

    # ------------------------------------------------------------ accessors
    @property
    def n_qubits(self) -> int:
        return self._n_qubits

    @property
    def n_words(self) -> int:
        return self._W

    @property
    def n_terms(self) -> int:
        return self._n_terms

    @property
    def n_xy(self) -> int:
        return self._n_xy

    def xy_set(self) -> np.ndarray:
        return self.xy

    def group(self, g: int) -> range:
        return range(int(self.group_offsets[g]), int(self.group_offsets[g + 1]))

    def find_xy(self, mask: np.ndarray) -> Optional[int]:
        return self._xy_lookup.get(np.ascontiguousarray(mask, dtype=np.uint64).tobytes())

    def diagonal_xy_index(self) -> Optional[int]:
        return None if self._diag < 0 else self._diag

    # ------------------------------------------------------------ device side
    def device_handle(self, device: int = 0) -> C.c_void_p:
        """The device-resident copy on CUDA ordinal ``device`` (created once)."""
        h = self._device.get(device)
        if h is None:
            h = C.c_void_p()
            _lib.check(_lib.lib().qvmc_cuda_ham_create_from_index(self._handle, device, C.byref(h)))
            self._device[device] = h
        return h

    def matrix_element(self, x: np.ndarray, x_prime: np.ndarray, device: int = 0) -> complex:
        """<x|H|x'> (hamiltonian.cpp:178-184), evaluated by the device kernel."""
        x = np.ascontiguousarray(x, dtype=np.uint64)
        xp = np.ascontiguousarray(x_prime, dtype=np.uint64)
        g = self.find_xy(x ^ xp)
        if g is None:
            return 0j
        return self.group_element(xp, g, device)

    def group_element(self, x_prime: np.ndarray, xy_index: int, device: int = 0) -> complex:
        keys = np.ascontiguousarray(np.asarray(x_prime, dtype=np.uint64).reshape(1, self._W))
        entries = np.array([[0, 0, xy_index]], dtype=np.uint32)
        out = np.zeros(2, dtype=np.float64)
        _lib.check(_lib.lib().qvmc_cuda_pair_elements(self.device_handle(device), 1, _ptr(keys), 1, _ptr(entries),
                                                      _ptr(out), None, _lib.MEM_HOST))
        return complex(out[0], out[1])

    def close(self) -> None:
        L = _lib.lib()
        for h in self._device.values():
            L.qvmc_cuda_ham_destroy(h)
        self._device.clear()
        if self._handle:
            L.qvmc_index_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
