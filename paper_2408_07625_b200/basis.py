"""Packed basis vectors (reference: proj/include/qvmc/basis_vector.hpp).

A basis vector of N qubits is ``n_words(N) = ceil(N/64)`` uint64 words with
qubit i at word i//64, bit i%64, and all bits >= N zero
(basis_vector.hpp:16-26). A batch is a C-contiguous ``uint64[n, n_words]``
array: exactly the device layout the kernels read.
"""
from __future__ import annotations

import numpy as np

MAX_BITS = 256  # BasisVector::kMaxBits (basis_vector.hpp:29)


def n_words(n_qubits: int) -> int:
    if n_qubits < 1 or n_qubits > MAX_BITS:
        raise ValueError("BasisVector: qubit count must be in [1, 256]")
    return (n_qubits + 63) // 64


def parse(s: str) -> np.ndarray:
    """BasisVector::parse (basis_vector.cpp:8-23): qubit i = character i."""
    if not s:
        raise ValueError("BasisVector::parse: empty string")
    w = np.zeros(n_words(len(s)), dtype=np.uint64)
    for i, c in enumerate(s):
        if c == "1":
            w[i // 64] |= np.uint64(1) << np.uint64(i % 64)
        elif c != "0":
            raise ValueError(f"BasisVector::parse: illegal character '{c}'")
    return w


def parse_batch(strings) -> np.ndarray:
    rows = [parse(s) for s in strings]
    if not rows:
        raise ValueError("empty batch")
    if len({len(s) for s in strings}) != 1:
        raise ValueError("BasisVector: length mismatch")
    return np.ascontiguousarray(np.stack(rows))


def to_str(words: np.ndarray, n_qubits: int) -> str:
    """BasisVector::str (basis_vector.cpp:25-30)."""
    return "".join("1" if (int(words[i // 64]) >> (i % 64)) & 1 else "0" for i in range(n_qubits))


def dec_value(words: np.ndarray, n_qubits: int) -> int:
    """BasisVector::dec_value (basis_vector.cpp:32-38): x0 is the most significant bit."""
    if n_qubits > 64:
        raise ValueError("BasisVector::dec_value: more than 64 qubits")
    d = 0
    for i in range(n_qubits):
        if (int(words[i // 64]) >> (i % 64)) & 1:
            d |= 1 << (n_qubits - 1 - i)
    return d


def from_bool_rows(bits: np.ndarray) -> np.ndarray:
    """[n, N] 0/1 array -> [n, n_words] uint64 keys (vectorised)."""
    bits = np.asarray(bits, dtype=np.uint8)
    n, nq = bits.shape
    W = n_words(nq)
    pad = np.zeros((n, 64 * W), dtype=np.uint8)
    pad[:, :nq] = bits
    packed = np.packbits(pad, axis=1, bitorder="little")  # [n, 8W] bytes, qubit i at byte i//8 bit i%8
    return np.ascontiguousarray(packed.view("<u8").astype(np.uint64, copy=False))


def to_bool_rows(keys: np.ndarray, n_qubits: int) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    bytes_ = keys.view(np.uint8).reshape(keys.shape[0], -1)
    return np.unpackbits(bytes_, axis=1, bitorder="little")[:, :n_qubits]


def popcount(keys: np.ndarray) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    return np.unpackbits(keys.view(np.uint8).reshape(keys.shape[0], -1), axis=1).sum(axis=1)
