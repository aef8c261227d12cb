"""The amplitude model on the device (reference: proj/include/qvmc/model.hpp, proj/src/model.cpp).

Mirrors the reference interface for the stage that feeds the local-energy
path: ``QuditLayout`` (model.hpp:21-30), ``SectorConstraint``
(model.hpp:32-37), ``AnqsModel`` (model.hpp:47-148: ``n_params``, ``params``,
``set_params``, ``log_psi``, ``in_sector``), the text checkpoint
(``save_checkpoint`` model.cpp:345-357 / ``load_checkpoint`` model.cpp:359-396)
and ``fill_amplitudes`` (sampler.cpp:104-120). ``log_psi`` / ``fill_amplitudes``
run in ``k_log_psi`` (csrc/qvmc_model.cuh) through the C ABI; there is no CPU
path. Errors follow the reference: ``std::invalid_argument`` -> ValueError.
"""
from __future__ import annotations

import re

import ctypes as C
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import _lib
from .hamiltonian import _ptr


@dataclass
class QuditLayout:
    """QuditLayout::make (model.cpp:33-45)."""
    n_qubits: int = 0
    bits_per_qudit: int = 6
    sizes: List[int] = field(default_factory=list)
    offsets: List[int] = field(default_factory=list)

    @staticmethod
    def make(n_qubits: int, bits_per_qudit: int = 6) -> "QuditLayout":
        if not 1 <= n_qubits <= 256:
            raise ValueError("QuditLayout: qubit count out of range")
        if not 1 <= bits_per_qudit <= 8:
            raise ValueError("QuditLayout: bits_per_qudit must be in [1, 8]")
        offs = list(range(0, n_qubits, bits_per_qudit))
        return QuditLayout(n_qubits, bits_per_qudit, [min(bits_per_qudit, n_qubits - o) for o in offs], offs)

    def count(self) -> int:
        return len(self.sizes)


@dataclass
class SectorConstraint:
    """SectorConstraint (model.hpp:32-37)."""
    n_electrons: int = 0
    spin_constraint: bool = False


class AnqsModel:
    """Device-resident AnqsModel: parameters in the reference's flat layout (model.cpp:65-80)."""

    def __init__(self, layout: QuditLayout, sector: SectorConstraint, hidden: int = 64, device: int = 0):
        self.layout, self.sector, self.hidden, self.device = layout, sector, hidden, device
        self.W = (layout.n_qubits + 63) // 64
        h = C.c_void_p()
        _lib.check(_lib.lib().qvmc_cuda_model_create(layout.n_qubits, layout.bits_per_qudit, sector.n_electrons,
                                                     int(sector.spin_constraint), hidden, device, C.byref(h)))
        self._h = h
        n = C.c_int64()
        _lib.check(_lib.lib().qvmc_cuda_model_n_params(h, C.byref(n)))
        self._n_params = int(n.value)
        self._params = np.zeros(self._n_params)
        _lib.check(_lib.lib().qvmc_cuda_model_set_params(h, self._n_params, _ptr(self._params)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.lib().qvmc_cuda_model_destroy(h)
            self._h = None

    def n_params(self) -> int:
        return self._n_params

    @property
    def params(self) -> np.ndarray:
        return self._params.copy()

    def set_params(self, p) -> None:
        """AnqsModel::set_params (model.cpp:99-103)."""
        p = np.ascontiguousarray(p, dtype=np.float64)
        if p.shape != (self._n_params,):
            raise ValueError("AnqsModel::set_params: size mismatch")
        _lib.check(_lib.lib().qvmc_cuda_model_set_params(self._h, p.size, _ptr(p)))
        self._params = p.copy()

    def set_stream(self, stream) -> None:
        """Run on a torch/CUDA stream (an int handle or None for the model's own)."""
        _lib.check(_lib.lib().qvmc_cuda_model_set_stream(self._h, C.c_void_p(stream or 0)))

    def in_sector(self, keys: np.ndarray) -> np.ndarray:
        """AnqsModel::in_sector (model.cpp:254-259), vectorised (host arithmetic on the keys)."""
        keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1, self.W)
        pop = np.zeros(keys.shape[0], dtype=np.int64)
        up = np.zeros(keys.shape[0], dtype=np.int64)
        for w in range(self.W):
            pop += np.bitwise_count(keys[:, w]).astype(np.int64)
            up += np.bitwise_count(keys[:, w] & np.uint64(0x5555555555555555)).astype(np.int64)
        ok = pop == self.sector.n_electrons
        if self.sector.spin_constraint:
            ok &= up == self.sector.n_electrons // 2
        return ok

    def log_psi(self, keys: np.ndarray):
        """AnqsModel::log_psi (model.cpp:262-271) for every key: (log|psi|, phase) arrays."""
        keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1, self.W)
        n = keys.shape[0]
        la, ph = np.empty(n), np.empty(n)
        _lib.check(_lib.lib().qvmc_cuda_log_psi(self._h, n, _ptr(keys), _lib.MEM_HOST, _ptr(la), _ptr(ph)))
        return la, ph

    def log_psi_device(self, keys_ptr: int, n: int, out_log_amp_ptr: int, out_phase_ptr: int) -> None:
        """Device pointers (e.g. torch tensors' data_ptr()), enqueued on the model's stream."""
        _lib.check(_lib.lib().qvmc_cuda_log_psi(self._h, n, C.c_void_p(keys_ptr), _lib.MEM_DEVICE,
                                                C.c_void_p(out_log_amp_ptr), C.c_void_p(out_phase_ptr)))

    def synchronize(self) -> None:
        _lib.check(_lib.lib().qvmc_cuda_model_synchronize(self._h))

    def adam_step(self, direction, learning_rate: float = 1e-3, beta1: float = 0.9, beta2: float = 0.999,
                  epsilon: float = 1e-8) -> None:
        """adam_step (optimizer.cpp:17-31) + set_params (optimizer.cpp:157) on the device, with the
        model's own Adam state; the host copy of the parameters is refreshed from the device."""
        d = np.ascontiguousarray(direction, dtype=np.float64)
        if d.shape != (self.n_params(),):
            raise ValueError("adam_step: size mismatch")
        _lib.check(_lib.lib().qvmc_cuda_model_adam_step(self._h, _ptr(d), learning_rate, beta1, beta2, epsilon,
                                                        _lib.MEM_HOST))
        out = np.zeros(self.n_params())
        _lib.check(_lib.lib().qvmc_cuda_model_get_params(self._h, _lib.MEM_HOST, _ptr(out)))
        self._params = out

    def sr_direction(self, keys: np.ndarray, log_probs, locals_, n_sr: int, grad, lam: float = 0.0):
        """The SR step of run_optimisation (optimizer.cpp:105-143) on the device: top_probability_indices,
        grad_log_psi rows, build_sr_context and sr_direction (sr.cpp:15-95). Returns (direction, lambda)."""
        keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1, self.W)
        lp = np.ascontiguousarray(log_probs, dtype=np.float64)
        loc = np.ascontiguousarray(locals_, dtype=np.complex128)
        g = np.ascontiguousarray(grad, dtype=np.float64)
        out = np.zeros(self.n_params())
        lam_out = C.c_double()
        _lib.check(_lib.lib().qvmc_cuda_sr_direction(self._h, keys.shape[0], _ptr(keys), _ptr(lp), _ptr(loc), n_sr,
                                                     lam, _ptr(g), _lib.MEM_HOST, _ptr(out), C.byref(lam_out)))
        return out, lam_out.value

    def sr_solve(self, stacked, lam: float, grad) -> np.ndarray:
        """sr_direction (sr.cpp:74-95) for a given stacked matrix [2 n_sr][cols] and lambda > 0."""
        S = np.ascontiguousarray(stacked, dtype=np.float64)
        g = np.ascontiguousarray(grad, dtype=np.float64)
        out = np.zeros(S.shape[1])
        _lib.check(_lib.lib().qvmc_cuda_sr_solve(self._h, S.shape[0], S.shape[1], _ptr(S), lam, _ptr(g),
                                                 _lib.MEM_HOST, _ptr(out)))
        return out

    def energy_gradient(self, keys: np.ndarray, weights, locals_) -> np.ndarray:
        """energy_gradient (energy.cpp:93-107) over batched_grad_log_psi rows (model.cpp:273-336) of
        ``keys``, contracted on the device (the Jacobian is never formed): [n_params], reference layout."""
        keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1, self.W)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        loc = np.ascontiguousarray(locals_, dtype=np.complex128)
        n = keys.shape[0]
        if w.shape != (n,) or loc.shape != (n,):
            raise ValueError("energy_gradient: misaligned inputs")
        g = np.zeros(self.n_params())
        _lib.check(_lib.lib().qvmc_cuda_energy_gradient(self._h, n, _ptr(keys), _ptr(w), _ptr(loc), _lib.MEM_HOST,
                                                        _ptr(g)))
        return g

    def save_checkpoint(self, seed: int) -> str:
        """Text checkpoint, format of AnqsModel::save_checkpoint (model.cpp:345-357)."""
        lines = ["qvmc-checkpoint v1", f"n_qubits {self.layout.n_qubits}",
                 f"bits_per_qudit {self.layout.bits_per_qudit}", f"hidden {self.hidden}",
                 f"n_electrons {self.sector.n_electrons}", f"spin_constraint {int(self.sector.spin_constraint)}",
                 f"seed {seed}", f"n_params {self._n_params}"]
        lines += [_hexfloat(float(v)) for v in self._params]
        return "\n".join(lines) + "\n"


def _hexfloat(v: float) -> str:
    """std::hexfloat spelling of a double (e.g. 0x1.8p+1), as the reference writes it."""
    if v == 0.0:
        return "-0x0p+0" if np.signbit(v) else "0x0p+0"
    h = float.hex(v)  # '0x1.8000000000000p+1'
    sign = "-" if h.startswith("-") else ""
    mant, exp = h.lstrip("-")[2:].split("p")
    mant = mant.rstrip("0").rstrip(".")
    return f"{sign}0x{mant}p{exp if exp.startswith('-') else exp}"


_HEX = re.compile(r"[+-]?0[xX]")


def _parse_double(tok: str) -> float:
    """strtod semantics (model.cpp:385-393 reads parameters with >>): hexfloat
    only with a 0x prefix, decimal otherwise; malformed -> RuntimeError."""
    try:
        return float.fromhex(tok) if _HEX.match(tok) else float(tok)
    except ValueError:
        raise RuntimeError(f"checkpoint: malformed parameter '{tok}'") from None


def load_checkpoint(text: str, device: int = 0):
    """load_checkpoint (model.cpp:359-396): (AnqsModel, seed); RuntimeError on malformed input."""
    toks = text.split()
    if not text.startswith("qvmc-checkpoint v1"):
        raise RuntimeError("checkpoint: bad magic line")
    it = iter(toks[2:])

    def kv(key):
        try:
            k, v = next(it), next(it)
        except StopIteration:
            raise RuntimeError(f"checkpoint: expected key '{key}'") from None
        if k != key:
            raise RuntimeError(f"checkpoint: expected key '{key}'")
        return int(v)

    n_qubits, bits, hidden = kv("n_qubits"), kv("bits_per_qudit"), kv("hidden")
    n_e, spin, seed, n_params = kv("n_electrons"), kv("spin_constraint") != 0, kv("seed"), kv("n_params")
    model = AnqsModel(QuditLayout.make(n_qubits, bits), SectorConstraint(n_e, spin), hidden, device)
    if model.n_params() != n_params:
        raise RuntimeError("checkpoint: parameter count mismatch")
    vals = []
    for _ in range(n_params):
        try:
            vals.append(_parse_double(next(it)))
        except StopIteration:
            raise RuntimeError("checkpoint: truncated parameters") from None
    model.set_params(np.array(vals))
    return model, seed


def fill_amplitudes(batch, model: AnqsModel, threads: int = 1) -> None:
    """fill_amplitudes (sampler.cpp:104-120): log_amps, phases, norm, log_norm of a SampleBatch, on the device."""
    keys = np.ascontiguousarray(batch.vectors, dtype=np.uint64).reshape(-1, model.W)
    lp = np.ascontiguousarray(batch.log_probs, dtype=np.float64)
    n = keys.shape[0]
    if lp.shape != (n,):
        raise ValueError("fill_amplitudes: log_probs size mismatch")
    la, ph, out2 = np.empty(n), np.empty(n), np.zeros(2)
    _lib.check(_lib.lib().qvmc_cuda_fill_amplitudes(model._h, n, _ptr(keys), _ptr(lp), _lib.MEM_HOST,
                                                    _ptr(la), _ptr(ph), _ptr(out2)))
    batch.log_amps, batch.phases = la, ph
    batch.norm, batch.log_norm = float(out2[0]), float(out2[1])


@dataclass(frozen=True)
class CounterRng:
    """CounterRng (rng.hpp:30-63): the keyed Philox4x32-10 stream the sampler draws from."""
    seed: int
    stream: int = 0


def sample_without_replacement(model: AnqsModel, k_samples: int, rng: CounterRng, iteration: int,
                               threads: int = 1, device_out: bool = False):
    """sample_without_replacement (sampler.cpp:37-102) on the device: a SampleBatch of
    min(K, sector size) distinct keys and their log-probabilities in the reference's order
    (log_amps / phases unfilled, as the reference leaves them for fill_amplitudes).
    ``threads`` is accepted for signature parity and ignored."""
    from .energy import SampleBatch
    if k_samples < 1:
        raise ValueError("sample_without_replacement: K must be >= 1")
    keys = np.zeros((k_samples, model.W), dtype=np.uint64)
    lp = np.zeros(k_samples)
    n = C.c_int64()
    _lib.check(_lib.lib().qvmc_cuda_sample(model._h, k_samples, rng.seed, rng.stream, iteration, _lib.MEM_HOST,
                                           _ptr(keys), _ptr(lp), C.byref(n)))
    return SampleBatch(keys[: n.value], lp[: n.value], np.zeros(0), np.zeros(0))
