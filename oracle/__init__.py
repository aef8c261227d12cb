"""CPU oracle for the surrogate local-energy path — TEST INFRASTRUCTURE ONLY.

Two libraries, both loaded through ctypes:

* ``_build/libqvmc_oracle.so`` — ``qvmc_oracle.c``, a plain-C restatement of
  the reference hot path (each function cites the reference file:line it
  follows). Always buildable (``make -C oracle oracle``).
* ``_ref/libqvmc_ref_hot.so`` — the UNMODIFIED reference sources
  (/root/reference/proj/src/{basis_vector,rng,hamiltonian,prefix_tree,
  coupling,energy,synthetic}.cpp) compiled in place with ``ref_capi.cpp`` and
  the Eigen shim (``make -C oracle ref``). Pins the restatement and serves as
  the CPU baseline ("kind": "reference") in bench.py.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this package. The product
(``paper_2408_07625_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libqvmc_oracle.so"
REF_SO = HERE / "_ref" / "libqvmc_ref_hot.so"

_P, _I64, _U64, _INT, _D = C.c_void_p, C.c_int64, C.c_uint64, C.c_int, C.c_double


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else None


def build(ref: bool = True) -> None:
    import subprocess
    subprocess.run(["make", "-s", "-C", str(HERE), "oracle"], check=True)
    if ref and Path(os.environ.get("REF_DIR", "/root/reference/proj")).exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


# ------------------------------------------------------------------ C oracle
_olib = None


def olib():
    global _olib
    if _olib is None:
        if not ORACLE_SO.exists():
            build(ref=False)
        L = C.CDLL(str(ORACLE_SO))
        L.qo_index_from_terms.restype = _P
        L.qo_index_from_terms.argtypes = [_INT, _INT, _I64, _P, _P, _P, _P]
        L.qo_index_free.argtypes = [_P]
        L.qo_index_info.argtypes = [_P, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64)]
        L.qo_index_export.argtypes = [_P, _P, _P, _P, _P, _P]
        L.qo_last_error.restype = C.c_char_p
        L.qo_group_element.argtypes = [_P, _P, _I64, _P]
        L.qo_matrix_element.argtypes = [_P, _P, _P, _P]
        L.qo_pairs.restype = _I64
        L.qo_pairs.argtypes = [_P, _I64, _P, _INT, C.POINTER(_P), C.POINTER(_U64)]
        L.qo_free.argtypes = [_P]
        L.qo_local_energies.argtypes = [_P, _I64, _P, _P, _P, _I64, _P, _P]
        L.qo_variational_energy.argtypes = [_I64, _P, _D, _D, _P, _P, _P]
        L.qo_eloc_rows.restype = _I64
        L.qo_eloc_rows.argtypes = [_P, _I64, _P, _P, _P, _I64, _I64, _INT, _P, _P]
        L.qo_rows_list.restype = _I64
        L.qo_rows_list.argtypes = [_P, _I64, _P, _P, _P, _I64, _P, _INT, C.POINTER(_P), _P, _P, _P]
        _olib = L
    return _olib


class OracleIndex:
    """from_terms restatement over (coeff, x, y, z) masks."""

    def __init__(self, n_qubits, coeff, x, y, z):
        W = (n_qubits + 63) // 64
        self.n_qubits, self.W = n_qubits, W
        coeff = np.ascontiguousarray(coeff, dtype=np.float64)
        x, y, z = (np.ascontiguousarray(a, dtype=np.uint64).reshape(-1, W) for a in (x, y, z))
        self._h = olib().qo_index_from_terms(n_qubits, W, len(coeff), _ptr(coeff), _ptr(x), _ptr(y), _ptr(z))
        if not self._h:
            raise ValueError(olib().qo_last_error().decode())
        nt, nxy, dg = _I64(), _I64(), _I64()
        olib().qo_index_info(self._h, C.byref(nt), C.byref(nxy), C.byref(dg))
        self.n_terms, self.n_xy, self.diag = nt.value, nxy.value, dg.value
        self.xy = np.zeros((self.n_xy, W), dtype=np.uint64)
        self.offsets = np.zeros(self.n_xy + 1, dtype=np.int64)
        self.coeff = np.zeros(self.n_terms)
        self.yz = np.zeros((self.n_terms, W), dtype=np.uint64)
        self.y_weight = np.zeros(self.n_terms, dtype=np.uint8)
        olib().qo_index_export(self._h, _ptr(self.xy), _ptr(self.offsets), _ptr(self.coeff), _ptr(self.yz),
                               _ptr(self.y_weight))

    def __del__(self):
        if getattr(self, "_h", None):
            olib().qo_index_free(self._h)

    def group_element(self, xp, g):
        out = np.zeros(2)
        olib().qo_group_element(self._h, _ptr(np.ascontiguousarray(xp, dtype=np.uint64)), g, _ptr(out))
        return complex(out[0], out[1])

    def matrix_element(self, x, xp):
        out = np.zeros(2)
        olib().qo_matrix_element(self._h, _ptr(np.ascontiguousarray(x, dtype=np.uint64)),
                                 _ptr(np.ascontiguousarray(xp, dtype=np.uint64)), _ptr(out))
        return complex(out[0], out[1])

    def pairs(self, keys, backend=0):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        p = _P()
        ops = _U64()
        n = olib().qo_pairs(self._h, keys.shape[0], _ptr(keys), backend, C.byref(p), C.byref(ops))
        if n < 0:
            raise ValueError(olib().qo_last_error().decode())
        arr = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint32)), shape=(max(n, 1) * 3,))[: n * 3].copy()
        olib().qo_free(p)
        return arr.reshape(n, 3), ops.value

    def local_energies(self, keys, la, ph, entries):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        entries = np.ascontiguousarray(entries, dtype=np.uint32).reshape(-1, 3)
        la, ph = (np.ascontiguousarray(a, dtype=np.float64) for a in (la, ph))
        out = np.zeros(keys.shape[0], dtype=np.complex128)
        st = olib().qo_local_energies(self._h, keys.shape[0], _ptr(keys), _ptr(la), _ptr(ph), entries.shape[0],
                                      _ptr(entries), _ptr(out))
        if st:
            raise RuntimeError(olib().qo_last_error().decode())
        return out

    def eloc_rows(self, keys, la, ph, r0, r1, threads=None, with_scale=False):
        """E_loc of rows [r0, r1) against all of keys -> (eloc, pairs visited[, abs-sum scale])."""
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        la, ph = (np.ascontiguousarray(a, dtype=np.float64) for a in (la, ph))
        out = np.zeros(r1 - r0, dtype=np.complex128)
        scale = np.zeros(r1 - r0) if with_scale else None
        threads = threads or os.cpu_count() or 1
        n = olib().qo_eloc_rows(self._h, keys.shape[0], _ptr(keys), _ptr(la), _ptr(ph), r0, r1, threads, _ptr(out),
                                _ptr(scale))
        if n < 0:
            raise RuntimeError(olib().qo_last_error().decode())
        return (out, n, scale) if with_scale else (out, n)

    def rows_list(self, keys, rows, la=None, ph=None, threads=None):
        """Listed rows against all of keys (terms semantics): -> (pairs [P, 3] canonical,
        rows in list order; per-row pair counts; E_loc or None; abs-sum scale or None)."""
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        k = len(rows)
        counts = np.zeros(k, dtype=np.int64)
        out = scale = None
        if la is not None:
            la, ph = (np.ascontiguousarray(a, dtype=np.float64) for a in (la, ph))
            out = np.zeros(k, dtype=np.complex128)
            scale = np.zeros(k)
        p = _P()
        threads = threads or os.cpu_count() or 1
        n = olib().qo_rows_list(self._h, keys.shape[0], _ptr(keys), _ptr(la) if la is not None else None,
                                _ptr(ph) if la is not None else None, k, _ptr(rows), threads, C.byref(p),
                                _ptr(counts), _ptr(out) if out is not None else None,
                                _ptr(scale) if scale is not None else None)
        if n < 0:
            if p.value:
                olib().qo_free(p)
            raise RuntimeError(olib().qo_last_error().decode())
        arr = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint32)), shape=(max(n, 1) * 3,))[: n * 3].copy()
        olib().qo_free(p)
        return arr.reshape(n, 3), counts, out, scale


def variational_energy(log_probs, norm, log_norm, eloc):
    """-> (status, e_var, im_residual, ipr, sum_w, sum_w|E|^2, weights)."""
    lp = np.ascontiguousarray(log_probs, dtype=np.float64)
    e = np.ascontiguousarray(eloc, dtype=np.complex128)
    out = np.zeros(5)
    w = np.zeros(len(lp))
    st = olib().qo_variational_energy(len(lp), _ptr(lp), norm, log_norm, _ptr(e), _ptr(out), _ptr(w))
    return st, out, w


# ------------------------------------------------------------- reference .so
_rlib = None


def ref_available() -> bool:
    return REF_SO.exists()


def rlib():
    global _rlib
    if _rlib is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        L = C.CDLL(str(REF_SO))
        L.qref_last_error.restype = C.c_char_p
        L.qref_index_parse.argtypes = [C.c_char_p, C.POINTER(_P)]
        L.qref_index_from_strings.argtypes = [_INT, _I64, _P, C.c_char_p, C.POINTER(_P)]
        L.qref_random_hamiltonian.argtypes = [_INT, _INT, _U64, _INT, C.POINTER(_P)]
        L.qref_index_free.argtypes = [_P]
        L.qref_index_info.argtypes = [_P, C.POINTER(_INT), C.POINTER(_U64), C.POINTER(C.c_uint32), C.POINTER(_I64)]
        L.qref_index_export.argtypes = [_P, _INT, _P, _P, _P, _P, _P, _P, _P, _P]
        L.qref_matrix_element.argtypes = [_P, _INT, _P, _P, _P]
        L.qref_group_element.argtypes = [_P, _INT, _P, C.c_uint32, _P]
        L.qref_random_distinct_vectors.argtypes = [_INT, _INT, _U64, _INT, _P]
        L.qref_pairs.argtypes = [_P, _I64, _INT, _P, _INT, _INT, _INT, C.POINTER(_P)]
        L.qref_pairs_free.argtypes = [_P]
        L.qref_pairs_info.argtypes = [_P, C.POINTER(_U64), C.POINTER(_U64), C.POINTER(_INT)]
        L.qref_pairs_copy.argtypes = [_P, _P]
        L.qref_pairs_from_triples.argtypes = [_U64, _P, C.POINTER(_P)]
        L.qref_local_energies.argtypes = [_P, _P, _I64, _INT, _P, _P, _P, _INT, _P]
        L.qref_variational_energy.argtypes = [_I64, _P, _D, _D, _P, _P, _P]
        L.qref_run_path.argtypes = [_P, _I64, _INT, _P, _P, _P, _P, _D, _D, _INT, _INT, _INT, _P, _P, _P,
                                    C.POINTER(_U64)]
        L.qref_rows_session.restype = _P
        L.qref_rows_session.argtypes = [_P, _I64, _INT, _P, _P, _P, _P, _D, _D, C.POINTER(_D)]
        L.qref_rows_session_free.argtypes = [_P]
        L.qref_rows_session_run.argtypes = [_P, _I64, _P, _INT, _P, C.POINTER(_U64), _P]
        L.qref_rng_new.restype = _P
        L.qref_rng_new.argtypes = [_U64, C.c_uint32]
        L.qref_rng_free.argtypes = [_P]
        L.qref_rng_uniform_int.restype = _U64
        L.qref_rng_uniform_int.argtypes = [_P, _U64]
        L.qref_rng_bits64.restype = _U64
        L.qref_rng_bits64.argtypes = [_P]
        L.qref_model_create.argtypes = [_INT, _INT, _INT, _INT, _INT, C.POINTER(_P)]
        L.qref_model_free.argtypes = [_P]
        L.qref_model_n_params.restype = _I64
        L.qref_model_n_params.argtypes = [_P]
        L.qref_model_init_params.argtypes = [_P, _U64]
        L.qref_model_get_params.argtypes = [_P, _P]
        L.qref_model_set_params.argtypes = [_P, _I64, _P]
        L.qref_model_log_psi.argtypes = [_P, _I64, _INT, _P, _INT, _P, _P]
        L.qref_fill_amplitudes.argtypes = [_P, _I64, _INT, _P, _P, _INT, _P, _P, _P]
        L.qref_sample.argtypes = [_P, _INT, _U64, C.c_uint32, C.c_uint32, _INT, _INT, _P, _P, C.POINTER(_I64)]
        L.qref_grad_log_psi.argtypes = [_P, _I64, _INT, _P, _INT, _P]
        L.qref_energy_gradient.argtypes = [_P, _I64, _INT, _P, _P, _P, _INT, _P]
        L.qref_condition_max.restype = C.c_double
        L.qref_condition_max.argtypes = [C.c_double] * 3
        L.qref_gumbel.restype = C.c_double
        L.qref_gumbel.argtypes = [_U64] + [C.c_uint32] * 5
        _rlib = L
    return _rlib


class RefError(Exception):
    pass


def _rcheck(status):
    if status != 0:
        msg = rlib().qref_last_error().decode()
        kind = msg.split(":", 1)[0]
        exc = {"invalid_argument": ValueError, "logic_error": RefError, "runtime_error": RuntimeError}.get(kind, RefError)
        raise exc(msg)


class RefIndex:
    """A reference HamiltonianIndex (the real class, compiled from the reference sources)."""

    def __init__(self, handle):
        self._h = handle
        nq, nt, nxy, dg = _INT(), _U64(), C.c_uint32(), _I64()
        _rcheck(rlib().qref_index_info(handle, C.byref(nq), C.byref(nt), C.byref(nxy), C.byref(dg)))
        self.n_qubits, self.n_terms, self.n_xy, self.diag = nq.value, nt.value, nxy.value, dg.value
        self.W = (self.n_qubits + 63) // 64
        W = self.W
        self.xy = np.zeros((self.n_xy, W), dtype=np.uint64)
        self.offsets = np.zeros(self.n_xy + 1, dtype=np.uint64)
        self.coeff = np.zeros(self.n_terms)
        self.x = np.zeros((self.n_terms, W), dtype=np.uint64)
        self.y = np.zeros((self.n_terms, W), dtype=np.uint64)
        self.z = np.zeros((self.n_terms, W), dtype=np.uint64)
        self.yz = np.zeros((self.n_terms, W), dtype=np.uint64)
        self.y_weight = np.zeros(self.n_terms, dtype=np.uint8)
        _rcheck(rlib().qref_index_export(handle, W, _ptr(self.xy), _ptr(self.offsets), _ptr(self.coeff),
                                         _ptr(self.x), _ptr(self.y), _ptr(self.z), _ptr(self.yz),
                                         _ptr(self.y_weight)))

    @staticmethod
    def parse(text: str) -> "RefIndex":
        h = _P()
        _rcheck(rlib().qref_index_parse(text.encode(), C.byref(h)))
        return RefIndex(h)

    @staticmethod
    def from_strings(n_qubits, coeffs, strings) -> "RefIndex":
        h = _P()
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        _rcheck(rlib().qref_index_from_strings(n_qubits, len(c), _ptr(c), "".join(strings).encode(), C.byref(h)))
        return RefIndex(h)

    @staticmethod
    def random(n_qubits, n_terms, seed, max_weight=4) -> "RefIndex":
        h = _P()
        _rcheck(rlib().qref_random_hamiltonian(n_qubits, n_terms, seed, max_weight, C.byref(h)))
        return RefIndex(h)

    def __del__(self):
        if getattr(self, "_h", None):
            rlib().qref_index_free(self._h)

    def matrix_element(self, x, xp):
        out = np.zeros(2)
        _rcheck(rlib().qref_matrix_element(self._h, self.W, _ptr(np.ascontiguousarray(x, dtype=np.uint64)),
                                           _ptr(np.ascontiguousarray(xp, dtype=np.uint64)), _ptr(out)))
        return complex(out[0], out[1])

    def group_element(self, xp, g):
        out = np.zeros(2)
        _rcheck(rlib().qref_group_element(self._h, self.W, _ptr(np.ascontiguousarray(xp, dtype=np.uint64)), g,
                                          _ptr(out)))
        return complex(out[0], out[1])

    def pairs(self, keys, backend=3, threshold=4096, threads=1):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        p = _P()
        _rcheck(rlib().qref_pairs(self._h, keys.shape[0], self.W, _ptr(keys), backend, threshold, threads,
                                  C.byref(p)))
        n, ops, be = _U64(), _U64(), _INT()
        rlib().qref_pairs_info(p, C.byref(n), C.byref(ops), C.byref(be))
        out = np.zeros((n.value, 3), dtype=np.uint32)
        rlib().qref_pairs_copy(p, _ptr(out))
        rlib().qref_pairs_free(p)
        return out, ops.value, be.value

    def local_energies(self, keys, la, ph, entries, threads=1):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        entries = np.ascontiguousarray(entries, dtype=np.uint32).reshape(-1, 3)
        la, ph = (np.ascontiguousarray(a, dtype=np.float64) for a in (la, ph))
        p = _P()
        _rcheck(rlib().qref_pairs_from_triples(entries.shape[0], _ptr(entries), C.byref(p)))
        out = np.zeros(keys.shape[0], dtype=np.complex128)
        try:
            _rcheck(rlib().qref_local_energies(self._h, p, keys.shape[0], self.W, _ptr(keys), _ptr(la), _ptr(ph),
                                               threads, _ptr(out)))
        finally:
            rlib().qref_pairs_free(p)
        return out

    def run_path(self, keys, la, ph, lp, norm, log_norm, backend=3, threshold=4096, threads=1, want_locals=True):
        """find_coupled_pairs -> local_energies -> variational_energy; returns (locals, out5, times3, n_pairs)."""
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        la, ph, lp = (np.ascontiguousarray(a, dtype=np.float64) for a in (la, ph, lp))
        locals_ = np.zeros(keys.shape[0], dtype=np.complex128) if want_locals else None
        out5, t3, npairs = np.zeros(5), np.zeros(3), _U64()
        _rcheck(rlib().qref_run_path(self._h, keys.shape[0], self.W, _ptr(keys), _ptr(la), _ptr(ph), _ptr(lp), norm,
                                     log_norm, backend, threshold, threads, _ptr(locals_), _ptr(out5), _ptr(t3),
                                     C.byref(npairs)))
        return locals_, out5, t3, npairs.value

    def row_session(self, keys, la, ph, lp, norm, log_norm):
        return RefRowSession(self, keys, la, ph, lp, norm, log_norm)


class RefRowSession:
    """Listed rows of the whole sample set against the whole sample set, through
    the reference (ref_capi.cpp qref_rows_session*): the per-row trie walk of
    loop_over_trie over the reference's PrefixTree builds of the full set
    (build_seconds: built once here), then the unmodified local_energies and
    variational_energy over the full batch."""

    def __init__(self, index: "RefIndex", keys, la, ph, lp, norm, log_norm):
        self._keys = np.ascontiguousarray(keys, dtype=np.uint64)
        la, ph, lp = (np.ascontiguousarray(a, dtype=np.float64) for a in (la, ph, lp))
        self.n = self._keys.shape[0]
        b = _D()
        self._s = rlib().qref_rows_session(index._h, self.n, index.W, _ptr(self._keys), _ptr(la), _ptr(ph),
                                           _ptr(lp), norm, log_norm, C.byref(b))
        if not self._s:
            raise RefError(rlib().qref_last_error().decode())
        self.build_seconds = b.value

    def run(self, rows, threads=1, want_locals=False):
        """-> (times3 = search, local_energies, variational_energy seconds; pairs; E_loc of the rows or None)"""
        rows = np.ascontiguousarray(np.sort(np.asarray(rows, dtype=np.int64)))
        t3, npairs = np.zeros(3), _U64()
        out = np.zeros(len(rows), dtype=np.complex128) if want_locals else None
        _rcheck(rlib().qref_rows_session_run(self._s, len(rows), _ptr(rows), threads, _ptr(t3), C.byref(npairs),
                                             _ptr(out) if out is not None else None))
        return t3, npairs.value, out

    def __del__(self):
        if getattr(self, "_s", None):
            rlib().qref_rows_session_free(self._s)


def ref_variational_energy(log_probs, norm, log_norm, eloc):
    lp = np.ascontiguousarray(log_probs, dtype=np.float64)
    e = np.ascontiguousarray(eloc, dtype=np.complex128)
    out = np.zeros(5)
    w = np.zeros(len(lp))
    _rcheck(rlib().qref_variational_energy(len(lp), _ptr(lp), norm, log_norm, _ptr(e), _ptr(out), _ptr(w)))
    return out, w


def ref_random_vectors(n_qubits, count, seed):
    W = (n_qubits + 63) // 64
    out = np.zeros((count, W), dtype=np.uint64)
    _rcheck(rlib().qref_random_distinct_vectors(n_qubits, count, seed, W, _ptr(out)))
    return out


class RefRng:
    """qvmc::SequentialRng (rng.hpp:70-93) from the compiled reference."""

    def __init__(self, seed, stream=0):
        self._r = rlib().qref_rng_new(seed, stream)

    def __del__(self):
        if getattr(self, "_r", None):
            rlib().qref_rng_free(self._r)

    def uniform_int(self, n):
        return int(rlib().qref_rng_uniform_int(self._r, n))


class RefModel:
    """The reference AnqsModel (model.cpp) compiled from the reference sources."""

    def __init__(self, n_qubits, bits_per_qudit, n_electrons, spin_constraint=False, hidden=64):
        self.n_qubits = n_qubits
        self.W = (n_qubits + 63) // 64
        h = _P()
        _rcheck(rlib().qref_model_create(n_qubits, bits_per_qudit, n_electrons, int(spin_constraint), hidden,
                                         C.byref(h)))
        self._h = h
        self.n_params = int(rlib().qref_model_n_params(h))

    def __del__(self):
        if getattr(self, "_h", None):
            rlib().qref_model_free(self._h)
            self._h = None

    def init_params(self, seed: int) -> None:
        _rcheck(rlib().qref_model_init_params(self._h, seed))

    @property
    def params(self) -> np.ndarray:
        p = np.zeros(self.n_params)
        _rcheck(rlib().qref_model_get_params(self._h, _ptr(p)))
        return p

    def set_params(self, p) -> None:
        p = np.ascontiguousarray(p, dtype=np.float64)
        _rcheck(rlib().qref_model_set_params(self._h, p.size, _ptr(p)))

    def log_psi(self, keys, threads: int = 1):
        keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1, self.W)
        n = keys.shape[0]
        la, ph = np.zeros(n), np.zeros(n)
        _rcheck(rlib().qref_model_log_psi(self._h, n, self.W, _ptr(keys), threads, _ptr(la), _ptr(ph)))
        return la, ph

    def fill_amplitudes(self, keys, log_probs, threads: int = 1):
        keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1, self.W)
        lp = np.ascontiguousarray(log_probs, dtype=np.float64)
        n = keys.shape[0]
        la, ph, out2 = np.zeros(n), np.zeros(n), np.zeros(2)
        _rcheck(rlib().qref_fill_amplitudes(self._h, n, self.W, _ptr(keys), _ptr(lp), threads, _ptr(la), _ptr(ph),
                                            _ptr(out2)))
        return la, ph, float(out2[0]), float(out2[1])

    def sample(self, k_samples: int, seed: int, stream: int = 0, iteration: int = 0, threads: int = 1):
        """sample_without_replacement (sampler.cpp:37-102): (keys [n][W], log_probs [n])."""
        keys = np.zeros((k_samples, self.W), dtype=np.uint64)
        lp = np.zeros(k_samples)
        n = C.c_int64()
        _rcheck(rlib().qref_sample(self._h, k_samples, seed, stream, iteration, threads, self.W, _ptr(keys), _ptr(lp),
                                   C.byref(n)))
        return keys[: n.value], lp[: n.value]


def _ref_model_grad(self, keys, threads: int = 1):
    """batched_grad_log_psi (model.cpp:273-336): complex rows [n][n_params]."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1, self.W)
    n = keys.shape[0]
    out = np.zeros((n, self.n_params), dtype=np.complex128)
    _rcheck(rlib().qref_grad_log_psi(self._h, n, self.W, _ptr(keys), threads, _ptr(out)))
    return out


def _ref_energy_gradient(self, keys, weights, locals_, threads: int = 1):
    """energy_gradient (energy.cpp:93-107) over batched_grad_log_psi rows."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1, self.W)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    loc = np.ascontiguousarray(locals_, dtype=np.complex128)
    g = np.zeros(self.n_params)
    _rcheck(rlib().qref_energy_gradient(self._h, keys.shape[0], self.W, _ptr(keys), _ptr(w), _ptr(loc), threads,
                                        _ptr(g)))
    return g


RefModel.grad_log_psi = _ref_model_grad
RefModel.energy_gradient = _ref_energy_gradient


def ref_condition_max(parent, z, child):
    return float(rlib().qref_condition_max(parent, z, child))


def ref_gumbel(seed, stream, c0, c1, c2, c3):
    return float(rlib().qref_gumbel(seed, stream, c0, c1, c2, c3))
