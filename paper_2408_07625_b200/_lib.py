"""ctypes binding of libqvmc_cuda.so (the C ABI in include/qvmc_cuda.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2408_07625_b200/csrc``). There is no Python or CPU fallback:
if the library is missing every entry point raises ``ImportError``.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libqvmc_cuda.so"

QVMC_OK = 0
QVMC_ERR_INVALID_ARGUMENT = 1
QVMC_ERR_LOGIC = 2
QVMC_ERR_RUNTIME = 3
QVMC_ERR_CUDA = 4
QVMC_ERR_NO_DEVICE = 5

MEM_HOST = 0
MEM_DEVICE = 1

BACKEND_TERMS, BACKEND_BATCH, BACKEND_TRIE, BACKEND_AUTO = 0, 1, 2, 3


class QvmcLogicError(RuntimeError):
    """Maps the reference's std::logic_error (energy.cpp:32-33: zero amplitude)."""


class QvmcStats(C.Structure):
    _fields_ = [
        ("rows", C.c_uint64),
        ("candidates", C.c_uint64),
        ("pairs", C.c_uint64),
        ("terms_equivalent", C.c_uint64),
        ("sector_mode", C.c_int32),
        ("sector_side", C.c_int32),
        ("minority_count", C.c_int32),
        ("join_mode", C.c_int32),
        ("table_ms", C.c_float),
        ("rows_ms", C.c_float),
        ("moments_ms", C.c_float),
        ("search_ms", C.c_float),
        ("eval_ms", C.c_float),
    ]


class QvmcPlanSummary(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("kind_a", "kind_b", "kind_c", "kind_d", "bitmap_bits", "singles",
                                          "doubles", "xy_tab_buckets")]


_P = C.c_void_p
_I64 = C.c_int64
_U64 = C.c_uint64
_INT = C.c_int

# (name, restype, argtypes) for every symbol include/qvmc_cuda.h declares
SIGNATURES = [
    ("qvmc_index_build", _INT, [_INT, _INT, _I64, _P, _P, _P, _P, C.POINTER(_P)]),
    ("qvmc_index_info", _INT, [_P, C.POINTER(_INT), C.POINTER(_U64), C.POINTER(C.c_uint32), C.POINTER(_I64)]),
    ("qvmc_index_export", _INT, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("qvmc_index_destroy", None, [_P]),
    ("qvmc_index_plan_summary", _INT, [_P, _P]),
    ("qvmc_cuda_ham_create", _INT, [_INT, _INT, C.c_uint32, _P, _P, _U64, _P, _P, _P, _I64, _INT, C.POINTER(_P)]),
    ("qvmc_cuda_ham_create_from_index", _INT, [_P, _INT, C.POINTER(_P)]),
    ("qvmc_cuda_ham_destroy", _INT, [_P]),
    ("qvmc_cuda_set_stream", _INT, [_P, _P]),
    ("qvmc_cuda_synchronize", _INT, [_P]),
    ("qvmc_cuda_set_speculative", _INT, [_P, _INT]),
    ("qvmc_cuda_last_stats", _INT, [_P, C.POINTER(QvmcStats)]),
    ("qvmc_cuda_pairs", _INT, [_P, _I64, _P, _INT, _INT, _INT, C.POINTER(_U64), C.POINTER(_U64), C.POINTER(_INT)]),
    ("qvmc_cuda_pairs_fetch", _INT, [_P, _P, _INT]),
    ("qvmc_cuda_pair_elements", _INT, [_P, _I64, _P, _U64, _P, _P, _P, _INT]),
    ("qvmc_cuda_pair_elements_fused", _INT, [_P, _I64, _P, _U64, _P, _P, _P, _INT]),
    ("qvmc_cuda_local_energies", _INT, [_P, _I64, _P, _P, _P, _U64, _P, _P, _INT]),
    ("qvmc_cuda_energy_moments", _INT, [_P, _I64, _P, C.c_double, _P, _P, _P, _INT]),
    ("qvmc_cuda_eloc_fused", _INT, [_P, _I64, _P, _P, _P, _P, C.c_double, _I64, _I64, _P, _P, _INT]),
    ("qvmc_shard_bounds", _INT, [_I64, _INT, _INT, C.POINTER(_I64), C.POINTER(_I64)]),
    ("qvmc_cuda_comm_unique_id", _INT, [_P, _U64]),
    ("qvmc_cuda_comm_init_nccl", _INT, [_INT, _INT, _INT, _P, C.POINTER(_P)]),
    ("qvmc_cuda_comm_wrap_nccl", _INT, [_P, _INT, _INT, C.POINTER(_P)]),
    ("qvmc_cuda_comm_init_host", _INT, [_INT, _INT, _P, _P, C.POINTER(_P)]),
    ("qvmc_cuda_comm_destroy", _INT, [_P]),
    ("qvmc_cuda_eloc_sharded", _INT, [_P, _P, _I64, _P, _P, _P, _P, C.c_double, _P, _P, _INT]),
    ("qvmc_cuda_last_error", C.c_char_p, []),
    ("qvmc_cuda_launch_count", _U64, []),
    ("qvmc_cuda_model_create", _INT, [_INT, _INT, _INT, _INT, _INT, _INT, C.POINTER(_P)]),
    ("qvmc_cuda_model_destroy", _INT, [_P]),
    ("qvmc_cuda_model_n_params", _INT, [_P, C.POINTER(_I64)]),
    ("qvmc_cuda_model_set_params", _INT, [_P, _I64, _P]),
    ("qvmc_cuda_model_set_stream", _INT, [_P, _P]),
    ("qvmc_cuda_log_psi", _INT, [_P, _I64, _P, _INT, _P, _P]),
    ("qvmc_cuda_fill_amplitudes", _INT, [_P, _I64, _P, _P, _INT, _P, _P, _P]),
    ("qvmc_cuda_model_last_fill_sampled", _INT, [_P]),
    ("qvmc_cuda_model_last_gradient_cached", _INT, [_P]),
    ("qvmc_cuda_model_synchronize", _INT, [_P]),
    ("qvmc_cuda_energy_gradient", _INT, [_P, _I64, _P, _P, _P, _INT, _P]),
    ("qvmc_cuda_model_get_params", _INT, [_P, _INT, _P]),
    ("qvmc_cuda_model_adam_step", _INT, [_P, _P, C.c_double, C.c_double, C.c_double, C.c_double, _INT]),
    ("qvmc_cuda_sr_solve", _INT, [_P, _I64, _I64, _P, C.c_double, _P, _INT, _P]),
    ("qvmc_cuda_sr_direction", _INT, [_P, _I64, _P, _P, _P, _INT, C.c_double, _P, _INT, _P, C.POINTER(C.c_double)]),
    ("qvmc_cuda_sample", _INT, [_P, _INT, _U64, C.c_uint32, C.c_uint32, _INT, _P, _P, C.POINTER(_I64)]),
]

_lib = None


def lib() -> C.CDLL:
    """Load libqvmc_cuda.so once; raise ImportError if it was never built."""
    global _lib
    if _lib is None:
        path = Path(os.environ.get("QVMC_CUDA_LIB", LIB_PATH))
        if not path.exists():
            raise ImportError(
                f"{path} is missing: the B200 kernels are not built. Run __graft_entry__.build() "
                "(there is no CPU fallback for the local-energy path).")
        handle = C.CDLL(str(path))
        for name, res, args in SIGNATURES:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().qvmc_cuda_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    """Raise the Python analogue of the reference's exception for a status."""
    if status == QVMC_OK:
        return
    msg = last_error()
    if status == QVMC_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == QVMC_ERR_LOGIC:
        raise QvmcLogicError(msg)
    if status == QVMC_ERR_NO_DEVICE:
        raise RuntimeError(f"no B200 device: {msg}")
    raise RuntimeError(msg)


# qvmc_host_allgather_fn (include/qvmc_cuda.h)
HOST_ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)


def launch_count() -> int:
    return int(lib().qvmc_cuda_launch_count())
