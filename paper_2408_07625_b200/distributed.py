"""Multi-GPU surrogate local energies: one process per GPU, rows sharded.

SURVEY.md §8(e): every rank owns a contiguous shard of the unique samples
(keys + log|psi| + phase + log p). The partner lookup needs the whole sample
set, so the shards are all-gathered over NVLink (NCCL through
torch.distributed), each rank evaluates E_loc for its own rows against the
gathered set with the fused kernel, and the five fp64 energy moments are
all-reduced. Per-rank row results never leave the rank unless the caller
asks for them (``gather_locals``).

The per-rank evaluation is ``qvmc_cuda_eloc_fused`` on device pointers; the
``evaluate`` hook exists so the gather/offset/reduce plumbing can be tested
with the gloo backend on CPU-only hosts.

``sharded_fill_amplitudes`` is the stage before it (fill_amplitudes,
sampler.cpp:104-120) on the same shards: log|psi| and phase of a rank's own
rows only (independent rows, no data-path collective), and the global
log_norm = logsumexp of the sampler's log_probs merged from per-rank
(max, scaled sum) pairs gathered in rank order (deterministic).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Callable, List, Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .hamiltonian import HamiltonianIndex


@dataclass
class Shard:
    """This rank's rows of the sample set (torch tensors on this rank's device)."""
    keys: torch.Tensor      # int64 viewed as uint64 words, [rows, n_words]
    log_amps: torch.Tensor  # float64 [rows]
    phases: torch.Tensor    # float64 [rows]
    log_probs: torch.Tensor # float64 [rows]


@dataclass
class ShardResult:
    locals: torch.Tensor    # complex128 [rows] (this rank's rows)
    moments: torch.Tensor   # float64 [5], already all-reduced over ranks
    row_begin: int
    row_end: int
    n_total: int

    @property
    def e_var(self) -> float:
        return float(self.moments[0])


def _gather_rows(t: torch.Tensor, counts: List[int], group) -> torch.Tensor:
    """All-gather variable-length row blocks (padded to the largest shard)."""
    world = len(counts)
    m = max(counts)
    pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    out = torch.empty((world * m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    if all(c == m for c in counts):
        return out
    return torch.cat([out[r * m: r * m + counts[r]] for r in range(world)])


def device_evaluate(index: HamiltonianIndex, device: int) -> Callable:
    """The fused kernel on device pointers, on torch's current stream."""
    h = index.device_handle(device)
    L = _lib.lib()

    def run(keys, la, ph, lp, log_norm, r0, r1, out_locals, out_moments):
        # torch's default stream is the legacy NULL stream: pass cudaStreamLegacy (0x1), since
        # NULL selects the handle's own non-blocking stream
        raw = torch.cuda.current_stream(device).cuda_stream or 0x1
        _lib.check(L.qvmc_cuda_set_stream(h, C.c_void_p(raw)))
        try:
            _lib.check(L.qvmc_cuda_eloc_fused(
                h, keys.shape[0], C.c_void_p(keys.data_ptr()), C.c_void_p(la.data_ptr()), C.c_void_p(ph.data_ptr()),
                C.c_void_p(lp.data_ptr()), float(log_norm), r0, r1,
                C.c_void_p(out_locals.data_ptr()) if out_locals is not None else None,
                C.c_void_p(out_moments.data_ptr()), _lib.MEM_DEVICE))
        finally:  # later calls on the shared handle use its own stream again
            _lib.check(L.qvmc_cuda_set_stream(h, None))

    return run


def sharded_surrogate_energy(shard: Shard, log_norm: float, evaluate: Callable, group=None,
                             gather_locals: bool = False) -> ShardResult:
    """E_loc for this rank's rows + globally reduced moments.

    ``log_norm`` is the global log sum_x p(x) (the sampler's value)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = shard.keys.device
    cnt = torch.tensor([shard.keys.shape[0]], dtype=torch.int64, device=dev)
    counts_t = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(counts_t, cnt, group=group)
    counts = [int(c) for c in counts_t.cpu()]
    r0 = sum(counts[:rank])
    r1 = r0 + counts[rank]
    keys = _gather_rows(shard.keys, counts, group)
    # amplitudes travel as one [rows, 3] block: one collective instead of three
    amps = _gather_rows(torch.stack([shard.log_amps, shard.phases, shard.log_probs], dim=1), counts, group)
    la, ph, lp = (amps[:, k].contiguous() for k in range(3))
    locals_ = torch.zeros(max(r1 - r0, 1), dtype=torch.complex128, device=dev)
    moments = torch.zeros(5, dtype=torch.float64, device=dev)
    evaluate(keys, la, ph, lp, log_norm, r0, r1, locals_, moments)
    dist.all_reduce(moments, op=dist.ReduceOp.SUM, group=group)
    res = ShardResult(locals_[: r1 - r0], moments, r0, r1, sum(counts))
    if gather_locals:
        res.locals = _gather_rows(res.locals, counts, group)
    return res


def shard_bounds(n: int, world: int, rank: int) -> tuple:
    """Contiguous, balanced row shard [begin, end) of rank (= qvmc_shard_bounds)."""
    base, rem = divmod(n, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


class Communicator:
    """qvmc_comm_t: the collectives of qvmc_cuda_eloc_sharded inside libqvmc_cuda.

    ``nccl(group, device)``: rank 0 draws an NCCL unique id
    (qvmc_cuda_comm_unique_id), the process group broadcasts it, every rank
    calls qvmc_cuda_comm_init_nccl: all-gathers run inside the library on the
    handle's stream over NVLink. ``host(group)``: a host all-gather callback
    over the process group (gloo works): the library stages through pinned
    host memory. Several ranks may then share one GPU (tests)."""

    def __init__(self, handle, world: int, rank: int, keepalive=None):
        self._h = handle
        self.world = world
        self.rank = rank
        self._keep = keepalive

    @classmethod
    def nccl(cls, device: int, group=None) -> "Communicator":
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            _lib.check(_lib.lib().qvmc_cuda_comm_unique_id(uid, 128))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0, group=group)
        uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        h = C.c_void_p()
        _lib.check(_lib.lib().qvmc_cuda_comm_init_nccl(device, world, rank, uid, C.byref(h)))
        return cls(h, world, rank)

    @classmethod
    def host(cls, group=None) -> "Communicator":
        world, rank = dist.get_world_size(group), dist.get_rank(group)

        def all_gather(ctx, send, recv, nbytes):
            try:
                src = np.ctypeslib.as_array((C.c_uint8 * max(nbytes, 1)).from_address(send))[:nbytes]
                t = torch.from_numpy(src.copy())
                outs = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(outs, t, group=group)
                dst = np.ctypeslib.as_array((C.c_uint8 * max(nbytes * world, 1)).from_address(recv))
                dst[: nbytes * world] = torch.cat(outs).numpy()
                return 0
            except Exception:  # noqa: BLE001 - reported to the library as a failed collective
                return 1

        cb = _lib.HOST_ALLGATHER_FN(all_gather)
        h = C.c_void_p()
        _lib.check(_lib.lib().qvmc_cuda_comm_init_host(world, rank, cb, None, C.byref(h)))
        return cls(h, world, rank, keepalive=cb)

    def close(self) -> None:
        if self._h:
            _lib.check(_lib.lib().qvmc_cuda_comm_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def sharded_surrogate_energy_capi(index: HamiltonianIndex, comm: Communicator, device: int, n_total: int,
                                  shard: Shard, log_norm: float) -> ShardResult:
    """qvmc_cuda_eloc_sharded on device pointers (torch's current stream): the
    gather, the fused evaluation of this rank's rows and the rank-order moment
    sum all run inside libqvmc_cuda. ``shard`` = rows qvmc_shard_bounds(rank)."""
    r0, r1 = shard_bounds(n_total, comm.world, comm.rank)
    if shard.keys.shape[0] != r1 - r0:
        raise ValueError(f"rank {comm.rank} holds {shard.keys.shape[0]} rows, its shard is {r1 - r0}")
    h = index.device_handle(device)
    L = _lib.lib()
    dev = shard.keys.device
    locals_ = torch.zeros(max(r1 - r0, 1), dtype=torch.complex128, device=dev)
    moments = torch.zeros(5, dtype=torch.float64, device=dev)
    raw = torch.cuda.current_stream(device).cuda_stream or 0x1  # 0x1 = cudaStreamLegacy
    _lib.check(L.qvmc_cuda_set_stream(h, C.c_void_p(raw)))
    try:
        _lib.check(L.qvmc_cuda_eloc_sharded(
            h, comm._h, n_total, C.c_void_p(shard.keys.data_ptr()), C.c_void_p(shard.log_amps.data_ptr()),
            C.c_void_p(shard.phases.data_ptr()), C.c_void_p(shard.log_probs.data_ptr()), float(log_norm),
            C.c_void_p(locals_.data_ptr()), C.c_void_p(moments.data_ptr()), _lib.MEM_DEVICE))
    finally:
        _lib.check(L.qvmc_cuda_set_stream(h, None))
    return ShardResult(locals_[: r1 - r0], moments, r0, r1, n_total)


def model_evaluate(model, device: int) -> Callable:
    """k_log_psi_part on device pointers, on torch's current stream."""

    def run(keys, out_la, out_ph):
        raw = torch.cuda.current_stream(device).cuda_stream or 0x1  # 0x1 = cudaStreamLegacy
        _lib.check(_lib.lib().qvmc_cuda_model_set_stream(model._h, C.c_void_p(raw)))
        try:
            model.log_psi_device(keys.data_ptr(), keys.shape[0], out_la.data_ptr(), out_ph.data_ptr())
        finally:
            _lib.check(_lib.lib().qvmc_cuda_model_set_stream(model._h, None))

    return run


def sharded_fill_amplitudes(shard: Shard, evaluate: Callable, group=None) -> float:
    """fill_amplitudes (sampler.cpp:104-120) for this rank's rows: writes shard.log_amps /
    shard.phases in place and returns the global log_norm of the sampler's log_probs."""
    world = dist.get_world_size(group)
    dev = shard.keys.device
    if shard.keys.shape[0]:
        evaluate(shard.keys, shard.log_amps, shard.phases)
    lp = shard.log_probs
    m = lp.max() if lp.numel() else torch.tensor(float("-inf"), dtype=torch.float64, device=dev)
    s = torch.exp(lp - m).sum() if lp.numel() and torch.isfinite(m) else torch.zeros((), dtype=torch.float64,
                                                                                       device=dev)
    pair = torch.stack([m.to(torch.float64), s.to(torch.float64)])
    flat = torch.empty(2 * world, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(flat, pair, group=group)
    pairs = flat.view(world, 2).cpu()
    gm, gs = float("-inf"), 0.0
    for r in range(world):  # merge in rank order
        mr, sr = float(pairs[r, 0]), float(pairs[r, 1])
        mm = max(gm, mr)
        if mm == float("-inf"):
            continue
        gs = gs * math.exp(gm - mm) + sr * math.exp(mr - mm)
        gm = mm
    return gm + math.log(gs) if gs > 0 else float("-inf")
