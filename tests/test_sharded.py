"""qvmc_cuda_eloc_sharded: the multi-GPU path behind the C ABI.

Each rank passes its shard (qvmc_shard_bounds rows); the library all-gathers
the packed shards, evaluates its rows with the fused kernels and sums the
per-rank moments in rank order. Checked on one B200:
  * world 1 over NCCL (ncclCommInitRank inside libqvmc_cuda): bit-identical
    to qvmc_cuda_eloc_fused, host and device memory;
  * world 2 and 3 with the host all-gather backend over gloo, every rank a
    process on cuda:0 (NCCL refuses two ranks on one GPU): each rank walks
    every world-th row of the locality order (or its own rows), partners
    after them, the mirrored fixed-point sums are all-reduced exactly and
    the rows assembled exactly, so each rank's rows are bit-identical to the
    unsharded (symmetric) E_loc; moments to fp64 reordering.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _problem(n_qubits=56, n_e=14, n_terms=300_000, n_unq=20_011, by_excitation=False):
    from paper_2408_07625_b200 import synthetic
    c, x, y, z = synthetic.jw_terms(n_qubits, n_terms, seed=1)
    keys = synthetic.near_hf_keys(n_qubits, n_e, n_unq, seed=4)
    if by_excitation:  # samples ordered by excitation rank (as a sampler's beam order can be):
        # contiguous shards then carry very different pair counts
        hf = (1 << n_e) - 1
        rank = np.array([bin(int(k) ^ hf).count("1") for k in keys[:, 0]])
        keys = keys[np.argsort(rank, kind="stable")]
    return n_qubits, (c, x, y, z), synthetic.sample_batch(keys, seed=3)


def test_world1_nccl_matches_fused(cuda_ok):
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import _lib
    from paper_2408_07625_b200.hamiltonian import _ptr
    n_qubits, masks, b = _problem()
    H = q.HamiltonianIndex.from_masks(n_qubits, *masks)
    ref = q.surrogate_energy(H, b)
    L = _lib.lib()
    uid = (C.c_uint8 * 128)()
    _lib.check(L.qvmc_cuda_comm_unique_id(uid, 128))
    comm = C.c_void_p()
    _lib.check(L.qvmc_cuda_comm_init_nccl(0, 1, 0, uid, C.byref(comm)))
    try:
        n = b.size()
        loc = np.zeros(n, dtype=np.complex128)
        mom = np.zeros(5)
        _lib.check(L.qvmc_cuda_eloc_sharded(H.device_handle(0), comm, n, _ptr(b.vectors), _ptr(b.log_amps),
                                            _ptr(b.phases), _ptr(b.log_probs), b.log_norm, _ptr(loc), _ptr(mom),
                                            _lib.MEM_HOST))
        assert np.array_equal(loc, ref.locals)
        assert mom[0] == ref.e_var
        # device memory through torch on its stream
        import torch
        from paper_2408_07625_b200.distributed import Communicator, Shard, sharded_surrogate_energy_capi
        dev = torch.device("cuda", 0)
        sh = Shard(torch.from_numpy(b.vectors.view(np.int64)).to(dev), torch.from_numpy(b.log_amps).to(dev),
                   torch.from_numpy(b.phases).to(dev), torch.from_numpy(b.log_probs).to(dev))
        cm = Communicator(comm, 1, 0)
        res = sharded_surrogate_energy_capi(H, cm, 0, n, sh, b.log_norm)
        torch.cuda.synchronize()
        assert np.array_equal(res.locals.cpu().numpy(), ref.locals)
        assert float(res.moments[0]) == ref.e_var
        cm._h = None  # destroyed below
    finally:
        _lib.check(L.qvmc_cuda_comm_destroy(comm))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_q, by_excitation=False):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2408_07625_b200 as q
        from paper_2408_07625_b200.distributed import Communicator, Shard, shard_bounds, sharded_surrogate_energy_capi
        n_qubits, masks, b = _problem(by_excitation=by_excitation)
        H = q.HamiltonianIndex.from_masks(n_qubits, *masks)
        r0, r1 = shard_bounds(b.size(), world, rank)
        dev = torch.device("cuda", 0)
        sh = Shard(torch.from_numpy(b.vectors[r0:r1].view(np.int64).copy()).to(dev),
                   torch.from_numpy(b.log_amps[r0:r1].copy()).to(dev), torch.from_numpy(b.phases[r0:r1].copy()).to(dev),
                   torch.from_numpy(b.log_probs[r0:r1].copy()).to(dev))
        comm = Communicator.host()
        res = sharded_surrogate_energy_capi(H, comm, 0, b.size(), sh, b.log_norm)
        torch.cuda.synchronize()
        st = q.last_stats(H)
        out_q.put((rank, res.row_begin, res.row_end, res.locals.cpu().numpy(), res.moments.cpu().numpy(),
                   st["join_mode"], st["pairs"]))
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dist,strided,by_exc", [
    (2, "1", "1", False), (3, "1", "1", False), (2, "0", "1", False),
    (3, "1", "0", False), (3, "1", "1", True), (3, "1", "0", True)])
def test_multi_rank_host_backend_matches_unsharded(cuda_ok, monkeypatch, world, dist, strided, by_exc):
    """dist = 1: the deletion index is built across the ranks (each sorts the buckets it owns,
    all-gather of members, all-reduce of ranges); 0: every rank builds the whole index.
    strided = 1 (default): rank r walks sorted positions r, r + world, ... and the rows are
    assembled by an exact all-reduce; 0: each rank walks its own caller rows. by_exc: samples
    ordered by excitation rank, where contiguous walks are unbalanced and strided ones are not."""
    monkeypatch.setenv("QVMC_DIST_INDEX", dist)
    monkeypatch.setenv("QVMC_STRIDED_SHARDS", strided)
    import torch.multiprocessing as mp
    import paper_2408_07625_b200 as q
    n_qubits, masks, b = _problem(by_excitation=by_exc)
    H = q.HamiltonianIndex.from_masks(n_qubits, *masks)
    ref = q.surrogate_energy(H, b)
    w = np.exp(b.log_probs - b.log_norm)
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, qu, by_exc)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted(qu.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    covered = 0
    pairs = [o[6] for o in outs]
    if strided == "1":  # neighbours in locality order cost about the same: balanced walks
        assert max(pairs) <= 1.1 * min(pairs), pairs
    bad = [(o[0], [(int(i) + o[1], complex(o[3][i]), complex(ref.locals[o[1] + i]))
                   for i in np.flatnonzero(o[3] != ref.locals[o[1]:o[2]])[:4]]) for o in outs]
    bad = [(r, v) for r, v in bad if v]
    assert not bad, bad  # rows differing from the unsharded E_loc, per rank
    for rank, r0, r1, loc, mom, mode, _ in outs:
        assert mode == (2 if dist == "1" else 1)
        # symmetric across ranks (each unordered pair once, mirrored sums all-reduced exactly):
        # every row is the single-GPU result bit for bit
        assert np.array_equal(loc, ref.locals[r0:r1])
        assert abs(mom[0] - ref.e_var) <= 1e-12 * max(1.0, abs(ref.e_var))
        assert abs(mom[3] - w.sum()) <= 1e-12 * w.sum()
        np.testing.assert_array_equal(mom, outs[0][4])  # every rank holds the same rank-order sum
        covered += r1 - r0
    assert covered == b.size()


def _sharded_threads(world, n_qubits, c, x, y, z, b):
    """world ranks as threads of this process, each with its own device handle on cuda:0 and a
    host all-gather over a thread barrier (the in-process form of the gloo tests above)."""
    import ctypes as C
    import threading
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import _lib
    from paper_2408_07625_b200.hamiltonian import _ptr
    n = b.size()
    barrier, bufs, outs = threading.Barrier(world), [None] * world, [None] * world
    L = _lib.lib()

    def make_fn(rank):
        def fn(ctx, send, recv, nbytes):
            bufs[rank] = C.string_at(send, nbytes)
            barrier.wait()
            C.memmove(recv, b"".join(bufs), nbytes * world)
            barrier.wait()
            return 0
        return _lib.HOST_ALLGATHER_FN(fn)

    fns = [make_fn(r) for r in range(world)]
    Hs = [q.HamiltonianIndex.from_masks(n_qubits, c, x, y, z) for _ in range(world)]
    errors = []

    def run(rank):
        try:
            comm = C.c_void_p()
            _lib.check(L.qvmc_cuda_comm_init_host(world, rank, fns[rank], None, C.byref(comm)))
            r0, r1 = C.c_int64(), C.c_int64()
            _lib.check(L.qvmc_shard_bounds(n, world, rank, C.byref(r0), C.byref(r1)))
            r0, r1 = r0.value, r1.value
            out = np.zeros(max(r1 - r0, 1), dtype=np.complex128)
            mom = np.zeros(5)
            sl = lambda a: np.ascontiguousarray(a[r0:r1])
            _lib.check(L.qvmc_cuda_eloc_sharded(Hs[rank].device_handle(0), comm, n, _ptr(sl(b.vectors)),
                                                _ptr(sl(b.log_amps)), _ptr(sl(b.phases)), _ptr(sl(b.log_probs)),
                                                b.log_norm, _ptr(out), _ptr(mom), _lib.MEM_HOST))
            _lib.check(L.qvmc_cuda_comm_destroy(comm))
            outs[rank] = (r0, r1, out[: r1 - r0], mom, q.last_stats(Hs[rank]))
        except Exception as e:  # noqa: BLE001 - surfaced by the test below
            errors.append(e)
            barrier.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errors:
        raise errors[0]
    return outs


@pytest.mark.parametrize("case,world", [("join56", 2), ("join56", 3), ("sector_lists", 2), ("mixed_popcount", 3),
                                        ("join_s32", 2)])
def test_sharded_row_paths_in_process(cuda_ok, monkeypatch, case, world):
    """Every row path under the sharded call: the join (strided walk, distributed index), the
    sector candidate lists (QVMC_JOIN=0) and a mixed-popcount set (flip-mask scan over a sample
    hash table) — the last two split contiguously. Each rank's rows bit-identical to the
    unsharded E_loc, the global moments equal on every rank and to 1e-12 of the unsharded ones."""
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import synthetic
    if case == "join56":
        n_qubits, (c, x, y, z) = 56, synthetic.jw_terms(56, 100_000, seed=1)
        keys = synthetic.near_hf_keys(56, 14, 3001, seed=4)
    elif case == "sector_lists":
        monkeypatch.setenv("QVMC_JOIN", "0")
        n_qubits, (c, x, y, z) = 48, synthetic.jw_terms(48, 20_000, seed=1)
        keys = synthetic.near_hf_keys(48, 24, 1201, seed=2)
    elif case == "mixed_popcount":
        n_qubits, (c, x, y, z) = 20, synthetic.jw_terms(20, 12_000, seed=1)
        keys = np.unique(np.concatenate([synthetic.random_sector_keys(20, 10, 1500, seed=2),
                                         synthetic.random_sector_keys(20, 9, 700, seed=3)]), axis=0)
        keys = keys[np.random.default_rng(5).permutation(len(keys))]
    else:
        n_qubits, (c, x, y, z) = 64, synthetic.jw_terms(64, 30_000, seed=1)
        keys = synthetic.near_hf_keys(64, 32, 800, seed=2)
    b = synthetic.sample_batch(keys, seed=3)
    H = q.HamiltonianIndex.from_masks(n_qubits, c, x, y, z)
    ref = q.surrogate_energy(H, b)
    st = q.last_stats(H)
    assert (st["join_mode"] == 1) == case.startswith("join")
    assert (st["sector_mode"] == 1) == (case != "mixed_popcount")
    outs = _sharded_threads(world, n_qubits, c, x, y, z, b)
    covered = 0
    for r0, r1, loc, mom, _ in outs:
        assert np.array_equal(loc, ref.locals[r0:r1])
        assert abs(mom[0] - ref.e_var) <= 1e-12 * max(1.0, abs(ref.e_var))
        np.testing.assert_array_equal(mom, outs[0][3])
        covered += r1 - r0
    assert covered == b.size()
