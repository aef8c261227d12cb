"""Small end-to-end exercise of every device path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): toy KAT, a reference golden
family, the join path at 118 and 56 qubits (pipelined search + chunk
evaluation, including the overflow regrow with a tiny first hit capacity),
pair materialisation + local_energies + fused pair elements, the join at
minority sets of 24 and 32 and the sector-list row kernel, the amplitude
model, sampler, gradient, SR and Adam, and the sharded call at world 1 (NCCL)
and world 2 (two threads, host all-gather: strided walk, distributed index). Sizes are small so the
instrumented run finishes in minutes.

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2408_07625_b200 as q  # noqa: E402
from paper_2408_07625_b200 import _lib, synthetic  # noqa: E402
from paper_2408_07625_b200.hamiltonian import _ptr  # noqa: E402


def join_case(n_qubits, n_e, n_terms, n_unq, hit_cap=None):
    if hit_cap:
        os.environ["QVMC_HIT_CAP"] = str(hit_cap)
    else:
        os.environ.pop("QVMC_HIT_CAP", None)
    H = synthetic.jw_hamiltonian(n_qubits, n_terms, seed=1)
    keys = synthetic.near_hf_keys(n_qubits, n_e, n_unq, seed=2)
    b = synthetic.sample_batch(keys, seed=3)
    rep = q.surrogate_energy(H, b)
    half = q.surrogate_energy(H, b, n_unq // 3, n_unq // 2, check=False)
    assert np.allclose(half.locals, rep.locals[n_unq // 3: n_unq // 2], rtol=0,
                       atol=1e-10 * max(1.0, np.abs(rep.locals).max()))
    p = q.loop_over_terms(keys, H)
    loc = q.local_energies(p, b, H)
    assert np.allclose(loc, rep.locals, rtol=0, atol=1e-9 * max(1.0, np.abs(loc).max()))
    e = np.ascontiguousarray(p.entries[: 5000], dtype=np.uint32)
    hh = np.zeros(len(e), dtype=np.complex128)
    kind = np.zeros(len(e), dtype=np.uint8)
    _lib.check(_lib.lib().qvmc_cuda_pair_elements_fused(H.device_handle(0), len(keys), _ptr(keys), len(e), _ptr(e),
                                                        _ptr(hh), _ptr(kind), _lib.MEM_HOST))
    print(f"join {n_qubits}q n={n_unq} pairs={len(p.entries)} e_var={rep.e_var:.6f}", flush=True)


def sharded_threads(world=2, n_unq=3000):
    """world ranks as threads of this process, each with its own device handle on cuda:0 and a
    host all-gather over a thread barrier: the strided walk, the distributed deletion index and
    the exact all-reduces of qvmc_cuda_eloc_sharded under the sanitizer in one process."""
    import ctypes as C
    import threading
    c, x, y, z = synthetic.jw_terms(56, 100_000, seed=1)
    keys = synthetic.near_hf_keys(56, 14, n_unq, seed=4)
    bb = synthetic.sample_batch(keys, seed=3)
    ref = q.surrogate_energy(q.HamiltonianIndex.from_masks(56, c, x, y, z), bb)
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
    Hs = [q.HamiltonianIndex.from_masks(56, c, x, y, z) for _ in range(world)]

    def run(rank):
        comm = C.c_void_p()
        _lib.check(L.qvmc_cuda_comm_init_host(world, rank, fns[rank], None, C.byref(comm)))
        r0, r1 = C.c_int64(), C.c_int64()
        _lib.check(L.qvmc_shard_bounds(n_unq, world, rank, C.byref(r0), C.byref(r1)))
        r0, r1 = r0.value, r1.value
        out = np.zeros(r1 - r0, dtype=np.complex128)
        mom = np.zeros(5)
        sl = lambda a: np.ascontiguousarray(a[r0:r1])
        _lib.check(L.qvmc_cuda_eloc_sharded(Hs[rank].device_handle(0), comm, n_unq, _ptr(sl(bb.vectors)),
                                            _ptr(sl(bb.log_amps)), _ptr(sl(bb.phases)), _ptr(sl(bb.log_probs)),
                                            bb.log_norm, _ptr(out), _ptr(mom), _lib.MEM_HOST))
        _lib.check(L.qvmc_cuda_comm_destroy(comm))
        outs[rank] = (r0, r1, out)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for r0, r1, out in outs:
        assert np.array_equal(out, ref.locals[r0:r1])
    print(f"sharded world {world} (threads, host all-gather): rows bit-identical", flush=True)


def main():
    import __graft_entry__
    __graft_entry__.smoke()
    from helpers import golden, instances, product_index
    g = golden("accept3")
    for _, pfx in instances("accept3")[:10]:
        H = product_index(g, pfx)
        keys = g[pfx + "keys"]
        q.loop_over_trie(keys, H)
        b = q.SampleBatch(keys, g[pfx + "lp"], g[pfx + "la"], g[pfx + "ph"], float(g[pfx + "norm"]),
                          float(g[pfx + "log_norm"]))
        q.surrogate_energy(H, b, check=False)
    join_case(118, 110, 300_000, 3000)
    join_case(118, 110, 300_000, 3000, hit_cap=512)
    join_case(56, 14, 100_000, 3000)
    # minority set of 24: the join with 276 buckets per row, and the sector-list row kernel (QVMC_JOIN=0)
    keys = synthetic.near_hf_keys(48, 24, 1000, seed=2)
    H = synthetic.jw_hamiltonian(48, 20_000, seed=1)
    q.surrogate_energy(H, synthetic.sample_batch(keys, seed=3))
    os.environ["QVMC_JOIN"] = "0"
    H = synthetic.jw_hamiltonian(48, 20_000, seed=1)
    q.surrogate_energy(H, synthetic.sample_batch(keys, seed=3))
    os.environ.pop("QVMC_JOIN")
    # half filling at 64 qubits: s = 32, the join's largest tables (496 buckets per row)
    H = synthetic.jw_hamiltonian(64, 30_000, seed=1)
    q.surrogate_energy(H, synthetic.sample_batch(synthetic.near_hf_keys(64, 32, 800, seed=2), seed=3))
    # amplitude model
    M = q.AnqsModel(q.QuditLayout.make(56, 6), q.SectorConstraint(14, True))
    M.set_params(np.random.default_rng(0).uniform(-0.1, 0.1, M.n_params()))
    keys = synthetic.near_hf_keys(56, 14, 2000, seed=2)
    M.log_psi(keys)
    # sampler, energy gradient, SR, Adam (round 2)
    b = q.sample_without_replacement(M, 3000, q.CounterRng(5), 1)
    q.fill_amplitudes(b, M)
    w = np.exp(b.log_probs - b.log_norm)
    loc = np.random.default_rng(1).normal(size=b.size()) + 0j
    grad = M.energy_gradient(b.vectors, w, loc)
    d, _ = M.sr_direction(b.vectors, b.log_probs, loc, 64, grad)
    M.adam_step(d)
    print(f"model paths: sampled {b.size()}, |grad| {np.linalg.norm(grad):.4f}", flush=True)
    # sharded path through the C ABI, world 1 over NCCL
    import ctypes as C
    H = synthetic.jw_hamiltonian(56, 100_000, seed=1)
    keys = synthetic.near_hf_keys(56, 14, 3000, seed=2)
    bb = synthetic.sample_batch(keys, seed=3)
    L = _lib.lib()
    uid = (C.c_uint8 * 128)()
    _lib.check(L.qvmc_cuda_comm_unique_id(uid, 128))
    comm = C.c_void_p()
    _lib.check(L.qvmc_cuda_comm_init_nccl(0, 1, 0, uid, C.byref(comm)))
    out = np.zeros(len(keys), dtype=np.complex128)
    mom = np.zeros(5)
    _lib.check(L.qvmc_cuda_eloc_sharded(H.device_handle(0), comm, len(keys), _ptr(bb.vectors), _ptr(bb.log_amps),
                                        _ptr(bb.phases), _ptr(bb.log_probs), bb.log_norm, _ptr(out), _ptr(mom),
                                        _lib.MEM_HOST))
    _lib.check(L.qvmc_cuda_comm_destroy(comm))
    sharded_threads(2)
    print("sanitize driver done", flush=True)


if __name__ == "__main__":
    main()
