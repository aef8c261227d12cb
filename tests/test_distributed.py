"""Multi-rank plumbing of distributed.sharded_surrogate_energy, world size 2, gloo, CPU.

The product's per-rank step is the fused kernel; on a CPU host the test
injects the oracle as the per-shard evaluator and checks what the plumbing
adds: uneven shards are all-gathered into exactly the full sample set, each
rank evaluates exactly its own rows, and the moments all-reduce to the
unsharded values.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    from paper_2408_07625_b200 import synthetic
    c, x, y, z = synthetic.jw_terms(12, 900, seed=1)
    keys = synthetic.sector_keys(12, 6, spin_balanced=True)
    b = synthetic.sample_batch(keys, seed=3)
    return (c, x, y, z), b


def _oracle_evaluator(masks):
    import oracle
    O = oracle.OracleIndex(12, *masks)

    def run(keys, la, ph, lp, log_norm, r0, r1, out_locals, out_moments):
        k = keys.numpy().view(np.uint64)
        loc, _ = O.eloc_rows(k, la.numpy(), ph.numpy(), r0, r1, threads=1)
        out_locals[: r1 - r0] = torch.from_numpy(loc)
        w = np.exp(lp.numpy()[r0:r1] - log_norm)
        out_moments[:] = torch.tensor([np.sum(w * loc.real), np.sum(w * loc.imag), np.sum(w * w), np.sum(w),
                                       np.sum(w * np.abs(loc) ** 2)])

    return run


def _worker(rank, world, port, splits, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2408_07625_b200.distributed import Shard, sharded_surrogate_energy
        masks, b = _problem()
        r0, r1 = splits[rank], splits[rank + 1]
        sh = Shard(torch.from_numpy(b.vectors[r0:r1].view(np.int64).copy()), torch.from_numpy(b.log_amps[r0:r1].copy()),
                   torch.from_numpy(b.phases[r0:r1].copy()), torch.from_numpy(b.log_probs[r0:r1].copy()))
        res = sharded_surrogate_energy(sh, b.log_norm, _oracle_evaluator(masks), gather_locals=True)
        out_q.put((rank, res.row_begin, res.row_end, res.n_total, res.locals.numpy(), res.moments.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("splits", [[0, 200, 400], [0, 123, 400]])
def test_two_rank_sharding_matches_unsharded(splits):
    import oracle
    masks, b = _problem()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, splits, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    O = oracle.OracleIndex(12, *masks)
    full, _ = O.eloc_rows(b.vectors, b.log_amps, b.phases, 0, 400, threads=1)
    w = np.exp(b.log_probs - b.log_norm)
    for rank, r0, r1, n_total, locals_, moments in outs:
        assert (r0, r1, n_total) == (splits[rank], splits[rank + 1], 400)
        assert np.array_equal(locals_, full)  # gathered rows in global order
        assert abs(moments[0] - np.sum(w * full.real)) <= 1e-12 * max(1.0, np.sum(w * np.abs(full)))
        assert abs(moments[3] - 1.0) <= 1e-12
    assert np.array_equal(outs[0][5], outs[1][5])  # every rank holds the same reduced moments


def test_shard_bounds_cover_rows():
    from paper_2408_07625_b200.distributed import shard_bounds
    for n in (1, 7, 1000, 1_000_000):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
