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


def _amp_worker(rank, world, port, splits, out_q):
    """sharded_fill_amplitudes with the model oracle as the per-shard evaluator, then
    sharded_surrogate_energy on the amplitudes it produced."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.model_oracle import ModelOracle
        from paper_2408_07625_b200.distributed import Shard, sharded_fill_amplitudes, sharded_surrogate_energy
        masks, b = _problem()
        p = np.random.default_rng(4).uniform(-0.2, 0.2, ModelOracle(12, 6, 6, True, 64, np.zeros(36608)).n_params)
        O = ModelOracle(12, 6, 6, True, 64, p)

        def evaluate(keys, out_la, out_ph):
            la, ph = O.log_psi(keys.numpy().view(np.uint64))
            out_la.copy_(torch.from_numpy(la))
            out_ph.copy_(torch.from_numpy(ph))

        r0, r1 = splits[rank], splits[rank + 1]
        lp = b.log_probs[r0:r1].copy()
        sh = Shard(torch.from_numpy(b.vectors[r0:r1].view(np.int64).copy()), torch.zeros(r1 - r0, dtype=torch.float64),
                   torch.zeros(r1 - r0, dtype=torch.float64), torch.from_numpy(lp))
        log_norm = sharded_fill_amplitudes(sh, evaluate)
        res = sharded_surrogate_energy(sh, log_norm, _oracle_evaluator(masks), gather_locals=True)
        out_q.put((rank, log_norm, sh.log_amps.numpy(), sh.phases.numpy(), res.locals.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("splits", [[0, 200, 400], [0, 0, 400], [0, 311, 400]])
def test_two_rank_fill_amplitudes_matches_unsharded(splits):
    """Rows are independent: each rank's log|psi|/phase equal the unsharded oracle's rows, the
    merged log_norm equals the single-process logsumexp (sampler.cpp:114-119), and the chained
    E_loc matches the unsharded E_loc on those amplitudes (an empty shard included)."""
    import oracle
    from oracle.model_oracle import ModelOracle
    masks, b = _problem()
    p = np.random.default_rng(4).uniform(-0.2, 0.2, ModelOracle(12, 6, 6, True, 64, np.zeros(36608)).n_params)
    O = ModelOracle(12, 6, 6, True, 64, p)
    la, ph, _, log_norm = O.fill_amplitudes(b.vectors, b.log_probs)
    full, _ = oracle.OracleIndex(12, *masks).eloc_rows(b.vectors, la, ph, 0, 400, threads=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_amp_worker, args=(r, 2, port, splits, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    outs = sorted(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, ln, la_r, ph_r, locals_ in outs:
        r0, r1 = splits[rank], splits[rank + 1]
        assert np.array_equal(la_r, la[r0:r1]) and np.array_equal(ph_r, ph[r0:r1])
        assert abs(ln - log_norm) <= 1e-13 * max(1.0, abs(log_norm))
        assert np.allclose(locals_, full, rtol=0, atol=1e-12)
    assert outs[0][1] == outs[1][1]
