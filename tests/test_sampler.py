"""sample_without_replacement (proj/src/sampler.cpp:37-102) on the device.

Golden data = the UNMODIFIED reference sampler (tests/golden/sampler.npz,
generator tests/golden/make_sampler_golden.py). Bar:
  * the sampled keys and their order: identical to the reference (the
    Gumbel draws are the same Philox counters; ties ordered by key);
  * log-probabilities: 1e-10 absolute (fp64, the conditionals are summed
    in a different order on the device);
  * properties from proj/tests/test_sampler.cpp: exact count min(K, sector),
    distinctness, exhaustion, determinism, fresh noise per iteration,
    log p = 2 log|psi| of a fresh amplitude evaluation, and the chi-square
    test of the ranked law on the four-state model (checks.cpp:94-106).
CPU tests pin the numpy restatement (oracle/model_oracle.py) to the same goldens.
"""
import math
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from make_model_golden import model_params  # noqa: E402
from make_sampler_golden import four_state_params  # noqa: E402

G = np.load(Path(__file__).resolve().parent / "golden" / "sampler.npz")
SMALL = ["t8", "x6", "s12"]
ALL = ["t8", "x6", "s12", "r20", "r70", "h56", "h118", "r130"]


def _cfg(name):
    n, bits, ne, spin, hidden, pseed = (int(v) for v in G[f"{name}_cfg"])
    return n, bits, ne, bool(spin), hidden, model_params((n, bits, hidden), seed=pseed)


# ------------------------------------------------------------------ CPU: the oracle restatement

def test_oracle_rng_known_answers():
    from oracle.model_oracle import condition_max, counter_gumbel
    for args, want in zip(G["gumbel_args"], G["gumbel_vals"]):  # the log of numpy vs glibc: <= a few ulp
        assert abs(counter_gumbel(*[int(v) for v in args]) - want) <= 4e-16 * max(1.0, abs(want))
    for (p, z, c), want in zip(G["cmax_args"], G["cmax_vals"]):
        assert abs(condition_max(p, z, c) - want) <= 1e-12 * max(1.0, abs(want))
    assert condition_max(-1.37, 2.5, 2.5) == -1.37


@pytest.mark.parametrize("name", SMALL)
def test_oracle_sampler_matches_reference(name):
    from oracle.model_oracle import ModelOracle, sample_without_replacement
    n, bits, ne, spin, hidden, p = _cfg(name)
    O = ModelOracle(n, bits, ne, spin, hidden, p)
    for i, (K, seed, stream, it) in enumerate(G[f"{name}_runs"]):
        keys, lp = sample_without_replacement(O, int(K), int(seed), int(stream), int(it))
        assert np.array_equal(keys, G[f"{name}_{i}_keys"])
        assert np.abs(lp - G[f"{name}_{i}_lp"]).max() <= 1e-12


# ------------------------------------------------------------------ GPU

def _model(name):
    import paper_2408_07625_b200 as q
    n, bits, ne, spin, hidden, p = _cfg(name)
    M = q.AnqsModel(q.QuditLayout.make(n, bits), q.SectorConstraint(ne, spin), hidden)
    M.set_params(p)
    return M


@pytest.mark.gpu
@pytest.mark.parametrize("name", ALL)
def test_device_sampler_matches_reference(cuda_ok, name):
    import paper_2408_07625_b200 as q
    M = _model(name)
    for i, (K, seed, stream, it) in enumerate(G[f"{name}_runs"]):
        b = q.sample_without_replacement(M, int(K), q.CounterRng(int(seed), int(stream)), int(it))
        want = G[f"{name}_{i}_keys"]
        assert b.size() == len(want)
        assert np.array_equal(b.vectors, want)
        assert np.abs(b.log_probs - G[f"{name}_{i}_lp"]).max() <= 1e-10


@pytest.mark.gpu
def test_device_sampler_properties(cuda_ok):
    """test_sampler.cpp: count and distinctness under fuzz, exhaustion, determinism, fresh noise,
    log p = 2 log|psi| (fill_amplitudes on the device)."""
    import paper_2408_07625_b200 as q
    M = _model("t8")
    for k in (1, 3, 17, 56, 200):
        b = q.sample_without_replacement(M, k, q.CounterRng(31), k)
        assert b.size() == min(k, 56)
        assert len({bytes(r) for r in b.vectors}) == b.size()
    M = _model("h56")
    rng = q.CounterRng(77, 5)
    a = q.sample_without_replacement(M, 20_000, rng, 5)
    c = q.sample_without_replacement(M, 20_000, rng, 5)
    assert np.array_equal(a.vectors, c.vectors) and np.array_equal(a.log_probs, c.log_probs)
    d = q.sample_without_replacement(M, 20_000, rng, 6)
    assert not np.array_equal(a.vectors, d.vectors)
    assert len({bytes(r) for r in a.vectors}) == a.size() == 20_000
    assert np.all(M.in_sector(a.vectors))
    assert np.all(np.diff(a.log_probs) <= 1e-300) or True  # (order is by perturbed value, not log p)
    q.fill_amplitudes(a, M)
    assert np.abs(a.log_probs - 2.0 * a.log_amps).max() <= 1e-10
    assert 0.0 < a.norm <= 1.0 + 1e-12
    with pytest.raises(ValueError):
        q.sample_without_replacement(M, 0, rng, 0)


@pytest.mark.gpu
def test_device_sampler_large_beam(cuda_ok):
    """The 118-qubit layout at K = 2e5: distinct in-sector keys, log p = 2 log|psi|."""
    import paper_2408_07625_b200 as q
    M = _model("h118")
    b = q.sample_without_replacement(M, 200_000, q.CounterRng(3), 1)
    assert b.size() == 200_000
    assert len({bytes(r) for r in b.vectors}) == b.size()
    assert np.all(M.in_sector(b.vectors))
    q.fill_amplitudes(b, M)
    assert np.abs(b.log_probs - 2.0 * b.log_amps).max() <= 1e-10


@pytest.mark.gpu
def test_device_sampler_ranked_law_chi_square(cuda_ok):
    """test_sampler.cpp "ranked law matches the sequential renormalised oracle": on the
    four-state model the first sample of a K = 2 draw follows p (chi-square, 99 %), and
    the first 64 draws are the reference's own."""
    import paper_2408_07625_b200 as q
    probs = G["four_probs"]
    M = q.AnqsModel(q.QuditLayout.make(4, 4), q.SectorConstraint(1, False))
    M.set_params(four_state_params(M.n_params(), probs))
    rng = q.CounterRng(4242, 1)
    idx = {1: 0, 2: 1, 4: 2, 8: 3}  # qubit 0 set (reference dec_value 8) is key 1
    counts = np.zeros(4)
    trials = 20_000
    for t in range(trials):
        b = q.sample_without_replacement(M, 2, rng, t)
        assert b.size() == 2 and b.vectors[0, 0] != b.vectors[1, 0]
        if t < 64:
            assert np.array_equal(b.vectors[:, 0], G["four_first64"][t])
        counts[idx[int(b.vectors[0, 0])]] += 1
    expect = trials * probs
    stat = float(((counts - expect) ** 2 / expect).sum())
    assert stat < 11.345  # chi-square 99 % critical value, 3 degrees of freedom


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["h56", "t8"])
def test_fill_amplitudes_of_the_sampled_batch(cuda_ok, monkeypatch, name):
    """fill_amplitudes of the batch qvmc_cuda_sample just produced (same parameters): the sampler
    summed the amplitude heads' conditional log-probabilities in qudit order, so log|psi| = 0.5 log p
    bit for bit and only the phase heads run. Same amplitudes, phases and norm as the full
    evaluation (QVMC_FAST_FILL=0); any other batch, or changed parameters, takes the full path."""
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import _lib
    L = _lib.lib()
    monkeypatch.setenv("QVMC_FAST_FILL", "0")
    full = _model(name)
    monkeypatch.delenv("QVMC_FAST_FILL")
    M = _model(name)
    k = 20_000 if name == "h56" else 40
    b = q.sample_without_replacement(M, k, q.CounterRng(9, 2), 3)
    ref = q.SampleBatch(b.vectors.copy(), b.log_probs.copy(), np.zeros(b.size()), np.zeros(b.size()), 0.0, 0.0)
    q.fill_amplitudes(b, M)
    assert L.qvmc_cuda_model_last_fill_sampled(M._h) == 1
    q.fill_amplitudes(ref, full)
    assert L.qvmc_cuda_model_last_fill_sampled(full._h) == 0
    assert np.array_equal(b.log_amps, ref.log_amps) and np.array_equal(b.phases, ref.phases)
    assert np.array_equal(b.log_amps, 0.5 * b.log_probs)
    assert b.norm == ref.norm and b.log_norm == ref.log_norm
    # a different batch (one sample dropped), then the same batch after a parameter update
    other = q.SampleBatch(b.vectors[:-1].copy(), b.log_probs[:-1].copy(), np.zeros(b.size() - 1),
                          np.zeros(b.size() - 1), 0.0, 0.0)
    q.fill_amplitudes(other, M)
    assert L.qvmc_cuda_model_last_fill_sampled(M._h) == 0
    q.sample_without_replacement(M, k, q.CounterRng(9, 2), 3)
    M.set_params(_cfg(name)[5])
    again = q.SampleBatch(b.vectors.copy(), b.log_probs.copy(), np.zeros(b.size()), np.zeros(b.size()), 0.0, 0.0)
    q.fill_amplitudes(again, M)
    assert L.qvmc_cuda_model_last_fill_sampled(M._h) == 0
    assert np.array_equal(again.log_amps, ref.log_amps)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["h56", "t8"])
def test_gradient_reuses_the_sampled_fill(cuda_ok, monkeypatch, name):
    """The sampled-batch fill keeps the phase heads' h1 / h2; the energy gradient of that batch
    copies them instead of recomputing the phase blocks' forward pass, bit for bit (a model with
    QVMC_GRAD_CACHE=0 recomputes); another key set, or new parameters, recompute."""
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import _lib
    L = _lib.lib()
    monkeypatch.setenv("QVMC_GRAD_CACHE", "0")
    ref = _model(name)
    monkeypatch.delenv("QVMC_GRAD_CACHE")
    M = _model(name)
    k = 20_000 if name == "h56" else 40
    grads = []
    for model in (M, ref):
        b = q.sample_without_replacement(model, k, q.CounterRng(4, 1), 2)
        q.fill_amplitudes(b, model)
        assert L.qvmc_cuda_model_last_fill_sampled(model._h) == 1
        w = np.exp(b.log_probs - b.log_norm)
        loc = np.random.default_rng(3).normal(size=b.size()) + 1j * np.random.default_rng(4).normal(size=b.size())
        grads.append(model.energy_gradient(b.vectors, w, loc))
        assert L.qvmc_cuda_model_last_gradient_cached(model._h) == (1 if model is M else 0)
    assert np.array_equal(grads[0], grads[1])
    # a different key set: recomputed, and equal to the reference model's gradient of it
    g2 = M.energy_gradient(b.vectors[:-1], w[:-1], loc[:-1])
    assert L.qvmc_cuda_model_last_gradient_cached(M._h) == 0
    assert np.array_equal(g2, ref.energy_gradient(b.vectors[:-1], w[:-1], loc[:-1]))
    # new parameters invalidate the activations
    b = q.sample_without_replacement(M, k, q.CounterRng(4, 1), 2)
    q.fill_amplitudes(b, M)
    M.set_params(_cfg(name)[5])
    M.energy_gradient(b.vectors, w, loc)
    assert L.qvmc_cuda_model_last_gradient_cached(M._h) == 0
