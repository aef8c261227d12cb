"""Stochastic reconfiguration on the device (the step after the gradient).

top_probability_indices, build_sr_context, sr_direction (proj/src/sr.cpp:15-95)
as run_optimisation chains them (optimizer.cpp:105-143). sr.cpp needs Eigen's
eigensolver, which this image lacks, so the numpy restatement
(oracle/model_oracle.py) is pinned the way the reference pins its own
implementation: against the dense regularised solve (Re S + lambda I) delta
= grad (checks.cpp "SR solve") and the cases of test_energy_sr.cpp:214-300
(push-through identity, lambda -> inf limit, tie order of the selection, the
ill-conditioned bowl, the condition-number error). The device path is then
held to the restatement: 1e-9 relative (fp64; GEMM and eigensolver orders
differ).
"""
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from make_model_golden import model_params  # noqa: E402

from oracle.model_oracle import build_sr_context, sr_direction, top_probability_indices  # noqa: E402


def test_restatement_is_the_dense_regularised_solve():
    rng = np.random.default_rng(3)
    for n, P in ((3, 6), (8, 40), (25, 300)):
        rows = rng.normal(size=(n, P)) + 1j * rng.normal(size=(n, P))
        lp = np.log(rng.uniform(0.1, 1.0, n))
        loc = rng.normal(size=n) + 0.3j * rng.normal(size=n)
        grad = rng.normal(size=P)
        S, _, lam = build_sr_context(lp, loc, np.arange(n), rows, 0.0)
        d = sr_direction(S, lam, grad)
        dense = np.linalg.solve(S.T @ S + lam * np.eye(P), grad)
        assert np.abs(d - dense).max() <= 1e-10 * max(1.0, np.abs(dense).max())


def test_restatement_reference_cases():
    """test_energy_sr.cpp:232-300."""
    rng = np.random.default_rng(1)
    rows = rng.uniform(-1, 1, (3, 6)) + 1j * rng.uniform(-1, 1, (3, 6))
    S, _, lam = build_sr_context(np.log([0.5, 0.3, 0.2]), np.array([0.4, -0.2, 0.9], dtype=complex), np.arange(3),
                                 rows, 1e9)
    g = np.array([1.0, -2, 3, -4, 5, -6])
    assert np.linalg.norm(sr_direction(S, lam, g) * 1e9 - g) < 1e-5 * np.linalg.norm(g)
    assert list(top_probability_indices(np.log([0.3, 0.4, 0.3]), 2)) == [1, 0]
    bad = np.zeros((4, 3))
    bad[0, 0] = 1e6
    with pytest.raises(RuntimeError, match="cond"):
        sr_direction(bad, 1e-18, np.ones(3))


def _bowl(solve):
    """test_energy_sr.cpp:263-288: SR descends at least as fast on an ill-conditioned bowl."""
    a = np.diag([10.0, 0.1])
    S = np.zeros((4, 2))
    S[0, 0], S[1, 1] = np.sqrt(10.0), np.sqrt(0.1)
    x_sr = np.ones(2)
    x_plain = np.ones(2)
    f = lambda x: 0.5 * x @ a @ x  # noqa: E731
    for _ in range(50):
        x_sr = x_sr - 0.19 * solve(S, 1e-2, a @ x_sr)
        x_plain = x_plain - 0.19 * (a @ x_plain)
        assert f(x_sr) <= f(x_plain) + 1e-12


def test_restatement_bowl():
    _bowl(sr_direction)


# ------------------------------------------------------------------ GPU

def _model(n, bits, ne, spin, pseed):
    import paper_2408_07625_b200 as q
    M = q.AnqsModel(q.QuditLayout.make(n, bits), q.SectorConstraint(ne, spin))
    M.set_params(model_params((n, bits, 64), seed=pseed))
    return M


@pytest.mark.gpu
def test_device_sr_solve(cuda_ok):
    M = _model(8, 3, 3, False, 401)
    rng = np.random.default_rng(5)
    for r, c in ((6, 6), (32, 500), (200, 20_000)):
        S = rng.normal(size=(r, c))
        g = rng.normal(size=c)
        want = sr_direction(S, 0.07, g)
        got = M.sr_solve(S, 0.07, g)
        assert np.abs(got - want).max() <= 1e-9 * max(1.0, np.abs(want).max())
    _bowl(lambda S, lam, g: M.sr_solve(S, lam, g))
    bad = np.zeros((4, 3))
    bad[0, 0] = 1e6
    with pytest.raises(RuntimeError, match="cond"):
        M.sr_solve(bad, 1e-18, np.ones(3))
    S = rng.normal(size=(6, 6))
    g = np.array([1.0, -2, 3, -4, 5, -6])
    assert np.linalg.norm(M.sr_solve(S, 1e9, g) * 1e9 - g) < 1e-5 * np.linalg.norm(g)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(20, 6, 10, False, 403, 300, 64), (56, 6, 14, True, 404, 2000, 100),
                                 (118, 6, 110, False, 405, 1000, 40)])
def test_device_sr_step_matches_restatement(cuda_ok, cfg):
    """The whole SR step: selection (with a forced tie), Jacobian rows, context, solve."""
    from oracle.model_oracle import ModelOracle, grad_log_psi
    from paper_2408_07625_b200 import synthetic
    n, bits, ne, spin, pseed, count, n_sr = cfg
    M = _model(n, bits, ne, spin, pseed)
    keys = synthetic.near_hf_keys(n, ne, count, seed=7) if n > 20 else synthetic.random_sector_keys(n, ne, count, 7)
    rng = np.random.default_rng(pseed)
    la, _ = M.log_psi(keys)
    lp = 2.0 * la
    lp[5] = lp[3]  # a tie: sample order decides (sr.cpp:17-21)
    loc = rng.normal(size=len(keys)) - 2.0 + 0.1j * rng.normal(size=len(keys))
    w = np.exp(lp - lp.max())
    w /= w.sum()
    grad = M.energy_gradient(keys, w, loc)
    got, lam = M.sr_direction(keys, lp, loc, n_sr, grad)
    sel = top_probability_indices(lp, n_sr)
    O = ModelOracle(n, bits, ne, spin, 64, model_params((n, bits, 64), seed=pseed))
    S, _, lam_o = build_sr_context(lp, loc, sel, grad_log_psi(O, keys[sel]), 0.0)
    assert abs(lam - lam_o) <= 1e-10 * lam_o
    want = sr_direction(S, lam_o, grad)
    assert np.abs(got - want).max() <= 1e-8 * max(1.0, np.abs(want).max())
    got2, _ = M.sr_direction(keys, lp, loc, n_sr, grad, lam=0.5)
    want2 = sr_direction(S, 0.5, grad)
    assert np.abs(got2 - want2).max() <= 1e-8 * max(1.0, np.abs(want2).max())


def _adam_ref(theta, m, v, t, d, lr, b1, b2, eps):
    """adam_step (optimizer.cpp:17-31)."""
    t += 1
    c1, c2 = 1.0 - b1 ** t, 1.0 - b2 ** t
    m = b1 * m + (1.0 - b1) * d
    v = b2 * v + (1.0 - b2) * (d * d)
    return theta - lr * (m / c1) / (np.sqrt(v / c2) + eps), m, v, t


@pytest.mark.gpu
def test_device_adam_and_params_relayout(cuda_ok):
    """Three device Adam steps equal the reference formula; the kernels' layout refreshed on the
    device gives log psi identical (bit for bit) to a host set_params of the same vector."""
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import synthetic
    M = _model(56, 6, 14, True, 404)
    theta = M.params
    m = np.zeros_like(theta)
    v = np.zeros_like(theta)
    t = 0
    rng = np.random.default_rng(2)
    for _ in range(3):
        d = rng.normal(size=theta.size) * 1e-2
        M.adam_step(d, 1e-3, 0.9, 0.999, 1e-8)
        theta, m, v, t = _adam_ref(theta, m, v, t, d, 1e-3, 0.9, 0.999, 1e-8)
        assert np.abs(M.params - theta).max() <= 1e-15 * max(1.0, np.abs(theta).max())
    keys = synthetic.near_hf_keys(56, 14, 3000, seed=4)
    la, ph = M.log_psi(keys)
    H = _model(56, 6, 14, True, 404)
    H.set_params(M.params)
    la2, ph2 = H.log_psi(keys)
    assert np.array_equal(la, la2) and np.array_equal(ph, ph2)
    bad = np.zeros(theta.size)
    bad[7] = np.nan
    with pytest.raises(RuntimeError, match="non-finite"):
        M.adam_step(bad)
    assert np.array_equal(M.params, H.params)  # nothing updated
