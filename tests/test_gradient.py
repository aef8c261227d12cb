"""Gradient consumers of the local energies.

energy_gradient (proj/src/energy.cpp:80-107) over the rows of
batched_grad_log_psi (proj/src/model.cpp:273-336), as run_optimisation
streams them (optimizer.cpp:105-140). Golden data = the UNMODIFIED reference
(tests/golden/grad.npz, generator tests/golden/make_grad_golden.py). Bar:
fp64, 1e-10 relative to the gradient's max entry (the device contracts the
rows with DGEMMs in a different summation order). CPU tests pin the numpy
restatement (oracle/model_oracle.py) to the same goldens.
"""
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from make_model_golden import model_params  # noqa: E402

G = np.load(Path(__file__).resolve().parent / "golden" / "grad.npz")
NAMES = ["s8", "s12", "r20", "h56", "h118"]


def _cfg(name):
    n, bits, ne, spin, hidden, pseed = (int(v) for v in G[f"{name}_cfg"])
    return n, bits, ne, bool(spin), hidden, model_params((n, bits, hidden), seed=pseed)


def _check(name, g):
    scale = max(1.0, float(G[f"{name}_gnorm"][0]))
    if f"{name}_grad" in G:
        want = G[f"{name}_grad"]
        assert np.abs(g - want).max() <= 1e-10 * scale
    else:
        assert np.abs(g[G[f"{name}_gcols"]] - G[f"{name}_grad_at"]).max() <= 1e-10 * scale
    assert abs(np.linalg.norm(g) - G[f"{name}_gnorm"][0]) <= 1e-10 * scale


@pytest.mark.parametrize("name", ["s8", "s12", "r20"])
def test_oracle_gradient_matches_reference(name):
    from oracle.model_oracle import ModelOracle, energy_gradient, grad_log_psi
    n, bits, ne, spin, hidden, p = _cfg(name)
    O = ModelOracle(n, bits, ne, spin, hidden, p)
    keys = G[f"{name}_keys"]
    J = grad_log_psi(O, keys)
    assert np.abs(J[:8, G[f"{name}_jcols"]] - G[f"{name}_jac"]).max() <= 1e-12
    assert np.abs(np.linalg.norm(J[:8], axis=1) - G[f"{name}_jnorm"]).max() <= 1e-12
    _check(name, energy_gradient(G[f"{name}_w"], G[f"{name}_loc"], J))


def _model(name):
    import paper_2408_07625_b200 as q
    n, bits, ne, spin, hidden, p = _cfg(name)
    M = q.AnqsModel(q.QuditLayout.make(n, bits), q.SectorConstraint(ne, spin), hidden)
    M.set_params(p)
    return M


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_energy_gradient_matches_reference(cuda_ok, name):
    M = _model(name)
    g = M.energy_gradient(G[f"{name}_keys"], G[f"{name}_w"], G[f"{name}_loc"])
    _check(name, g)
    again = M.energy_gradient(G[f"{name}_keys"], G[f"{name}_w"], G[f"{name}_loc"])
    assert np.array_equal(g, again)  # deterministic


@pytest.mark.gpu
def test_device_energy_gradient_chunked_and_masked(cuda_ok):
    """More samples than one 32768-row chunk (accumulated over chunks) agree with the
    numpy restatement on a subset-weighted problem; a masked key raises like
    grad_log_psi (model.cpp:274-275)."""
    import paper_2408_07625_b200 as q
    from oracle.model_oracle import ModelOracle, energy_gradient, grad_log_psi
    from paper_2408_07625_b200 import synthetic
    n, bits, ne, spin, hidden, p = _cfg("r20")
    M = _model("r20")
    keys = synthetic.random_sector_keys(n, ne, 70_000, seed=9)
    rng = np.random.default_rng(1)
    w = np.zeros(len(keys))
    hot = rng.choice(len(keys), 300, replace=False)  # nonzero weights only on rows the oracle evaluates
    w[hot] = rng.uniform(0.1, 1.0, 300)
    w /= w.sum()
    loc = rng.normal(size=len(keys)) + 0.1j * rng.normal(size=len(keys))
    g = M.energy_gradient(keys, w, loc)
    O = ModelOracle(n, bits, ne, spin, hidden, p)
    mean = (w * loc).sum()
    hot.sort()
    J = grad_log_psi(O, keys[hot])
    c = w[hot] * (loc[hot] - mean)
    want = 2.0 * (c.real @ J.real - c.imag @ J.imag)
    assert np.abs(g - want).max() <= 1e-10 * max(1.0, np.abs(want).max())
    bad = keys[:5].copy()
    bad[0, 0] ^= np.uint64(1)
    with pytest.raises(ValueError, match="masked"):
        M.energy_gradient(bad, np.full(5, 0.2), np.ones(5, dtype=complex))
