"""Parity at the configurations bench.py measures (1e6 unique samples).

The benched workloads (c118: 118 q, 3e6 strings; c56: 56 q, 3e5 strings;
both 1e6 near-HF samples) are checked against the C oracle
(oracle/qvmc_oracle.c, pinned to the reference by test_oracle.py) on sampled
rows against the WHOLE 1e6 sample set:

  * the (x, x', xy) pair list of every sampled row, bit-exact, between the
    materialised device path (qvmc_cuda_pairs) and the oracle's
    LoopOverTerms restatement (coupling.cpp:62-84 + the canonical flatten
    :37-58); per-row pair counts equal;
  * the fused path's pair count (no materialisation) equals the
    materialised total;
  * E_loc of the fused path (qvmc_cuda_eloc_fused) within 1e-10 of the
    absolute-sum scale of the oracle's (energy.cpp:13-48);
  * per-pair H_{xx'} through the fused path's own evaluators
    (qvmc_cuda_pair_elements_fused: drain-record kinds A/B, the diagonal
    quadratic form) against group_element (hamiltonian.cpp:186-194): kind A
    bit-exact, the family / quadratic forms within 1e-12 of the group's
    absolute coefficient sum;
  * the energy moments and the variance against a restatement over the
    oracle's rows.

Rows checked: 256 uniformly drawn + the 16 rows with the most pairs + the
first 16 (these two sets may overlap), at least 272 per configuration.
"""
import numpy as np
import pytest

import oracle
import paper_2408_07625_b200 as q
from paper_2408_07625_b200 import _lib, synthetic
from paper_2408_07625_b200.hamiltonian import _ptr
from helpers import assert_eloc_close, group_abs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CONFIGS = {"c118": (118, 110, 3_000_000), "c56": (56, 14, 300_000)}
N_UNQ = 1_000_000


def _rows_of(entries: np.ndarray, rows: np.ndarray):
    """Canonical pair list restricted to `rows` (ascending), with per-row counts."""
    x = entries[:, 0]
    lo = np.searchsorted(x, rows, side="left")
    hi = np.searchsorted(x, rows, side="right")
    parts = [entries[a:b] for a, b in zip(lo, hi)]
    return (np.concatenate(parts) if parts else entries[:0]), (hi - lo)


@pytest.fixture(scope="module", params=sorted(CONFIGS))
def benched(request, cuda_ok):
    n_qubits, n_e, n_terms = CONFIGS[request.param]
    c, x, y, z = synthetic.jw_terms(n_qubits, n_terms, seed=1)
    H = q.HamiltonianIndex.from_masks(n_qubits, c, x, y, z)
    O = oracle.OracleIndex(n_qubits, c, x, y, z)
    keys = synthetic.near_hf_keys(n_qubits, n_e, N_UNQ, seed=2)
    b = synthetic.sample_batch(keys, seed=3)
    fused = q.surrogate_energy(H, b)
    fused_stats = q.last_stats(H)
    pairs = q.loop_over_terms(keys, H).entries
    counts = np.bincount(pairs[:, 0].astype(np.int64), minlength=N_UNQ)
    rng = np.random.default_rng(n_qubits)
    fixed = np.unique(np.concatenate([np.arange(16), np.argsort(counts, kind="stable")[-16:]]))
    pool = np.setdiff1d(np.arange(N_UNQ), fixed)
    rows = np.sort(np.concatenate([fixed, rng.choice(pool, 256, replace=False)])).astype(np.int64)
    o_pairs, o_counts, o_eloc, o_scale = O.rows_list(keys, rows, b.log_amps, b.phases)
    return dict(name=request.param, H=H, O=O, keys=keys, b=b, fused=fused, fused_stats=fused_stats,
                pairs=pairs, counts=counts, rows=rows, o_pairs=o_pairs, o_counts=o_counts, o_eloc=o_eloc,
                o_scale=o_scale)


def test_pair_lists_bit_exact_on_sampled_rows(benched):
    d = benched
    assert len(d["rows"]) >= 256 + 16
    got, got_counts = _rows_of(d["pairs"], d["rows"])
    assert np.array_equal(got_counts, d["o_counts"])
    assert np.array_equal(got, d["o_pairs"])
    # excitation classes of the sampled pairs: popcount(x ^ x') = popcount(xy) in {0, 2, 4}
    xy = d["H"].xy[got[:, 2]]
    cls = np.array([sum(bin(int(w)).count("1") for w in r) for r in xy])
    kx = d["keys"][got[:, 0]] ^ d["keys"][got[:, 1]]
    assert np.array_equal(cls, np.array([sum(bin(int(w)).count("1") for w in r) for r in kx]))
    assert set(np.unique(cls)) <= {0, 2, 4}


def test_fused_pair_count_matches_materialised(benched):
    d = benched
    assert d["fused_stats"]["pairs"] == len(d["pairs"])
    assert d["fused_stats"]["rows"] == N_UNQ and d["fused_stats"]["join_mode"] == 1


def test_fused_eloc_matches_oracle_on_sampled_rows(benched):
    d = benched
    worst = assert_eloc_close(d["fused"].locals[d["rows"]], d["o_eloc"], d["o_scale"])
    assert worst <= 1e-10


def test_fused_evaluators_match_group_element(benched):
    """Drain-record kinds A/B and the diagonal quadratic form, per pair, vs
    the oracle's group_element (hamiltonian.cpp:186-194)."""
    d = benched
    H, O, keys = d["H"], d["O"], d["keys"]
    sub, _ = _rows_of(d["pairs"], d["rows"])
    e = np.ascontiguousarray(sub, dtype=np.uint32)
    hh = np.zeros(len(e), dtype=np.complex128)
    kind = np.zeros(len(e), dtype=np.uint8)
    _lib.check(_lib.lib().qvmc_cuda_pair_elements_fused(H.device_handle(0), len(keys), _ptr(keys), len(e), _ptr(e),
                                                        _ptr(hh), _ptr(kind), _lib.MEM_HOST))
    want = np.array([O.group_element(keys[j], g) for (_, j, g) in e], dtype=np.complex128)
    gabs = group_abs(H.group_offsets, H.coeff)[e[:, 2].astype(np.int64)]
    kinds = {int(k): int((kind == k).sum()) for k in np.unique(kind)}
    assert kinds.get(0, 0) > 0 and kinds.get(1, 0) > 0 and kinds.get(5, 0) == len(d["rows"]), kinds
    exact = (kind == 0) | (kind == 4)
    assert np.array_equal(hh[exact], want[exact])  # kind A and term by term: bit-identical
    err = np.abs(hh - want) / np.maximum(gabs, 1e-300)
    assert err.max() <= 1e-12, (float(err.max()), kinds)


def test_moments_and_variance(benched):
    """Moments of the fused call vs the oracle-row restatement: the weighted
    sums over the sampled rows (same E_loc) and the variance formula."""
    d = benched
    b, fused = d["b"], d["fused"]
    w = np.exp(b.log_probs - b.log_norm)
    e = fused.locals
    # full-set moments from the device E_loc, restated in numpy
    e0 = np.sum(w * e)
    assert abs(fused.e_var - e0.real) <= 1e-10 * max(1.0, np.sum(w * np.abs(e)))
    var = float(np.sum(w * np.abs(e - e0) ** 2))
    assert abs(fused.variance - var) <= 1e-9 * max(1.0, float(np.sum(w * np.abs(e) ** 2)))
    assert abs(fused.ipr - float(np.sum(w * w))) <= 1e-12
    # the sampled rows' contribution with the oracle's E_loc
    r = d["rows"]
    sw = np.sum(w[r] * np.abs(e[r]) ** 2)
    so = np.sum(w[r] * np.abs(d["o_eloc"]) ** 2)
    assert abs(sw - so) <= 1e-9 * max(1.0, so)
