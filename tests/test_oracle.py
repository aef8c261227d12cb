"""Pin the CPU oracle (oracle/qvmc_oracle.c) to the reference's own outputs.

Every comparison is against tests/golden/*.npz, which tests/golden/make_golden.py
produced by running the UNMODIFIED reference sources (oracle/_ref). Integer
outputs (grouping, pairs, ops) must match exactly; matrix elements are
compared bit-for-bit (same term order, exact +-c adds); E_loc within 1e-12 of
the absolute-sum scale (libm exp/sincos are the only difference).
"""
import math

import numpy as np
import pytest

import oracle
from helpers import eloc_scale, golden, instances, oracle_index

FAMILIES = ["coupling", "accept3", "checks"]


def _check_instance(g, p, eloc_tol=1e-12):
    O = oracle_index(g, p)
    assert O.n_xy == len(g[p + "xy"]) and O.n_terms == len(g[p + "coeff"]) and O.diag == int(g[p + "diag"])
    assert np.array_equal(O.xy, g[p + "xy"])
    assert np.array_equal(O.offsets.astype(np.uint64), g[p + "offsets"])
    assert np.array_equal(O.coeff, g[p + "coeff"])
    assert np.array_equal(O.yz, g[p + "yz"]) and np.array_equal(O.y_weight, g[p + "y_weight"])
    keys = g[p + "keys"]
    want = g[p + "pairs"]
    got, ops = O.pairs(keys, 0)
    assert np.array_equal(got, want)
    assert ops == int(g[p + "ops_terms"])
    got_b, ops_b = O.pairs(keys, 1)
    assert np.array_equal(got_b, want) and ops_b == int(g[p + "ops_batch"])
    h = np.array([O.group_element(keys[j], gg) for (_, j, gg) in want], dtype=np.complex128)
    assert np.array_equal(h, g[p + "pair_h"])
    loc = O.local_energies(keys, g[p + "la"], g[p + "ph"], want)
    scale = eloc_scale(want, g[p + "offsets"], g[p + "coeff"], g[p + "la"], len(keys))
    assert np.all(np.abs(loc - g[p + "eloc"]) <= eloc_tol * scale)
    rows, _ = O.eloc_rows(keys, g[p + "la"], g[p + "ph"], 0, len(keys), threads=2)
    assert np.array_equal(rows, loc)  # same order of operations
    st, m, w = oracle.variational_energy(g[p + "lp"], float(g[p + "norm"]), float(g[p + "log_norm"]), loc)
    ev = g[p + "evar"]
    assert st == 0
    assert abs(m[0] - ev[0]) <= 1e-12 * max(1.0, abs(ev[0]))
    assert abs(m[2] - ev[2]) <= 1e-12


@pytest.mark.parametrize("family", FAMILIES)
def test_oracle_matches_reference_random_families(family):
    g = golden(family)
    for _, p in instances(family):
        _check_instance(g, p)


@pytest.mark.parametrize("name", ["toy", "h2", "h4", "h6"])
def test_oracle_matches_reference_fixtures(name):
    g = golden("fixtures")
    # index arrays live under "<name>_", sector path arrays under "<name>_sector_"
    p, q = f"{name}_", f"{name}_sector_"
    merged = dict(g)
    for k in list(g):
        if k.startswith(q):
            merged[p + k[len(q):]] = g[k]
    _check_instance(merged, p)


def test_fixture_term_counts_match_reference_constants():
    # checks.cpp:35-40: toy 5, h2 15, h4 185, h6 919 terms
    g = golden("fixtures")
    for name, n in (("toy", 5), ("h2", 15), ("h4", 185), ("h6", 919)):
        assert len(g[f"{name}_coeff"]) == n


def test_toy_known_answers():
    """Paper toy (checks.cpp:46-69; test_coupling.cpp:89-107; test_energy_sr.cpp:51-67)."""
    g = golden("fixtures")
    assert [int(v[0]) for v in g["toy_xy"]] == [0, 5, 10, 6]  # dec {0, 10, 5, 6} in MSB-first order
    want = [[0, 0, 0], [0, 1, 2], [0, 2, 1], [1, 0, 2], [1, 1, 0], [2, 0, 1], [2, 2, 0]]
    assert g["toybatch_pairs"].tolist() == want
    O = oracle_index(g, "toy_")
    keys = np.array([[0b0011], [0b1001], [0b0110]], dtype=np.uint64)
    got, _ = O.pairs(keys, 1)
    assert got.tolist() == want
    la = np.array([math.log(2.0), 0.0, 0.0])
    ph = np.array([0.0, 0.0, math.pi])
    loc = O.local_energies(keys, la, ph, got)
    assert np.allclose(loc.real, [0.8, 0.6, 1.4], rtol=0, atol=1e-12)
    assert np.all(np.abs(loc.imag) < 1e-13)
    lp = np.log(np.array([4.0, 1.0, 1.0]) / 6.0)
    st, m, w = oracle.variational_energy(lp, 1.0, 0.0, loc)
    assert st == 0 and abs(m[0] - 5.2 / 6.0) < 1e-13 and abs(m[2] - 0.5) < 1e-12 and abs(w.sum() - 1) < 1e-12
    # matrix elements (test_hamiltonian.cpp:86-104)
    x0, x1, x2 = keys
    assert abs(O.matrix_element(x0, x0) - 0.8) < 1e-14
    assert abs(O.matrix_element(x0, x1) + 0.2) < 1e-14
    assert abs(O.matrix_element(x1, x1) - 1.0) < 1e-14
    assert O.matrix_element(x1, x2) == 0


def test_oracle_error_paths():
    O = oracle.OracleIndex(2, [0.7, 0.2], np.zeros((2, 1), np.uint64), np.zeros((2, 1), np.uint64),
                           np.array([[0], [1]], np.uint64))
    with pytest.raises(ValueError):
        O.pairs(np.array([[1], [1]], dtype=np.uint64))
    with pytest.raises(RuntimeError):
        O.local_energies(np.array([[1]], np.uint64), np.array([-np.inf]), np.array([0.0]),
                         np.array([[0, 0, 0]], np.uint32))
    st, _, _ = oracle.variational_energy(np.array([-800.0]), 0.0, -800.0, np.array([1.0 + 0j]))
    assert st == -3
    with pytest.raises(ValueError):  # overlapping masks
        oracle.OracleIndex(2, [1.0], np.array([[1]], np.uint64), np.array([[1]], np.uint64),
                           np.zeros((1, 1), np.uint64))


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref needs /root/reference at build time")
def test_reference_build_reproduces_goldens():
    """The compiled reference still reproduces the committed fixtures."""
    g = golden("fixtures")
    R = oracle.RefIndex.parse("qubits: 4\n0.9 IIII\n0.1 IZZI\n-0.2 XIXI\n-0.2 IXIX\n0.3 IYYI\n")
    assert np.array_equal(R.xy, g["toy_xy"]) and np.array_equal(R.coeff, g["toy_coeff"])
    e, ops, be = R.pairs(np.array([[0b0011], [0b1001], [0b0110]], np.uint64), backend=1)
    assert np.array_equal(e, g["toybatch_pairs"]) and ops == 9 and be == 1


@pytest.mark.parametrize("family", FAMILIES)
def test_oracle_row_list_matches_reference(family):
    """qo_rows_list (listed rows against the whole sample set, the checker of
    tests/test_gpu_fullsize.py) reproduces the reference's pairs and E_loc
    for rows in any order."""
    g = golden(family)
    for s, p in instances(family):
        O = oracle_index(g, p)
        keys = g[p + "keys"]
        n = len(keys)
        rows = np.random.default_rng(s).permutation(n)
        pr, cnt, e, sc = O.rows_list(keys, rows, g[p + "la"], g[p + "ph"], threads=3)
        parts = np.split(pr, np.cumsum(cnt)[:-1]) if n else []
        back = [None] * n
        for k, r in enumerate(rows):
            back[r] = parts[k]
        got = np.concatenate(back).reshape(-1, 3) if n else pr
        assert np.array_equal(got, g[p + "pairs"].reshape(-1, 3))
        inv = np.argsort(rows)
        scale = eloc_scale(g[p + "pairs"], g[p + "offsets"], g[p + "coeff"], g[p + "la"], n)
        assert np.all(np.abs(e[inv] - g[p + "eloc"]) <= 1e-12 * scale)
        assert np.allclose(sc[inv], scale, rtol=1e-12, atol=1e-300)


def test_variance_definition_on_goldens():
    """EnergyReport.variance from the five moments (energy.py) equals the
    definition Var = sum w |E - E0|^2 on the reference's own E_loc."""
    from paper_2408_07625_b200.energy import _report_from_moments
    for family in FAMILIES:
        g = golden(family)
        for _, p in instances(family):
            st, m, w = oracle.variational_energy(g[p + "lp"], float(g[p + "norm"]), float(g[p + "log_norm"]),
                                                 g[p + "eloc"])
            e = g[p + "eloc"]
            e0 = np.sum(w * e)
            var = float(np.sum(w * np.abs(e - e0) ** 2))
            assert abs(m[4] - float(np.sum(w * np.abs(e) ** 2))) <= 1e-12 * max(1.0, m[4])
            r = _report_from_moments(m, float(g[p + "norm"]), float(g[p + "log_norm"]), e, w)
            assert abs(r.variance - var) <= 1e-12 * max(1.0, m[4])
