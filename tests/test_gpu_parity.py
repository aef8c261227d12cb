"""Parity of the sm_100a kernels (through the C ABI) with the reference.

Golden data = outputs of the UNMODIFIED reference (tests/golden). Bar:
  * pairs (x, x', xy), ops (terms/batch) and excitation class: bit-exact;
  * H_{xx'} per pair: bit-exact (same term order, exact +-c adds);
  * E_loc: |gpu - ref| <= 1e-10 x absolute-sum scale (helpers.ELOC_RTOL);
  * variational energy / ipr: 1e-10.
Large synthetic configurations are checked against the C oracle on sampled
rows, plus size-independent properties (Hermitian symmetry of the pair set,
full-sector Rayleigh quotient).
"""
import math

import numpy as np
import pytest

import oracle
import paper_2408_07625_b200 as q
from paper_2408_07625_b200 import synthetic
from helpers import assert_eloc_close, eloc_scale, golden, instances, product_index


def scale_rows(H, b, keys):
    p = q.loop_over_terms(keys, H)
    return eloc_scale(p.entries, H.group_offsets, H.coeff, b.log_amps, len(keys))

pytestmark = pytest.mark.gpu

FAMILIES = ["coupling", "accept3", "checks"]


def _batch(g, p):
    return q.SampleBatch(g[p + "keys"], g[p + "lp"], g[p + "la"], g[p + "ph"], float(g[p + "norm"]),
                         float(g[p + "log_norm"]))


def _check_path(H, g, p, sp=None):
    sp = sp or p
    keys = g[sp + "keys"]
    want = g[sp + "pairs"]
    for be, ops_key in ((q.loop_over_terms, "ops_terms"), (q.loop_over_batch, "ops_batch")):
        got = be(keys, H)
        assert np.array_equal(got.entries, want)
        assert got.ops == int(g[sp + ops_key])
    trie = q.loop_over_trie(keys, H)
    assert np.array_equal(trie.entries, want) and trie.backend == q.CouplingBackend.kTrie
    n = len(keys)
    # per-pair matrix elements + excitation class, bit-exact
    import ctypes as C
    from paper_2408_07625_b200 import _lib
    from paper_2408_07625_b200.hamiltonian import _ptr
    hh = np.zeros(len(want), dtype=np.complex128)
    cls = np.zeros(len(want), dtype=np.uint8)
    if len(want):
        e = np.ascontiguousarray(want, dtype=np.uint32)
        _lib.check(_lib.lib().qvmc_cuda_pair_elements(H.device_handle(0), n, _ptr(np.ascontiguousarray(keys)),
                                                      len(e), _ptr(e), _ptr(hh), _ptr(cls), _lib.MEM_HOST))
    assert np.array_equal(hh, g[sp + "pair_h"])
    xyw = np.array([bin(int(sum(int(w) << (64 * k) for k, w in enumerate(H.xy[gg])))).count("1")
                    for gg in want[:, 2]], dtype=np.uint8) if len(want) else cls
    assert np.array_equal(cls, xyw)
    # local energies from the pair list, and the fused path
    b = _batch(g, sp)
    scale = eloc_scale(want, g[p + "offsets"], g[p + "coeff"], g[sp + "la"], n)
    loc = q.local_energies(q.CoupledPairs(want, 0, q.CouplingBackend.kTerms), b, H)
    assert_eloc_close(loc, g[sp + "eloc"], scale)
    rep = q.variational_energy(b, loc, index=H)
    ev = g[sp + "evar"]
    assert abs(rep.e_var - ev[0]) <= 1e-10 * max(1.0, abs(ev[0]))
    assert abs(rep.ipr - ev[2]) <= 1e-12
    fused = q.surrogate_energy(H, b, check=False)
    assert_eloc_close(fused.locals, g[sp + "eloc"], scale)
    assert abs(fused.e_var - ev[0]) <= 1e-10 * max(1.0, float(np.sum(np.exp(g[sp + "lp"] - g[sp + "log_norm"])
                                                                      * scale)))
    return fused


@pytest.mark.parametrize("family", FAMILIES)
def test_random_families_match_reference(cuda_ok, family):
    g = golden(family)
    for _, p in instances(family):
        _check_path(product_index(g, p), g, p)


@pytest.mark.parametrize("name", ["toy", "h2", "h4", "h6"])
def test_fixture_sectors_match_reference(cuda_ok, name):
    g = golden("fixtures")
    H = product_index(g, f"{name}_")
    _check_path(H, g, f"{name}_", f"{name}_sector_")
    st = q.last_stats(H)
    assert st["sector_mode"] == 1  # one particle sector: the sector candidate lists ran


def test_toy_known_answers(cuda_ok):
    """checks.cpp:110-154 / acceptance criterion 1 through the device."""
    H = q.HamiltonianIndex.parse("qubits: 4\n0.9 IIII\n0.1 IZZI\n-0.2 XIXI\n-0.2 IXIX\n0.3 IYYI\n")
    keys = q.basis.parse_batch(["1100", "1001", "0110"])
    want = [[0, 0, 0], [0, 1, 2], [0, 2, 1], [1, 0, 2], [1, 1, 0], [2, 0, 1], [2, 2, 0]]
    for be in (q.loop_over_terms, q.loop_over_batch, q.loop_over_trie):
        assert be(keys, H).entries.tolist() == want
    x0, x1, x2 = keys
    assert abs(H.matrix_element(x0, x0) - 0.8) <= 1e-12
    assert abs(H.matrix_element(x0, x1) + 0.2) <= 1e-12
    assert abs(H.matrix_element(x2, x0) + 0.2) <= 1e-12
    assert abs(H.matrix_element(x1, x1) - 1.0) <= 1e-12
    assert H.matrix_element(x1, x2) == 0
    la = np.array([math.log(2.0), 0.0, 0.0])
    b = q.SampleBatch(keys, np.log(np.array([4.0, 1.0, 1.0]) / 6), la, np.array([0.0, 0.0, math.pi]), 1.0, 0.0)
    pairs = q.loop_over_batch(keys, H)
    loc = q.local_energies(pairs, b, H)
    assert np.allclose(loc, [0.8, 0.6, 1.4], rtol=0, atol=1e-12)
    rep = q.variational_energy(b, loc)
    assert abs(rep.e_var - 5.2 / 6) < 1e-13 and abs(rep.ipr - 0.5) < 1e-12 and abs(rep.weights.sum() - 1) < 1e-12
    fused = q.surrogate_energy(H, b)
    assert np.allclose(fused.locals, [0.8, 0.6, 1.4], rtol=0, atol=1e-12)
    # lone YY gives -coeff (test_hamiltonian.cpp:98-103)
    yy = q.HamiltonianIndex.parse("qubits: 4\n0.3 IYYI\n")
    e = yy.matrix_element(q.basis.parse("0110"), q.basis.parse("0000"))
    assert abs(e.real + 0.3) < 1e-14 and abs(e.imag) < 1e-14


def test_degenerate_inputs(cuda_ok):
    """test_coupling.cpp:109-136 and test_energy_sr.cpp:69-88."""
    ident = q.HamiltonianIndex.parse("qubits: 4\n1.0 IIII\n")
    p = q.loop_over_terms(q.basis.parse_batch(["0101"]), ident)
    assert p.entries.tolist() == [[0, 0, 0]]
    zz = q.HamiltonianIndex.parse("qubits: 4\n0.5 ZZII\n")
    batch = q.basis.parse_batch(["1100", "0011"])
    for be in (q.loop_over_terms, q.loop_over_batch, q.loop_over_trie):
        e = be(batch, zz).entries
        assert len(e) == 2 and all(r[0] == r[1] for r in e)
    empty = q.HamiltonianIndex.from_terms(4, [(0.4, "XYII"), (-0.4, "XYII")])
    assert len(q.loop_over_batch(batch, empty).entries) == 0
    assert len(q.loop_over_trie(batch, empty).entries) == 0
    # single sample: E_var = E_loc = 0.7 - 0.2
    h = q.HamiltonianIndex.parse("qubits: 2\n0.7 II\n0.2 ZI\n")
    b = q.SampleBatch(q.basis.parse_batch(["10"]), np.array([-0.3]), np.array([-0.15]), np.array([0.4]),
                      math.exp(-0.3), -0.3)
    loc = q.local_energies(q.loop_over_batch(b.vectors, h), b, h)
    rep = q.variational_energy(b, loc)
    assert abs(rep.e_var - loc[0].real) < 1e-14 and abs(rep.e_var - 0.5) < 1e-13
    fused = q.surrogate_energy(h, b)
    assert abs(fused.e_var - 0.5) < 1e-13
    # diagonal H => model-independent E_loc (test_oracle.cpp:77-90 analogue)
    d = q.HamiltonianIndex.parse("qubits: 4\n0.5 IIII\n0.25 ZIII\n")
    keys = q.basis.parse_batch(["0100", "0010"])
    b = q.SampleBatch(keys, np.array([-1.0, -2.0]), np.array([-0.5, -1.0]), np.array([0.3, 2.0]), 1.0, 0.0)
    assert np.allclose(q.surrogate_energy(d, b, check=False).locals, [0.75, 0.75], atol=1e-15)


def test_error_paths(cuda_ok):
    h = q.HamiltonianIndex.parse("qubits: 2\n0.7 II\n0.1 XX\n")
    keys = q.basis.parse_batch(["10", "01"])
    b = q.SampleBatch(keys, np.array([-1.0, -1.0]), np.array([-np.inf, 0.0]), np.zeros(2), 1.0, 0.0)
    with pytest.raises(q.QvmcLogicError, match="zero amplitude"):
        q.local_energies(q.loop_over_batch(keys, h), b, h)
    with pytest.raises(q.QvmcLogicError, match="zero amplitude"):
        q.surrogate_energy(h, b, check=False)
    with pytest.raises(ValueError, match="duplicate"):
        q.loop_over_terms(q.basis.parse_batch(["10", "10"]), h)
    b2 = q.SampleBatch(q.basis.parse_batch(["10"]), np.array([-800.0]), np.array([-400.0]), np.zeros(1),
                       math.exp(-800.0), -800.0)
    with pytest.raises(RuntimeError, match="norm is zero"):
        q.variational_energy(b2, np.array([1.0 + 0j]))
    with pytest.raises(ValueError):
        q.local_energies(q.CoupledPairs(np.array([[0, 5, 0]], np.uint32), 0, q.CouplingBackend.kTerms),
                         q.SampleBatch(keys, np.zeros(2), np.zeros(2), np.zeros(2), 1.0, 0.0), h)
    # the handle stays usable after errors
    assert len(q.loop_over_terms(keys, h).entries) == 4


def test_full_sector_rayleigh_quotient(cuda_ok):
    """With U = the full sector the surrogate energy is the Rayleigh quotient
    (test_energy_sr.cpp:90-124): psi^H H psi / psi^H psi with H from the oracle."""
    g = golden("fixtures")
    H = product_index(g, "h4_")
    O = oracle.OracleIndex(8, g["h4_coeff"], g["h4_x"], g["h4_y"], g["h4_z"])
    keys = g["h4_sector_keys"]
    la, ph = g["h4_sector_la"], g["h4_sector_ph"]
    lp, norm, log_norm = q.normalise(la)
    b = q.SampleBatch(keys, lp, la, ph, norm, log_norm)
    rep = q.surrogate_energy(H, b)
    psi = np.exp(la) * np.exp(1j * ph)
    n = len(keys)
    Hm = np.array([[O.matrix_element(keys[r], keys[c]) for c in range(n)] for r in range(n)])
    assert np.allclose(Hm, Hm.conj().T, atol=1e-14)
    rq = (psi.conj() @ Hm @ psi).real / (psi.conj() @ psi).real
    assert abs(rep.e_var - rq) <= 1e-10


def _synthetic_rows_vs_oracle(n_qubits, n_e, n_terms, n_unq, n_check, seed):
    c, x, y, z = synthetic.jw_terms(n_qubits, n_terms, seed=1)
    H = q.HamiltonianIndex.from_masks(n_qubits, c, x, y, z)
    O = oracle.OracleIndex(n_qubits, c, x, y, z)
    keys = synthetic.near_hf_keys(n_qubits, n_e, n_unq, seed=2)
    b = synthetic.sample_batch(keys, seed=3)
    rep = q.surrogate_energy(H, b)
    st = q.last_stats(H)
    assert st["sector_mode"] == 1 and st["rows"] == n_unq
    rng = np.random.default_rng(seed)
    rows = np.unique(np.concatenate([np.arange(min(64, n_unq)), rng.choice(n_unq, n_check, replace=False)]))
    want = np.zeros(len(rows), dtype=np.complex128)
    scale = np.zeros(len(rows))
    for k, r in enumerate(rows):
        e, _, s = O.eloc_rows(keys, b.log_amps, b.phases, int(r), int(r) + 1, with_scale=True)
        want[k], scale[k] = e[0], s[0]
    assert_eloc_close(rep.locals[rows], want, scale)
    return H, rep, st


@pytest.mark.parametrize("n_qubits,n_e,n_terms,n_unq", [(56, 14, 300_000, 20_000), (118, 110, 3_000_000, 20_000)])
def test_synthetic_configs_match_oracle(cuda_ok, n_qubits, n_e, n_terms, n_unq):
    _synthetic_rows_vs_oracle(n_qubits, n_e, n_terms, n_unq, 96, seed=n_qubits)


def test_pairs_symmetric_and_shard_invariant(cuda_ok, monkeypatch):
    """Size-independent properties at a medium synthetic size: the pair set is
    exchange-symmetric, the fused pair count equals the materialised one, and
    row-sharded fused calls reproduce each other bit for bit whatever the split
    (every row walks all its partners) and the whole-set call (symmetric mode:
    each unordered pair once, mirrored contributions summed exactly) to fp64
    reordering; with QVMC_SYMMETRIC=0 the whole-set call is the shards' own
    arithmetic, bit for bit."""
    H = synthetic.jw_hamiltonian(56, 300_000, seed=1)
    keys = synthetic.near_hf_keys(56, 14, 50_000, seed=2)
    b = synthetic.sample_batch(keys, seed=3)
    p = q.loop_over_terms(keys, H)
    e = p.entries.astype(np.int64)
    fwd = set(map(tuple, e[:, :2].tolist()))
    assert all((j, i) in fwd for i, j in fwd)
    assert np.all(np.diff(e[:, 0]) >= 0)
    full = q.surrogate_energy(H, b)
    st = q.last_stats(H)
    assert st["pairs"] == len(e)
    parts = [q.surrogate_energy(H, b, r0, r1, check=False) for r0, r1 in ((0, 17_000), (17_000, 33_333), (33_333, 50_000))]
    parts2 = [q.surrogate_energy(H, b, r0, r1, check=False) for r0, r1 in ((0, 5_000), (5_000, 50_000))]
    cat = np.concatenate([r.locals for r in parts])
    assert np.array_equal(cat, np.concatenate([r.locals for r in parts2]))
    assert abs(sum(r.e_var for r in parts) - full.e_var) <= 1e-12 * max(1, abs(full.e_var))
    loc = q.local_energies(p, b, H)
    scale = eloc_scale(p.entries, H.group_offsets, H.coeff, b.log_amps, len(keys))
    assert_eloc_close(full.locals, loc, scale)
    assert_eloc_close(full.locals, cat, scale, rtol=1e-12)
    assert np.array_equal(q.surrogate_energy(H, b).locals, full.locals)  # deterministic (exact fixed point)
    monkeypatch.setenv("QVMC_SYMMETRIC", "0")
    H2 = synthetic.jw_hamiltonian(56, 300_000, seed=1)
    assert np.array_equal(q.surrogate_energy(H2, b).locals, cat)


def test_cpp_dropin_acceptance(cuda_ok):
    """The reference's own HamiltonianIndex/BasisVector/generators linked against
    libqvmc_dropin.so in place of coupling.cpp + energy.cpp
    (paper_2408_07625_b200/dropin/test_dropin.cpp)."""
    import subprocess
    from pathlib import Path
    exe = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "test_dropin"
    if not exe.exists():
        pytest.skip("test_dropin is built only in the container that has the reference sources")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_ops_counters(cuda_ok):
    """test_coupling.cpp:170-190: terms = N*|XY|, batch = N^2, trie bounded."""
    g = golden("opscale")
    keys = g["small_keys"]
    for tag in ("small", "large"):
        H = product_index(g, f"{tag}_")
        assert q.loop_over_terms(keys, H).ops == 128 * H.n_xy == int(g[f"{tag}_ops_terms"])
        assert q.loop_over_batch(keys, H).ops == 128 * 128
        t = q.loop_over_trie(keys, H)
        assert t.ops <= 2 * 24 * 128 * 128 + 2 * 128
        assert np.array_equal(t.entries, g[f"{tag}_pairs"])
    # pruning: two far-apart states under the identity (test_coupling.cpp:192-203)
    ident = q.HamiltonianIndex.parse("qubits: 40\n1.0 " + "I" * 40 + "\n")
    keys = np.array([[0], [(1 << 40) - 1]], dtype=np.uint64)
    t = q.loop_over_trie(keys, ident)
    assert len(t.entries) == 2 and t.ops <= (4 * 40 + 4) * 2


@pytest.mark.parametrize("hit_cap", ["4096", "100000"])
def test_join_hit_buffer_regrow(cuda_ok, monkeypatch, hit_cap):
    """Split path (QVMC_FUSED=0: search kernel -> hit chunks in HBM -> chunk
    evaluation): a tiny first hit-buffer capacity exercises the overflow
    detection and the rerun with grown buffers: same E_loc, pair count and
    moments as a handle with the default capacity, and as the pairs-based
    evaluation."""
    n_unq = 20_000
    keys = synthetic.near_hf_keys(118, 110, n_unq, seed=7)
    b = synthetic.sample_batch(keys, seed=3)
    c, x, y, z = synthetic.jw_terms(118, 3_000_000, seed=1)
    monkeypatch.setenv("QVMC_FUSED", "0")
    monkeypatch.delenv("QVMC_HIT_CAP", raising=False)
    H0 = q.HamiltonianIndex.from_masks(118, c, x, y, z)
    ref = q.surrogate_energy(H0, b)
    n_pairs = q.last_stats(H0)["pairs"]
    monkeypatch.setenv("QVMC_HIT_CAP", hit_cap)
    H = q.HamiltonianIndex.from_masks(118, c, x, y, z)
    got = q.surrogate_energy(H, b)
    st = q.last_stats(H)
    assert st["join_mode"] == 1 and st["pairs"] == n_pairs
    assert np.array_equal(got.locals, ref.locals)  # deterministic: same chunks, same order
    assert got.e_var == ref.e_var
    half = q.surrogate_energy(H, b, 5_000, 15_000, check=False)  # a row shard: same rows, the full walk
    assert_eloc_close(half.locals, got.locals[5_000:15_000], scale_rows(H, b, keys)[5_000:15_000], rtol=1e-12)
    p = q.loop_over_terms(keys, H)
    loc = q.local_energies(p, b, H)
    scale = eloc_scale(p.entries, H.group_offsets, H.coeff, b.log_amps, n_unq)
    assert_eloc_close(got.locals, loc, scale)


@pytest.mark.parametrize("n_qubits,n_e,n_terms,n_unq", [(118, 110, 3_000_000, 50_000), (56, 14, 300_000, 50_000)])
def test_fused_matches_split_evaluation(cuda_ok, monkeypatch, n_qubits, n_e, n_terms, n_unq):
    """The fused warp-specialised kernel (default) and the split search +
    chunk-evaluation kernels give the same E_loc (to fp64 reordering: chunk
    sums are added in a different order), the same pair count, and the
    fused result is deterministic and row-shard invariant bit for bit."""
    keys = synthetic.near_hf_keys(n_qubits, n_e, n_unq, seed=11)
    b = synthetic.sample_batch(keys, seed=3)
    c, x, y, z = synthetic.jw_terms(n_qubits, n_terms, seed=1)
    monkeypatch.setenv("QVMC_FUSED", "0")
    Hs = q.HamiltonianIndex.from_masks(n_qubits, c, x, y, z)
    split = q.surrogate_energy(Hs, b)
    n_pairs = q.last_stats(Hs)["pairs"]
    monkeypatch.setenv("QVMC_FUSED", "1")
    H = q.HamiltonianIndex.from_masks(n_qubits, c, x, y, z)
    fused = q.surrogate_energy(H, b)
    st = q.last_stats(H)
    assert st["pairs"] == n_pairs and st["join_mode"] == 1
    p = q.loop_over_terms(keys, H)
    scale = eloc_scale(p.entries, H.group_offsets, H.coeff, b.log_amps, n_unq)
    assert_eloc_close(fused.locals, split.locals, scale, rtol=1e-12)
    again = q.surrogate_energy(H, b)
    assert np.array_equal(again.locals, fused.locals) and again.e_var == fused.e_var
    part = q.surrogate_energy(H, b, n_unq // 4, n_unq // 2, check=False)
    assert np.array_equal(part.locals, fused.locals[n_unq // 4: n_unq // 2])


@pytest.mark.parametrize("n_qubits,n_e,n_terms,n_unq,join", [
    (48, 24, 200_000, 5_000, 1),    # minority set of 24: the join's largest bucket tables (276 per row)
    (48, 24, 200_000, 5_000, 0),    # the same through the sector candidate lists (k_rows, QVMC_JOIN=0)
    (40, 20, 100_000, 5_000, 1),    # half filling (c40h shape), 190 buckets per row
    (64, 32, 200_000, 4_000, 1),    # half filling at 64 q: s = 32 (a warp's lanes), 496 buckets per row
    (130, 122, 400_000, 10_000, 1),  # 3 key words, n > 128: join without the pair-existence bitmaps
    (20, 10, 12_000, 20_000, 1),     # BASELINE config 2 shape (c20), random sector states
])
def test_other_row_paths_match_oracle(cuda_ok, monkeypatch, n_qubits, n_e, n_terms, n_unq, join):
    if not join:
        monkeypatch.setenv("QVMC_JOIN", "0")
    if n_qubits == 20:
        c, x, y, z = synthetic.jw_terms(20, n_terms, seed=1)
        H = q.HamiltonianIndex.from_masks(20, c, x, y, z)
        O = oracle.OracleIndex(20, c, x, y, z)
        keys = synthetic.random_sector_keys(20, 10, n_unq, seed=2)
        b = synthetic.sample_batch(keys, seed=3)
        rep = q.surrogate_energy(H, b)
        st = q.last_stats(H)
        rows = np.arange(0, n_unq, 97)
        want = np.zeros(len(rows), dtype=np.complex128)
        scale = np.zeros(len(rows))
        for k, r in enumerate(rows):
            e, _, s = O.eloc_rows(keys, b.log_amps, b.phases, int(r), int(r) + 1, with_scale=True)
            want[k], scale[k] = e[0], s[0]
        assert_eloc_close(rep.locals[rows], want, scale)
    else:
        _, rep, st = _synthetic_rows_vs_oracle(n_qubits, n_e, n_terms, n_unq, 64, seed=n_qubits)
    assert st["join_mode"] == join


def _restated_moments(lp, log_norm, eloc):
    """Var = sum_x w_x |E_loc(x) - E|^2, E = sum_x w_x E_loc(x), w = exp(lp - log_norm)
    (the reference computes no variance; this is the definition)."""
    w = np.exp(np.asarray(lp) - log_norm)
    e0 = np.sum(w * eloc)
    return float(np.sum(w * np.abs(eloc - e0) ** 2)), float(np.sum(w * np.abs(eloc) ** 2)), w


def _check_variance(H, b, want_eloc, scale):
    var, m4, w = _restated_moments(b.log_probs, b.log_norm, want_eloc)
    tol = 1e-9 * max(1.0, float(np.sum(w * (np.abs(want_eloc) + scale) ** 2)))
    fused = q.surrogate_energy(H, b, check=False)
    assert abs(fused.variance - var) <= tol, (fused.variance, var)
    # moment 5 itself (sum w |E|^2) through the moments entry point, on the golden E_loc
    rep = q.variational_energy(b, want_eloc, index=H) if abs(np.sum(w * want_eloc).imag) <= 1e-6 * max(
        1.0, abs(np.sum(w * want_eloc).real)) else None
    if rep is not None:
        assert abs(rep.variance - var) <= 1e-12 * max(1.0, m4)
        assert abs((rep.variance + rep.e_var ** 2 + rep.im_residual ** 2) - m4) <= 1e-12 * max(1.0, m4)
    return fused


@pytest.mark.parametrize("family", FAMILIES)
def test_variance_matches_restatement_families(cuda_ok, family):
    g = golden(family)
    for _, p in instances(family):
        H = product_index(g, p)
        b = _batch(g, p)
        scale = eloc_scale(g[p + "pairs"], g[p + "offsets"], g[p + "coeff"], g[p + "la"], b.size())
        _check_variance(H, b, g[p + "eloc"], scale)


@pytest.mark.parametrize("name", ["toy", "h2", "h4", "h6"])
def test_variance_matches_restatement_fixtures(cuda_ok, name):
    g = golden("fixtures")
    H = product_index(g, f"{name}_")
    sp = f"{name}_sector_"
    b = _batch(g, sp)
    scale = eloc_scale(g[sp + "pairs"], g[f"{name}_offsets"], g[f"{name}_coeff"], g[sp + "la"], b.size())
    _check_variance(H, b, g[sp + "eloc"], scale)


def test_c20_energy_and_variance_at_1e5(cuda_ok):
    """BASELINE config 2 shape: 20 q, n_e = 10, 1e5 unique random sector states
    (DESIGN §7), every row's E_loc vs the oracle, energy and variance."""
    c, x, y, z = synthetic.jw_terms(20, 12_000, seed=1)
    H = q.HamiltonianIndex.from_masks(20, c, x, y, z)
    O = oracle.OracleIndex(20, c, x, y, z)
    keys = synthetic.random_sector_keys(20, 10, 100_000, seed=2)
    b = synthetic.sample_batch(keys, seed=3)
    want, _, scale = O.eloc_rows(keys, b.log_amps, b.phases, 0, len(keys), with_scale=True)
    fused = _check_variance(H, b, want, scale)
    assert_eloc_close(fused.locals, want, scale)
    st, m, _ = oracle.variational_energy(b.log_probs, b.norm, b.log_norm, want)
    assert abs(fused.e_var - m[0]) <= 1e-10 * max(1.0, float(np.sum(np.exp(b.log_probs - b.log_norm) * scale)))


def test_symmetric_fixed_point_range_fallback(cuda_ok, monkeypatch):
    """Log amplitudes spread over 60 nats make some mirrored contributions psi(x)/psi(y) exceed the
    exact fixed-point range (2^46): the call must notice and redo the evaluation unpaired, giving
    exactly the QVMC_SYMMETRIC=0 result; a narrow spread stays paired and agrees to fp64 reordering."""
    H = synthetic.jw_hamiltonian(56, 300_000, seed=1)
    keys = synthetic.near_hf_keys(56, 14, 20_000, seed=12)
    b = synthetic.sample_batch(keys, seed=3)
    b.log_amps = np.random.default_rng(4).uniform(-60.0, 0.0, len(keys))
    b.log_probs = 2.0 * b.log_amps
    b.log_norm = float(np.log(np.exp(b.log_probs - b.log_probs.max()).sum()) + b.log_probs.max())
    wide = q.surrogate_energy(H, b, check=False)
    monkeypatch.setenv("QVMC_SYMMETRIC", "0")
    H0 = synthetic.jw_hamiltonian(56, 300_000, seed=1)
    assert np.array_equal(wide.locals, q.surrogate_energy(H0, b, check=False).locals)
