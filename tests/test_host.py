"""CPU-side checks of the product: host index builder, parser, C-ABI exports.

No kernel is launched here (the container has no GPU); the device path is
covered by test_gpu_parity.py.
"""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2408_07625_b200 as q
from paper_2408_07625_b200 import _lib, basis
from helpers import golden, instances, product_index

ROOT = Path(__file__).resolve().parents[1]


def _same_grouping(H, g, p):
    assert H.n_xy == len(g[p + "xy"]) and H.n_terms == len(g[p + "coeff"])
    assert np.array_equal(H.xy, g[p + "xy"])
    assert np.array_equal(H.group_offsets, g[p + "offsets"])
    assert np.array_equal(H.coeff, g[p + "coeff"])
    assert np.array_equal(H.yz, g[p + "yz"]) and np.array_equal(H.y_weight, g[p + "y_weight"])
    assert np.array_equal(H.x_masks, g[p + "x"]) and np.array_equal(H.z_masks, g[p + "z"])
    d = int(g[p + "diag"])
    assert H.diagonal_xy_index() == (None if d < 0 else d)


@pytest.mark.parametrize("family", ["coupling", "accept3", "checks", "opscale"])
def test_index_build_matches_reference_grouping(family):
    g = golden(family)
    prefixes = ["small_", "large_"] if family == "opscale" else [p for _, p in instances(family)]
    for p in prefixes:
        _same_grouping(product_index(g, p), g, p)


def test_fixture_parse_matches_reference_grouping():
    g = golden("fixtures")
    for name in ("toy", "h2", "h4", "h6"):
        # rebuild the text from the reference's merged strings (grouped order re-groups identically)
        n = int(g[f"{name}_n_qubits"])
        lines = [f"qubits: {n}"]
        for c, x, y, z in zip(g[f"{name}_coeff"], g[f"{name}_x"], g[f"{name}_y"], g[f"{name}_z"]):
            s = "".join("X" if (int(x[i // 64]) >> (i % 64)) & 1 else "Y" if (int(y[i // 64]) >> (i % 64)) & 1
                        else "Z" if (int(z[i // 64]) >> (i % 64)) & 1 else "I" for i in range(n))
            lines.append(f"{float(c).hex()} {s}  # comment")
        H = q.HamiltonianIndex.parse("\n".join(lines) + "\n")
        _same_grouping(H, g, f"{name}_")


def test_toy_grouping_and_merge_rules():
    """test_hamiltonian.cpp:24-57."""
    H = q.HamiltonianIndex.parse("qubits: 4\n0.9 IIII\n0.1 IZZI\n-0.2 XIXI\n-0.2 IXIX\n0.3 IYYI\n")
    assert H.n_qubits == 4 and H.n_terms == 5 and H.n_xy == 4
    assert [basis.dec_value(H.xy[g], 4) for g in range(4)] == [0, 10, 5, 6]
    assert len(H.group(0)) == 2 and len(H.group(3)) == 1 and H.diagonal_xy_index() == 0
    H2 = q.HamiltonianIndex.parse("qubits: 4\n0.3 XYZI\n-0.3 XYZI\n0.9 IIII\n")
    assert H2.n_terms == 1 and H2.n_xy == 1 and basis.dec_value(H2.xy[0], 4) == 0
    H3 = q.HamiltonianIndex.from_terms(4, [(0.4, "XYII"), (-0.4, "XYII")])
    assert H3.n_terms == 0 and H3.n_xy == 0 and H3.diagonal_xy_index() is None
    yy = q.HamiltonianIndex.parse("qubits: 4\n0.3 IYYI\n")
    assert basis.dec_value(yy.yz[0], 4) == 6 and int(yy.y_weight[0]) == 2


@pytest.mark.parametrize("text,msg", [
    ("0.9 IIII\n", "hamiltonian line 1: expected header 'qubits: <N>'"),
    ("qubits: 4\n0.9\n", "hamiltonian line 2: expected '<coeff> <pauli_string>'"),
    ("qubits: 4\n0.9 IIII extra\n", "hamiltonian line 2: trailing content 'extra'"),
    ("qubits: 4\nabc IIII\n", "hamiltonian line 2: cannot parse coefficient 'abc' as a real number"),
    ("qubits: 4\ninf IIII\n", "hamiltonian line 2: non-finite coefficient"),
    ("qubits: 4\n# c\n\n0.9 III\n", "hamiltonian line 4: pauli string has length 3, expected 4"),
    ("qubits: 4\n0.9 IIQI\n", "hamiltonian line 2: illegal Pauli character 'Q'"),
    ("# nothing\n", "hamiltonian: missing 'qubits:' header"),
])
def test_parse_errors_follow_reference(text, msg):
    """hamiltonian.cpp:119-170: runtime_error with line numbers."""
    with pytest.raises(RuntimeError) as e:
        q.HamiltonianIndex.parse(text)
    assert str(e.value) == msg


def test_from_terms_errors():
    with pytest.raises(ValueError, match="pauli string length 3 != qubits 4"):
        q.HamiltonianIndex.from_terms(4, [(1.0, "III")])
    with pytest.raises(ValueError, match="illegal Pauli character 'Q'"):
        q.HamiltonianIndex.from_terms(4, [(1.0, "IXQZ")])
    with pytest.raises(ValueError):
        q.HamiltonianIndex.from_terms(0, [])
    with pytest.raises(ValueError):  # overlapping masks through the raw-mask entry
        q.HamiltonianIndex.from_masks(2, [1.0], [[1]], [[1]], [[0]])
    with pytest.raises(RuntimeError, match="cannot open hamiltonian file"):
        q.HamiltonianIndex.load("/nonexistent/x.ham")


def test_backend_names():
    assert q.parse_backend("trie") == q.CouplingBackend.kTrie
    assert q.backend_name(q.CouplingBackend.kBatch) == "batch"
    with pytest.raises(ValueError, match="unknown coupling backend: quantum"):
        q.parse_backend("quantum")


def test_basis_vectors():
    """basis_vector.hpp / test_basis_vector.cpp round trips incl. multi-word widths."""
    for n in (7, 63, 64, 65, 70, 129, 200, 256):
        rng = np.random.default_rng(n)
        bits = rng.integers(0, 2, (5, n)).astype(np.uint8)
        keys = basis.from_bool_rows(bits)
        assert keys.shape == (5, basis.n_words(n))
        assert np.array_equal(basis.to_bool_rows(keys, n), bits)
        s = "".join(map(str, bits[0]))
        assert np.array_equal(basis.parse(s), keys[0]) and basis.to_str(keys[0], n) == s
    assert basis.dec_value(basis.parse("1100"), 4) == 12
    with pytest.raises(ValueError):
        basis.parse("10a")
    with pytest.raises(ValueError):
        basis.n_words(257)


def _header_functions():
    text = (ROOT / "include" / "qvmc_cuda.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qvmc_[a-z_0-9]+)\s*\(", text)))


def test_cabi_exports_every_declared_symbol():
    lib = _lib.lib()
    names = _header_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
    assert {n for n, _, _ in _lib.SIGNATURES} == set(names)


def test_synth_library_is_separate():
    """qvmc_synth.h symbols live in libqvmc_synth.so only: the reference arm of
    bench.py generates its inputs without loading the kernels' library."""
    import ctypes as C
    from paper_2408_07625_b200 import synthetic
    text = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "qvmc_synth.h").read_text(), flags=re.S)
    names = sorted(set(re.findall(r"\b(qvmc_[a-z_0-9]+)\s*\(", text)))
    assert len(names) == 3
    slib = synthetic._slib()
    for name in names:
        assert hasattr(slib, name), name
        assert not hasattr(_lib.lib(), name), name
    deps = subprocess.run(["ldd", str(synthetic.SYNTH_PATH)], capture_output=True, text=True).stdout
    assert "cuda" not in deps and "qvmc_cuda" not in deps


def test_cabi_reports_missing_device_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    H = q.HamiltonianIndex.parse("qubits: 2\n0.7 II\n")
    with pytest.raises(RuntimeError):
        H.device_handle(0)
    assert "device" in _lib.last_error().lower()


def test_synthetic_generators_structure():
    from paper_2408_07625_b200 import synthetic
    H = synthetic.jw_hamiltonian(20, 12_000, seed=1)
    w = np.array([bin(int(v[0])).count("1") for v in H.xy])
    assert set(np.unique(w)) <= {0, 2, 4}
    d = H.diagonal_xy_index()
    assert len(H.group(d)) == 1 + 20 + 190  # identity + Z + ZZ
    keys = synthetic.near_hf_keys(56, 14, 2000, seed=2)
    assert len({k.tobytes() for k in keys}) == 2000
    assert np.all(basis.popcount(keys) == 14)
    up = basis.to_bool_rows(keys, 56)[:, 0::2].sum(axis=1)
    assert np.all(up == 7)


def test_no_cpu_fallback_when_library_missing(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setenv("QVMC_CUDA_LIB", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        _lib.lib()


DROPIN = ROOT / "paper_2408_07625_b200" / "lib" / "libqvmc_dropin.so"
REF_SRC = Path("/root/reference/proj/src")


def _defined_symbols(path, demangle=True, kinds="TW"):
    import subprocess
    args = ["nm", "-g", "--defined-only"] + (["-C"] if demangle else []) + [str(path)]
    out = subprocess.run(args, capture_output=True, text=True, check=True).stdout
    return {line.split(" ", 2)[2].replace("[abi:cxx11]", "") for line in out.splitlines()
            if line.count(" ") >= 2 and line.split(" ")[1] in kinds}


@pytest.mark.skipif(not DROPIN.exists(), reason="drop-in is built only where the reference headers exist")
def test_dropin_defines_the_replaced_translation_units():
    """libqvmc_dropin.so defines every global function of coupling.cpp and energy.cpp."""
    syms = _defined_symbols(DROPIN)
    want = ["qvmc::parse_backend(", "qvmc::backend_name(", "qvmc::loop_over_terms(", "qvmc::loop_over_batch(",
            "qvmc::loop_over_trie(", "qvmc::find_coupled_pairs(", "qvmc::local_energies(",
            "qvmc::variational_energy(", "qvmc::energy_gradient(", "qvmc::GradientAccumulator::add(",
            "qvmc::GradientAccumulator::take(", "qvmc::GradientAccumulator::GradientAccumulator("]
    for w in want:
        assert any(s.startswith(w) for s in syms), w
    if REF_SRC.exists():
        import subprocess
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            for tu in ("coupling", "energy"):
                obj = Path(d) / f"{tu}.o"
                subprocess.run(["g++", "-std=c++20", "-c", "-w", "-I/root/reference/proj/include",
                                f"-I{ROOT / 'paper_2408_07625_b200' / 'dropin' / 'eigen_shim'}",
                                str(REF_SRC / f"{tu}.cpp"), "-o", str(obj)], check=True)
                # strong definitions only: inline header functions are weak in every TU
                ref_syms = {s for s in _defined_symbols(obj, demangle=False, kinds="T") if s.startswith("_ZN4qvmc")}
                mine = _defined_symbols(DROPIN, demangle=False)
                missing = {s for s in ref_syms if s not in mine}
                assert not missing, missing


def _expected_plan(H):
    """Python restatement of the planner's record rules (host_index.cpp plan_device):
    kind A = weight-2/4 group, one shared Z string, 1 + W + terms <= 8 words."""
    W = H.n_words
    diag = H.diagonal_xy_index()
    a = singles = doubles = 0
    for g in range(H.n_xy):
        if g == diag:
            continue
        xy = [int(v) for v in H.xy[g]]
        wt = sum(bin(v).count("1") for v in xy)
        singles += wt == 2
        doubles += wt == 4
        t0, t1 = int(H.group_offsets[g]), int(H.group_offsets[g + 1])
        zs = {tuple(int(H.yz[t][w]) & ~xy[w] for w in range(W)) for t in range(t0, t1)}
        a += wt in (2, 4) and 1 <= t1 - t0 <= 7 - W and len(zs) == 1
    return a, singles, doubles


@pytest.mark.parametrize("name", ["h4", "h6"])
def test_device_plan_records_and_bitmaps(name):
    """The host-side device plan (no GPU): every group gets exactly one drain
    record kind, kind A exactly where the shared-Z rule holds, and the pair
    bitmaps hold one bit per single and six (every split into two pairs) per double."""
    g = golden("fixtures")
    H = product_index(g, f"{name}_")
    ps = H.plan_summary()
    a, singles, doubles = _expected_plan(H)
    n_groups = H.n_xy - (0 if H.diagonal_xy_index() is None else 1)
    assert ps["kind_a"] + ps["kind_b"] + ps["kind_c"] + ps["kind_d"] == n_groups
    assert ps["kind_a"] == a
    assert (ps["singles"], ps["doubles"]) == (singles, doubles)
    assert ps["bitmap_bits"] == singles + 6 * doubles
    assert ps["xy_tab_buckets"] >= 64 and ps["xy_tab_buckets"] * 2 >= H.n_xy
    if name == "h6":  # the 2 + 2(N-2)-term single excitations compress to families (kind B)
        assert ps["kind_b"] == 12 and ps["kind_c"] == ps["doubles"] - ps["kind_a"]


def test_device_plan_synthetic_jw_structure():
    """JW-structured synthetic H: doubles share their Z string (kind A), the
    2 + 2(N-2)-term singles compress to two families (kind B)."""
    from paper_2408_07625_b200 import synthetic
    H = synthetic.jw_hamiltonian(56, 20_000, seed=1)
    ps = H.plan_summary()
    assert ps["kind_a"] == ps["doubles"] and ps["kind_b"] == ps["singles"] and ps["kind_c"] == ps["kind_d"] == 0
    assert ps["bitmap_bits"] == ps["singles"] + 6 * ps["doubles"]
    big = synthetic.jw_hamiltonian(130, 2_000, seed=1)  # N > 128: no pair bitmaps
    assert big.plan_summary()["bitmap_bits"] == 0


def test_shard_bounds_match_python():
    """qvmc_shard_bounds (C ABI, no device needed) == distributed.shard_bounds."""
    import ctypes as C

    from paper_2408_07625_b200 import _lib
    from paper_2408_07625_b200.distributed import shard_bounds
    L = _lib.lib()
    for n, world in ((0, 1), (5, 8), (1_000_003, 8), (17, 3)):
        tot = 0
        for r in range(world):
            b, e = C.c_int64(), C.c_int64()
            _lib.check(L.qvmc_shard_bounds(n, world, r, C.byref(b), C.byref(e)))
            assert (b.value, e.value) == shard_bounds(n, world, r)
            tot += e.value - b.value
        assert tot == n
    with pytest.raises(ValueError):
        _lib.check(L.qvmc_shard_bounds(10, 2, 2, None, None))
