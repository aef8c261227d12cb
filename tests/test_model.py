"""Amplitude evaluation: AnqsModel::log_psi / fill_amplitudes.

CPU tests pin the numpy restatement (oracle/model_oracle.py) against the
reference itself (golden vectors from oracle/_ref, tests/golden/model.npz,
and the compiled reference when present). GPU tests run k_log_psi through the
C ABI and compare with the golden vectors and the oracle.

Tolerance (fp64; the device sums layer 1 over the prefix minority and
reorders the GEMM sums): |Δ log|ψ|| and |Δ φ| ≤ 1e-10 · max(1, |value|),
the north_star's fp64 bar.
"""
from __future__ import annotations

import math
from pathlib import Path

import numpy as np
import pytest

import oracle
from oracle.model_oracle import ModelOracle

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "model.npz")
NAMES = sorted({k.split("_")[0] for k in GOLD.files if k.endswith("_cfg")} - {"init"})
TOL = 1e-10


def _params(name):
    import importlib.util
    spec = importlib.util.spec_from_file_location("mmg", Path(__file__).resolve().parent / "golden" /
                                                  "make_model_golden.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    n, bits, _, _, hidden, seed = (int(v) for v in GOLD[f"{name}_cfg"])
    return mod.model_params((n, bits, hidden), seed)


def _close(got, want, tol=TOL):
    got, want = np.asarray(got), np.asarray(want)
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(got), fin)
    assert np.array_equal(got[~fin], want[~fin])
    if fin.any():
        err = np.abs(got[fin] - want[fin]) / np.maximum(1.0, np.abs(want[fin]))
        assert err.max() <= tol, err.max()


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_golden(name):
    n, bits, ne, spin, hidden, _ = (int(v) for v in GOLD[f"{name}_cfg"])
    O = ModelOracle(n, bits, ne, spin, hidden, _params(name))
    la, ph = O.log_psi(GOLD[f"{name}_keys"])
    _close(la, GOLD[f"{name}_la"], 1e-12)
    _close(ph, GOLD[f"{name}_ph"], 1e-12)
    _, _, norm, log_norm = O.fill_amplitudes(GOLD[f"{name}_keys"], GOLD[f"{name}_lp"])
    assert abs(log_norm - GOLD[f"{name}_norm"][1]) <= 1e-12 * max(1.0, abs(log_norm))


def test_oracle_sector_is_normalised():
    """model.cpp normalises by construction: Σ_sector e^{2 log|ψ|} = 1 (test_model.cpp:124-151)."""
    for name in ("s8", "s12"):
        n, bits, ne, spin, hidden, _ = (int(v) for v in GOLD[f"{name}_cfg"])
        O = ModelOracle(n, bits, ne, spin, hidden, _params(name))
        la, _ = O.log_psi(GOLD[f"{name}_keys"])
        assert abs(np.exp(2 * la[np.isfinite(la)]).sum() - 1.0) < 1e-10


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_reference_init_params_golden():
    """SequentialRng-driven init_params (model.cpp:105-127) of the compiled reference is what the golden holds."""
    R = oracle.RefModel(12, 6, 6, True, 64)
    R.init_params(42)
    assert np.array_equal(R.params[:64], GOLD["init_params_head"])
    la, ph = R.log_psi(GOLD["init_keys"])
    assert np.array_equal(la, GOLD["init_la"]) and np.array_equal(ph, GOLD["init_ph"])
    O = ModelOracle(12, 6, 6, True, 64, R.params)
    la2, ph2 = O.log_psi(GOLD["init_keys"])
    _close(la2, la, 1e-12)
    _close(ph2, ph, 1e-12)


def test_layout_errors_follow_reference():
    from paper_2408_07625_b200.model import QuditLayout
    lay = QuditLayout.make(14, 6)
    assert lay.sizes == [6, 6, 2] and lay.offsets == [0, 6, 12]  # test_model.cpp:34-38
    with pytest.raises(ValueError, match="bits_per_qudit"):
        QuditLayout.make(4, 0)
    with pytest.raises(ValueError, match="qubit count"):
        QuditLayout.make(0, 6)


def test_checkpoint_hexfloat_spelling():
    from paper_2408_07625_b200.model import _hexfloat
    for v, s in ((1.0, "0x1p+0"), (1.5, "0x1.8p+0"), (0.1, "0x1.999999999999ap-4"), (-2.0, "-0x1p+1"),
                 (0.0, "0x0p+0")):
        assert _hexfloat(v) == s
        assert float.fromhex(s) == v


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_log_psi_matches_reference(cuda_ok, name):
    import paper_2408_07625_b200 as q
    n, bits, ne, spin, hidden, _ = (int(v) for v in GOLD[f"{name}_cfg"])
    M = q.AnqsModel(q.QuditLayout.make(n, bits), q.SectorConstraint(ne, bool(spin)), hidden)
    M.set_params(_params(name))
    keys = GOLD[f"{name}_keys"]
    la, ph = M.log_psi(keys)
    _close(la, GOLD[f"{name}_la"])
    _close(ph, GOLD[f"{name}_ph"])
    b = q.SampleBatch(keys, GOLD[f"{name}_lp"], np.zeros(len(keys)), np.zeros(len(keys)))
    q.fill_amplitudes(b, M)
    _close(b.log_amps, GOLD[f"{name}_la"])
    want_ln = GOLD[f"{name}_norm"][1]
    assert abs(b.log_norm - want_ln) <= 1e-12 * max(1.0, abs(want_ln))
    assert abs(b.norm - math.exp(want_ln)) <= 1e-12 * math.exp(want_ln)


@pytest.mark.gpu
def test_gpu_reference_init_params_and_normalisation(cuda_ok):
    import paper_2408_07625_b200 as q
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not shipped")
    R = oracle.RefModel(12, 6, 6, True, 64)
    R.init_params(42)
    M = q.AnqsModel(q.QuditLayout.make(12, 6), q.SectorConstraint(6, True))
    M.set_params(R.params)
    la, ph = M.log_psi(GOLD["init_keys"])
    _close(la, GOLD["init_la"])
    _close(ph, GOLD["init_ph"])
    assert abs(np.exp(2 * la).sum() - 1.0) < 1e-10  # normalised over the Sz = 0 sector


@pytest.mark.gpu
def test_gpu_log_psi_large_batch_and_ragged_tiles(cuda_ok):
    """1e5 near-HF samples at 118 qubits (a ragged final tile), sampled rows vs the oracle,
    and batch-invariance: a sub-batch gives bit-identical values."""
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import synthetic
    n, bits, ne = 118, 6, 110
    p = _params("h118")
    M = q.AnqsModel(q.QuditLayout.make(n, bits), q.SectorConstraint(ne, False))
    M.set_params(p)
    keys = synthetic.near_hf_keys(n, ne, 100_003, seed=5)
    la, ph = M.log_psi(keys)
    assert np.isfinite(la).all()
    O = ModelOracle(n, bits, ne, False, 64, p)
    rows = np.random.default_rng(1).choice(len(keys), 300, replace=False)
    la_o, ph_o = O.log_psi(keys[rows])
    _close(la[rows], la_o)
    _close(ph[rows], ph_o)
    la2, ph2 = M.log_psi(keys[777:777 + 1001])
    assert np.array_equal(la2, la[777:777 + 1001]) and np.array_equal(ph2, ph[777:777 + 1001])


@pytest.mark.gpu
def test_gpu_model_errors(cuda_ok):
    import paper_2408_07625_b200 as q
    lay = q.QuditLayout.make(12, 6)
    with pytest.raises(ValueError, match="hidden = 64"):
        q.AnqsModel(lay, q.SectorConstraint(6, True), hidden=32)
    with pytest.raises(ValueError, match="spin constraint requires even"):
        q.AnqsModel(lay, q.SectorConstraint(5, True))
    with pytest.raises(ValueError, match="electron count"):
        q.AnqsModel(lay, q.SectorConstraint(13, False))
    M = q.AnqsModel(lay, q.SectorConstraint(6, True))
    with pytest.raises(ValueError, match="size mismatch"):
        M.set_params(np.zeros(3))
    # empty batch is a no-op; all-zero parameters give the uniform distribution over allowed values
    la, ph = M.log_psi(np.zeros((0, 1), dtype=np.uint64))
    assert la.size == 0
    b = q.SampleBatch(np.zeros((0, 1), dtype=np.uint64), np.zeros(0), np.zeros(0), np.zeros(0))
    q.fill_amplitudes(b, M)  # the reference's empty-batch arithmetic (sampler.cpp:114-119)
    assert b.norm == 0.0 and b.log_norm == -math.inf
    from paper_2408_07625_b200 import synthetic
    keys = synthetic.sector_keys(12, 6, spin_balanced=True)
    la, ph = M.log_psi(keys)
    assert abs(np.exp(2 * la).sum() - 1.0) < 1e-12 and not ph.any()


@pytest.mark.gpu
def test_gpu_checkpoint_round_trip(cuda_ok):
    import paper_2408_07625_b200 as q
    M = q.AnqsModel(q.QuditLayout.make(20, 6), q.SectorConstraint(10, False))
    M.set_params(_params("r20"))
    text = M.save_checkpoint(seed=42)
    M2, seed = q.load_checkpoint(text)
    assert seed == 42 and np.array_equal(M2.params, M.params)
    keys = GOLD["r20_keys"]
    assert np.array_equal(M2.log_psi(keys)[0], M.log_psi(keys)[0])
    with pytest.raises(RuntimeError, match="bad magic"):
        q.load_checkpoint("nope\n")


@pytest.mark.gpu
def test_gpu_log_psi_device_pointers(cuda_ok):
    import torch
    import paper_2408_07625_b200 as q
    n, bits, ne, spin, hidden, _ = (int(v) for v in GOLD["h56_cfg"])
    M = q.AnqsModel(q.QuditLayout.make(n, bits), q.SectorConstraint(ne, bool(spin)), hidden)
    M.set_params(_params("h56"))
    keys = torch.from_numpy(GOLD["h56_keys"].view(np.int64)).cuda()
    la = torch.empty(keys.shape[0], dtype=torch.float64, device="cuda")
    ph = torch.empty_like(la)
    M.log_psi_device(keys.data_ptr(), keys.shape[0], la.data_ptr(), ph.data_ptr())
    M.synchronize()
    _close(la.cpu().numpy(), GOLD["h56_la"])
    _close(ph.cpu().numpy(), GOLD["h56_ph"])


@pytest.mark.gpu
def test_gpu_sharded_fill_amplitudes_world1(cuda_ok):
    """distributed.sharded_fill_amplitudes with the device evaluator on an NCCL group of one rank."""
    import os
    import socket

    import torch
    import torch.distributed as dist
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200.distributed import Shard, model_evaluate, sharded_fill_amplitudes
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        n, bits, ne, spin, hidden, _ = (int(v) for v in GOLD["h56_cfg"])
        M = q.AnqsModel(q.QuditLayout.make(n, bits), q.SectorConstraint(ne, bool(spin)), hidden)
        M.set_params(_params("h56"))
        keys = GOLD["h56_keys"]
        dev = torch.device("cuda:0")
        sh = Shard(torch.from_numpy(keys.view(np.int64)).to(dev), torch.zeros(len(keys), dtype=torch.float64, device=dev),
                   torch.zeros(len(keys), dtype=torch.float64, device=dev), torch.from_numpy(GOLD["h56_lp"]).to(dev))
        log_norm = sharded_fill_amplitudes(sh, model_evaluate(M, 0))
        torch.cuda.synchronize()
        _close(sh.log_amps.cpu().numpy(), GOLD["h56_la"])
        _close(sh.phases.cpu().numpy(), GOLD["h56_ph"])
        want = GOLD["h56_norm"][1]
        assert abs(log_norm - want) <= 1e-12 * max(1.0, abs(want))
    finally:
        dist.destroy_process_group()


def test_checkpoint_parameter_parsing_follows_strtod():
    """Parameters parse like the reference's stream extraction: hexfloat only with a
    0x prefix, decimal otherwise ('0.5' is 0.5, not hex 0.3125); malformed -> RuntimeError."""
    from paper_2408_07625_b200.model import _parse_double
    assert _parse_double("0.5") == 0.5
    assert _parse_double("1e-3") == 1e-3
    assert _parse_double("-0x1.8p+1") == -3.0
    assert _parse_double("0X1p-2") == 0.25
    with pytest.raises(RuntimeError):
        _parse_double("abc")
