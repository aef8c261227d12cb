"""Speculative (host-sync-free) device-memory calls of qvmc_cuda_eloc_fused.

With qvmc_cuda_set_speculative(h, 1), a QVMC_MEM_DEVICE call reuses the
previous call's sector plan (checked on the device) and checks its hit
buffers on the device, so it never waits for the host; qvmc_cuda_synchronize
verifies it and reruns it synchronously if the plan did not hold or a buffer
overflowed. Checked on the B200: same results as the synchronous path, a
re-plan (a different particle sector at the same sample count), an overflow
(tiny first hit capacity), and a CUDA-graph capture of the call replayed.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(n_qubits=56, n_terms=300_000):
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import synthetic
    c, x, y, z = synthetic.jw_terms(n_qubits, n_terms, seed=1)
    return q.HamiltonianIndex.from_masks(n_qubits, c, x, y, z)


def _dev(b):
    import torch
    d = torch.device("cuda", 0)
    return (torch.from_numpy(b.vectors.view(np.int64).copy()).to(d), torch.from_numpy(b.log_amps.copy()).to(d),
            torch.from_numpy(b.phases.copy()).to(d), torch.from_numpy(b.log_probs.copy()).to(d))


def _call(H, t, b, loc, mom, stream=None):
    import torch
    from paper_2408_07625_b200 import _lib
    L = _lib.lib()
    h = H.device_handle(0)
    raw = (stream or torch.cuda.current_stream(0)).cuda_stream or 0x1
    _lib.check(L.qvmc_cuda_set_stream(h, C.c_void_p(raw)))
    k, la, ph, lp = t
    n = k.shape[0]
    _lib.check(L.qvmc_cuda_eloc_fused(h, n, C.c_void_p(k.data_ptr()), C.c_void_p(la.data_ptr()),
                                      C.c_void_p(ph.data_ptr()), C.c_void_p(lp.data_ptr()), b.log_norm, 0, n,
                                      C.c_void_p(loc.data_ptr()), C.c_void_p(mom.data_ptr()), _lib.MEM_DEVICE))


def _sync(H):
    from paper_2408_07625_b200 import _lib
    _lib.check(_lib.lib().qvmc_cuda_synchronize(H.device_handle(0)))


def test_speculative_matches_sync_and_replans(cuda_ok):
    import torch
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import _lib, synthetic
    H = _setup()
    b1 = synthetic.sample_batch(synthetic.near_hf_keys(56, 14, 20_000, seed=3), seed=3)
    b2 = synthetic.sample_batch(synthetic.near_hf_keys(56, 16, 20_000, seed=4), seed=4)  # another sector
    want1 = q.surrogate_energy(H, b1).locals
    want2 = q.surrogate_energy(H, b2).locals
    _lib.check(_lib.lib().qvmc_cuda_set_speculative(H.device_handle(0), 1))
    loc = torch.zeros(20_000, dtype=torch.complex128, device="cuda")
    mom = torch.zeros(5, dtype=torch.float64, device="cuda")
    t1, t2 = _dev(b1), _dev(b2)
    _call(H, t1, b1, loc, mom)  # plans (one host read) and caches the plan
    _sync(H)
    assert np.array_equal(loc.cpu().numpy(), want1)
    for _ in range(3):  # speculative: no host synchronisation inside the call
        loc.zero_()
        _call(H, t1, b1, loc, mom)
        _sync(H)
        assert np.array_equal(loc.cpu().numpy(), want1)
    loc.zero_()
    _call(H, t2, b2, loc, mom)  # the cached plan (14 electrons) does not hold: rerun at synchronize
    _sync(H)
    assert np.array_equal(loc.cpu().numpy(), want2)
    _lib.check(_lib.lib().qvmc_cuda_set_speculative(H.device_handle(0), 0))


def test_speculative_overflow_rerun(cuda_ok, monkeypatch):
    import torch
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import _lib, synthetic
    monkeypatch.setenv("QVMC_HIT_CAP", "4096")
    H = _setup(118, 3_000_000)
    # random sector states couple to few others; near-HF states to many: the buffers sized by the
    # first (synchronous) call overflow in the speculative second one
    small = synthetic.sample_batch(synthetic.random_sector_keys(118, 110, 20_000, seed=5), seed=3)
    big = synthetic.sample_batch(synthetic.near_hf_keys(118, 110, 20_000, seed=7), seed=3)
    p_small = q.loop_over_terms(small.vectors, H).entries.shape[0]
    p_big = q.loop_over_terms(big.vectors, H).entries.shape[0]
    assert p_big > 2 * p_small
    want = q.surrogate_energy(_setup(118, 3_000_000), big).locals
    h = H.device_handle(0)
    _lib.check(_lib.lib().qvmc_cuda_set_speculative(h, 1))
    loc = torch.zeros(20_000, dtype=torch.complex128, device="cuda")
    mom = torch.zeros(5, dtype=torch.float64, device="cuda")
    _call(H, _dev(small), small, loc, mom)
    _sync(H)
    for _ in range(2):
        loc.zero_()
        _call(H, _dev(big), big, loc, mom)
        _sync(H)
        assert np.array_equal(loc.cpu().numpy(), want)


def test_speculative_call_in_a_cuda_graph(cuda_ok):
    import torch
    import paper_2408_07625_b200 as q
    from paper_2408_07625_b200 import _lib, synthetic
    H = _setup()
    b = synthetic.sample_batch(synthetic.near_hf_keys(56, 14, 30_000, seed=8), seed=3)
    want = q.surrogate_energy(H, b)
    _lib.check(_lib.lib().qvmc_cuda_set_speculative(H.device_handle(0), 1))
    t = _dev(b)
    loc = torch.zeros(30_000, dtype=torch.complex128, device="cuda")
    mom = torch.zeros(5, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):  # plan + size every buffer outside the capture
            _call(H, t, b, loc, mom, s)
            _sync(H)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        _call(H, t, b, loc, mom, s)
    loc.zero_()
    mom.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    _sync(H)
    assert np.array_equal(loc.cpu().numpy(), want.locals)
    assert float(mom[0]) == pytest.approx(want.e_var, rel=1e-12, abs=1e-12)
