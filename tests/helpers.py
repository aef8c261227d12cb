"""Shared test helpers: golden-fixture loading and the parity tolerance."""
from __future__ import annotations

from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"

# E_loc parity bar (BASELINE.json north_star: "within 1e-10 relative in fp64"),
# relative to the absolute-sum scale sum_{pairs} sum_{t in group} |c_t| * |psi(x')/psi(x)|
# (GPU reductions reorder sums, so relative-to-|E_loc| would
# blow up on cancellations).
ELOC_RTOL = 1e-10


@lru_cache(maxsize=None)
def golden(name: str):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def instances(name: str):
    g = golden(name)
    return [(int(s), f"s{int(s)}_") for s in g["seeds"]]


def product_index(g: dict, p: str):
    """Build the product HamiltonianIndex from the reference's merged strings."""
    from paper_2408_07625_b200 import HamiltonianIndex
    return HamiltonianIndex.from_masks(int(g[p + "n_qubits"]), g[p + "coeff"], g[p + "x"], g[p + "y"], g[p + "z"])


def oracle_index(g: dict, p: str):
    import oracle
    return oracle.OracleIndex(int(g[p + "n_qubits"]), g[p + "coeff"], g[p + "x"], g[p + "y"], g[p + "z"])


def group_abs(offsets: np.ndarray, coeff: np.ndarray) -> np.ndarray:
    cs = np.concatenate([[0.0], np.cumsum(np.abs(coeff))])
    off = offsets.astype(np.int64)
    return cs[off[1:]] - cs[off[:-1]]


def eloc_scale(pairs: np.ndarray, offsets, coeff, la, n: int) -> np.ndarray:
    """Per-row absolute-sum scale of E_loc."""
    gabs = group_abs(offsets, coeff)
    s = np.zeros(n)
    if len(pairs):
        x, j, g = pairs[:, 0].astype(np.int64), pairs[:, 1].astype(np.int64), pairs[:, 2].astype(np.int64)
        np.add.at(s, x, gabs[g] * np.exp(la[j] - la[x]))
    return np.maximum(s, 1e-300)


def assert_eloc_close(got, want, scale, rtol=ELOC_RTOL):
    err = np.abs(np.asarray(got) - np.asarray(want)) / scale
    worst = float(err.max()) if err.size else 0.0
    assert worst <= rtol, f"E_loc deviation {worst:.3e} of the absolute-sum scale (bar {rtol:g})"
    return worst
