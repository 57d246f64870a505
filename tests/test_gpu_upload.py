"""Uploads from ordinary (pageable) numpy arrays: large column / weight arrays are staged
through pinned slots by host threads (csrc/sc_hostcopy.cuh) on a worker thread beside the row
validation.  The device graph, and every iterate, must be identical to the direct
cudaMemcpyAsync path (SC_STAGE_OFF) and to the oracle; bad input still fails loudly."""

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_10939_b200 import DeviceGraph, SpeclusterError, from_edges
from paper_2310_10939_b200.graph import Graph

pytestmark = pytest.mark.gpu


def _big_weighted(seed=5, n=600_000, m=6_000_000):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, m)
    v = (u + rng.integers(1, 5000, m)) % n   # some locality, rows of ~20 entries
    g, _ = from_edges(n, u, v, 0.5 + rng.random(m), drop_isolated=True)
    return g


def _run(g, T, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        with DeviceGraph(g) as dg:
            x0 = dg.sample_irwin_hall(3, return_host=True)
            xT, f = dg.power_iterate(T)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return x0, xT, f


def test_staged_upload_matches_direct_and_oracle():
    g = _big_weighted()
    assert g.nnz * 4 >= 16 << 20  # the column array takes the staged path (> kStageMin)
    assert g.col_indices.flags["C_CONTIGUOUS"]
    x0a, xa, fa = _run(g, 12, {})
    x0b, xb, fb = _run(g, 12, {"SC_STAGE_OFF": "1"})
    assert np.array_equal(x0a, x0b) and np.array_equal(xa, xb) and np.array_equal(fa, fb)
    xo, fo = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0a, 12)
    assert np.array_equal(xa, xo) and np.array_equal(fa, fo)


def test_staged_upload_bad_column_fails_loudly():
    g = _big_weighted(seed=7, n=300_000, m=5_000_000)
    col = np.array(g.col_indices)
    col[len(col) // 2 + 12345] = g.n + 7  # out of range, deep inside a staged chunk
    bad = Graph(g.n, g.row_offsets, col, g.weights, g.degrees)
    with pytest.raises(SpeclusterError):
        DeviceGraph(bad)
