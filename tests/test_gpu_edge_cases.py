"""Edge cases of the device path against the C oracle: folded self-loop degrees with an
empty CSR row (a vertex whose only edge is a self-loop), the smallest graphs, k = n,
rows of exactly 256 / 257 entries (the SELL / wide-row boundary) and an all-wide graph."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_10939_b200 import (DeviceGraph, SpectralParams, fast_spectral_cluster,
                                   from_edges)

pytestmark = pytest.mark.gpu


def _check_pipeline(g, k, T, seed=0):
    with DeviceGraph(g) as dg:
        x0 = dg.sample_irwin_hall(seed, return_host=True)
        xT, f = dg.power_iterate(T)
    assert np.array_equal(x0, O.irwin_hall(g.degrees, seed))
    xo, fo = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0, T)
    assert np.array_equal(xT, xo) and np.array_equal(f, fo)
    res = fast_spectral_cluster(g, SpectralParams(k=k, t=T, mode="one_vector", seed=seed))
    lab, _ = O.lloyd(fo, k, O.kmeans_seed(seed))
    assert np.array_equal(res.partition.labels, lab)


def test_self_loops_and_empty_rows():
    rng = np.random.default_rng(1)
    n = 500
    u, v = rng.integers(0, n - 1, 3000), rng.integers(0, n - 1, 3000)
    u = np.concatenate([u, [n - 1, 3, 3]])        # vertex n-1: self-loop only (empty row)
    v = np.concatenate([v, [n - 1, 3, 7]])
    w = np.concatenate([0.5 + rng.random(3000), [2.5, 0.75, 1.25]])
    g, _ = from_edges(n, u, v, w, allow_self_loops=True, drop_isolated=True)
    assert np.diff(g.row_offsets)[-1] == 0 and g.degrees[-1] > 0
    _check_pipeline(g, 4, 30)


@pytest.mark.parametrize("n,k", [(2, 2), (3, 2), (5, 5)])
def test_smallest_graphs(n, k):
    u = np.arange(n - 1)
    g, _ = from_edges(n, u, u + 1)
    _check_pipeline(g, k, 7)


def test_sell_wide_boundary_rows():
    """Hubs with exactly 256 (last SELL row length) and 257 (first wide row) neighbours."""
    rng = np.random.default_rng(2)
    n = 3000
    hub_a = rng.choice(np.arange(2, n), 256, replace=False)
    hub_b = rng.choice(np.arange(2, n), 257, replace=False)
    u = np.concatenate([np.zeros(256, int), np.ones(257, int), rng.integers(2, n, 6000)])
    v = np.concatenate([hub_a, hub_b, rng.integers(2, n, 6000)])
    keep = u != v
    g, _ = from_edges(n, u[keep], v[keep], 0.5 + rng.random(keep.sum()), drop_isolated=True)
    lens = np.diff(g.row_offsets)
    assert 256 in lens and 257 in lens
    with DeviceGraph(g) as dg:
        assert dg.info()["long_rows"] >= 1
    _check_pipeline(g, 6, 25)


def test_all_rows_wide():
    """A complete graph on 300 vertices: every row has 299 entries (> 256), so the whole
    step runs in the wide-row kernel."""
    n = 300
    iu, iv = np.triu_indices(n, 1)
    g, _ = from_edges(n, iu, iv, 1.0 + (iu * 7 + iv) % 5)
    with DeviceGraph(g) as dg:
        assert dg.info()["long_rows"] == n
    _check_pipeline(g, 3, 12)


def test_fp32_value_variant_within_tolerance():
    """SC_CREATE_FP32_VALUES: weights stored as fp32 (products and sums still fp64); x_T and
    f agree with the fp64 oracle within 1e-5 relative (the north star's bound for this
    optional variant), on a weighted graph with wide rows and T = 200."""
    from paper_2310_10939_b200.generate import sample_dcsbm

    g = sample_dcsbm(200_000, 20, seed=4).graph
    x0 = O.irwin_hall(g.degrees, 2)
    with DeviceGraph(g, fp32_values=True) as dg:
        dg.set_x0(x0)
        xT, f = dg.power_iterate(200)
        assert dg.info()["long_rows"] > 0
    xo, fo = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0, 200)
    assert np.max(np.abs(xT - xo) / np.abs(xo)) < 1e-5
    assert np.max(np.abs(f - fo) / np.abs(fo)) < 1e-5
    assert not np.array_equal(xT, xo)  # it really is the reduced-precision variant
