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


@pytest.mark.parametrize("kind", ["sbm", "heavy_tail", "wide"])
def test_device_renumbering_equals_host_sell_order(kind):
    """The graph handle builds its SELL renumbering on the device; multi-GPU plans rename
    columns with the host sc_sell_order -- the two must agree exactly."""
    import ctypes

    from paper_2310_10939_b200 import _lib
    from paper_2310_10939_b200.distributed import sell_order
    from paper_2310_10939_b200.generate import SbmParams, sample_dcsbm, sample_sbm

    if kind == "sbm":
        g = sample_sbm(SbmParams(n=20000, k=4, p=0.004, q=0.0004, seed=1)).graph
    elif kind == "heavy_tail":
        g = sample_dcsbm(50_000, 10, seed=3).graph
    else:
        n = 3000
        iu, iv = np.triu_indices(300, 1)
        rng = np.random.default_rng(5)
        u = np.concatenate([iu, rng.integers(300, n, 9000)])
        v = np.concatenate([iv, rng.integers(300, n, 9000)])
        keep = u != v
        g, _ = from_edges(n, u[keep], v[keep], drop_isolated=True)
    with DeviceGraph(g) as dg:
        perm = np.empty(g.n, dtype=np.int32)
        _lib.check(_lib.load().sc_graph_order(dg.handle, _lib.ptr(perm)))
    assert np.array_equal(perm, sell_order(g.row_offsets))


def test_invalid_rows_rejected_on_device():
    """row_ptr / degree errors are detected by the device validation with the same messages."""
    from paper_2310_10939_b200 import from_csr
    from paper_2310_10939_b200.errors import InputError

    n = 1 << 21  # above the host-validation threshold
    rp = np.arange(n + 1, dtype=np.int64)
    col = ((np.arange(n) + 1) % n).astype(np.int32)
    deg = np.ones(n)
    rp_bad = rp.copy()
    rp_bad[777] = rp_bad[779]  # row 777 ends before it starts
    with pytest.raises(InputError, match="row_ptr decreases at 777"):
        DeviceGraph(from_csr(n, rp_bad, col, None, deg))
    deg_bad = deg.copy()
    deg_bad[123456] = 0.0
    with pytest.raises(InputError, match="degree of row 123456"):
        DeviceGraph(from_csr(n, rp, col, None, deg_bad))
    with DeviceGraph(from_csr(n, rp, col, None, deg)) as dg:
        assert dg.info()["n"] == n


def test_bfs_reorder_is_exact():
    """The BFS locality pre-order only moves where z values live: x_T, f and the labels are
    bit-identical to the default layout and to the oracle (weighted, hubs, several components)."""
    rng = np.random.default_rng(8)
    n = 30000
    u, v = rng.integers(0, n, 150000), rng.integers(0, n, 150000)
    u = np.concatenate([u, np.zeros(600, int)])
    v = np.concatenate([v, rng.integers(1, n, 600)])
    keep = u != v
    g, _ = from_edges(n, u[keep], v[keep], 0.5 + rng.random(keep.sum()), drop_isolated=True)
    x0 = O.irwin_hall(g.degrees, 1)
    out = []
    for reorder in (None, "bfs"):
        with DeviceGraph(g, reorder=reorder) as dg:
            dg.set_x0(x0)
            out.append(dg.power_iterate(40))
    xo, fo = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0, 40)
    for xT, f in out:
        assert np.array_equal(xT, xo) and np.array_equal(f, fo)
    r = fast_spectral_cluster(g, SpectralParams(k=6, t=40, mode="one_vector", seed=1,
                                                reorder="bfs"))
    lab, _ = O.lloyd(r.embedding.data[:, 0], 6, O.kmeans_seed(1))
    assert np.array_equal(r.partition.labels, lab)
