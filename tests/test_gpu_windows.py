"""Row-window layout (SC_CREATE_WINDOWS, csrc/sc_window.cuh): bit-identical to the SELL kernel
on the same handle and to the C oracle -- geometric k-NN graphs behind the BFS pre-order
(weighted and unit), banded graphs with ragged sizes (odd n, a partial last panel), hubs (wide
rows beside the windows), items cut by the far-slot cap, the fp32-value variant, graphs the
layout declines, and the pipeline's layout switch."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_10939_b200 import DeviceGraph, SpectralParams, fast_spectral_cluster, from_edges
from paper_2310_10939_b200.generate import DeviceCSR

pytestmark = pytest.mark.gpu


def _graph(n, u, v, w=None):
    u, v = np.asarray(u, np.int64), np.asarray(v, np.int64)
    keep = u != v
    a, b = np.minimum(u[keep], v[keep]), np.maximum(u[keep], v[keep])
    key, first = np.unique(a * n + b, return_index=True)
    ww = None if w is None else np.asarray(w)[keep][first]
    g, _ = from_edges(n, key // n, key % n, ww, drop_isolated=True)
    return g


def _banded(n, half, extra_far, seed, weighted):
    """vertex i is joined to `half` random ids within +-64 and to `extra_far` ids anywhere"""
    rng = np.random.default_rng(seed)
    u = np.repeat(np.arange(n), half + extra_far)
    near = np.clip(u + rng.integers(-64, 65, u.size), 0, n - 1)
    far = rng.integers(0, n, u.size)
    v = np.where(np.tile(np.arange(half + extra_far) < half, n), near, far)
    w = 0.5 + rng.random(u.size) if weighted else None
    return _graph(n, u, v, w)


def _knn2d(n, k, seed, weighted):
    """k-NN graph of random 2-D points with random ids (no id locality)"""
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    pts = rng.random((n, 2))
    d, j = cKDTree(pts).query(pts, k + 1)
    u = np.repeat(np.arange(n), k)
    v = j[:, 1:].ravel()
    w = np.exp(-(d[:, 1:].ravel() ** 2) * n / 8.0) + 1e-3 if weighted else None
    return _graph(n, u, v, w)


def _compare(g, T, reorder=None, expect=True, fp32=False, seed=0):
    with DeviceGraph(g, reorder=reorder, windows=True, fp32_values=fp32) as dg:
        info = dg.info()
        assert (info["window_items"] > 0) == expect, info
        x0 = dg.sample_irwin_hall(seed, return_host=True)
        out = {}
        for sym in (False, True):
            for sign in (1.0, -1.0):
                a = dg.power_iterate(T, sym=sym, sign=sign)
                b = dg.power_iterate(T, sym=sym, sign=sign, force_sell=True)
                c = dg.power_iterate(T, sym=sym, sign=sign, cuda_graph=False)
                for p, q in zip(a, b):
                    assert np.array_equal(p, q), (sym, sign)
                for p, q in zip(a, c):
                    assert np.array_equal(p, q), (sym, sign)
                out[(sym, sign)] = a
    if not fp32:
        xo, fo = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0, T)
        assert np.array_equal(out[(False, 1.0)][0], xo)
        assert np.array_equal(out[(False, 1.0)][1], fo)
    return info


def test_knn_weighted_bfs():
    g = _knn2d(70_001, 8, seed=1, weighted=True)
    assert not g.unit_weights()
    info = _compare(g, 15, reorder="bfs")
    assert info["panel_groups"] == 0


def test_knn_unit_bfs():
    g = _knn2d(50_000, 10, seed=2, weighted=False)
    assert g.unit_weights()
    _compare(g, 11, reorder="bfs")


def test_banded_odd_n_partial_panel():
    g = _banded(20_481 + 4096 * 3 + 7, 12, 1, seed=3, weighted=True)
    assert g.n % 4096 != 0
    _compare(g, 9)


def test_small_graph_one_panel():
    g = _banded(1500, 6, 0, seed=4, weighted=False)
    _compare(g, 7)


def test_items_cut_by_far_cap():
    """~1/3 of the entries leave the panel: 2048 rows hold more far entries than an item's far
    slots, so panels are cut into shorter items"""
    g = _banded(60_000, 22, 9, seed=5, weighted=True)
    info = _compare(g, 8)
    assert info["window_items"] > 2 * ((g.n + 2047) // 2048) // 2


def test_hub_rows_beside_windows():
    """rows longer than 256 entries go to the wide-row kernel, the rest through the windows"""
    rng = np.random.default_rng(6)
    n = 30_000
    u = np.repeat(np.arange(n), 10)
    v = np.clip(u + rng.integers(-50, 51, u.size), 0, n - 1)
    hub_u = np.concatenate([np.full(900, 17), np.full(400, 20_000)])
    hub_v = rng.integers(0, n, hub_u.size)
    g = _graph(n, np.concatenate([u, hub_u]), np.concatenate([v, hub_v]),
               0.5 + rng.random(u.size + hub_u.size))
    info = _compare(g, 10)
    assert info["long_rows"] >= 2


def test_fp32_values_same_as_sell():
    g = _banded(40_000, 10, 1, seed=7, weighted=True)
    _compare(g, 12, fp32=True)


def test_declined_without_locality():
    rng = np.random.default_rng(8)
    n = 50_000
    g = _graph(n, rng.integers(0, n, 300_000), rng.integers(0, n, 300_000))
    _compare(g, 6, expect=False)


def test_build_on_existing_handle_and_panels_win():
    """sc_graph_build_windows on a live handle; a handle with a panel layout keeps it"""
    from paper_2310_10939_b200 import _lib

    g = _banded(30_000, 10, 1, seed=9, weighted=True)
    with DeviceGraph(g) as dg:
        x0 = dg.sample_irwin_hall(3, return_host=True)
        a = dg.power_iterate(9)
        assert dg.info()["window_items"] == 0
        _lib.check(_lib.load().sc_graph_build_windows(dg.handle))
        assert dg.info()["window_items"] > 0
        b = dg.power_iterate(9)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    xo, fo = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0, 9)
    assert np.array_equal(b[0], xo) and np.array_equal(b[1], fo)


def test_pipeline_layouts_identical():
    g = _knn2d(40_000, 8, seed=10, weighted=True)
    out = {}
    for layout in ("windows", "sell", "auto"):
        out[layout] = fast_spectral_cluster(g, SpectralParams(k=4, t=70, mode="one_vector", seed=2,
                                                              reorder="bfs", layout=layout))
    for layout in ("sell", "auto"):
        assert np.array_equal(out[layout].embedding.data, out["windows"].embedding.data)
        assert np.array_equal(out[layout].partition.labels, out["windows"].partition.labels)


def test_config4_shape_device_csr():
    """the config-4 generator at reduced size (3-D 16-NN, weighted), BFS pre-order + windows
    built from the device CSR, against the oracle"""
    with DeviceCSR.knn3d(300_000, 20, 0) as d:
        g = d.download().graph
        with DeviceGraph.from_device_csr(d, reorder="bfs", windows=True) as dg:
            assert dg.info()["window_items"] > 0
            x0 = dg.sample_irwin_hall(0, return_host=True)
            xT, f = dg.power_iterate(30)
    xo, fo = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0, 30)
    assert np.array_equal(xT, xo) and np.array_equal(f, fo)


def test_multi_gpu_shards_with_windows():
    """the in-process multi-GPU handle (three shards sharing the GPU): every shard builds its
    own window layout over the shared z space; x_T and f equal the single handle's and the
    oracle's"""
    g = _banded(90_000, 10, 1, seed=11, weighted=True)
    with DeviceGraph(g, windows=True) as dg:
        x0 = dg.sample_irwin_hall(4, return_host=True)
        single = dg.power_iterate(14)
    with DeviceGraph(g, windows=True, devices=[0, 0, 0]) as mg:
        info = mg.info()
        assert info["n_gpus"] == 3 and info["window_items"] > 0, info
        x0m = mg.sample_irwin_hall(4, return_host=True)
        multi = mg.power_iterate(14)
    assert np.array_equal(x0, x0m)
    assert np.array_equal(single[0], multi[0]) and np.array_equal(single[1], multi[1])
    xo, fo = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0, 14)
    assert np.array_equal(multi[0], xo) and np.array_equal(multi[1], fo)
