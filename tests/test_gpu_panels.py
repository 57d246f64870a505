"""Column-panel layout (SC_CREATE_PANELS, csrc/sc_panel.cuh): bit-identical to the SELL kernel
on the same handle and to the C oracle, for planted-partition graphs numbered by block (dense
panels), graphs without id locality (sparse groups only), ragged sizes (odd n, a partial last
row block and panel) and graphs the layout declines (weighted, wide rows, tiny)."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_10939_b200 import DeviceGraph, from_edges

pytestmark = pytest.mark.gpu


def _simple(n, u, v):
    """unit-weight graph from an edge list: self loops and repeated pairs dropped (from_edges
    would sum repeated pairs into weight 2)"""
    u, v = np.asarray(u, np.int64), np.asarray(v, np.int64)
    keep = u != v
    a, b = np.minimum(u[keep], v[keep]), np.maximum(u[keep], v[keep])
    key = np.unique(a * n + b)
    g, _ = from_edges(n, key // n, key % n, drop_isolated=True)
    assert g.unit_weights()
    return g


def _blocked(n, blk, d_in, d_out, seed):
    """Edges: every vertex draws d_in partners inside its block of `blk` consecutive ids and
    d_out anywhere (symmetrised by from_edges)."""
    rng = np.random.default_rng(seed)
    u = np.repeat(np.arange(n), d_in + d_out)
    b0 = (u // blk) * blk
    size = np.minimum(blk, n - b0)
    v = np.where(np.tile(np.arange(d_in + d_out) < d_in, n),
                 b0 + (rng.random(u.size) * size).astype(np.int64),
                 rng.integers(0, n, u.size))
    return _simple(n, u, v)


def _compare(g, T, seed=0, expect_panels=True):
    with DeviceGraph(g, panels=True) as dg:
        info = dg.info()
        assert (info["panel_groups"] > 0) == expect_panels, info
        x0 = dg.sample_irwin_hall(seed, return_host=True)
        out = {}
        for sym in (False, True):
            for sign in (1.0, -1.0):
                a = dg.power_iterate(T, sym=sym, sign=sign)
                b = dg.power_iterate(T, sym=sym, sign=sign, force_sell=True)
                c = dg.power_iterate(T, sym=sym, sign=sign, cuda_graph=False)
                for u, v in zip(a, b):
                    assert np.array_equal(u, v), (sym, sign)
                for u, v in zip(a, c):
                    assert np.array_equal(u, v), (sym, sign)
                out[(sym, sign)] = a
    xo, fo = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0, T)
    assert np.array_equal(out[(False, 1.0)][0], xo)
    assert np.array_equal(out[(False, 1.0)][1], fo)
    return info


def test_block_numbered_sbm_dense_panels():
    g = _blocked(120_000, 40_000, 20, 2, seed=3)
    info = _compare(g, 12)
    assert info["panel_bytes"] > 0


def test_odd_n_partial_blocks():
    g = _blocked(50_001, 16_667, 24, 2, seed=4)
    assert g.n % 2 == 1
    _compare(g, 9)


def test_no_locality_declined():
    """ids without locality: few entries fall into dense panels -> SELL only"""
    rng = np.random.default_rng(5)
    n = 600_000  # large enough that no 8192-column panel gets 1024 entries of a row block
    u = rng.integers(0, n, 8 * n)
    v = rng.integers(0, n, 8 * n)
    _compare(_simple(n, u, v), 3, expect_panels=False)


def test_small_graph_all_panels_dense():
    """few panels: every panel is dense even without id locality"""
    rng = np.random.default_rng(9)
    n = 40_000
    u = rng.integers(0, n, 8 * n)
    v = rng.integers(0, n, 8 * n)
    _compare(_simple(n, u, v), 7)


def test_mixed_dense_and_sparse_groups():
    """half of every row's entries local, half random: dense panels and long sparse groups
    (split by the stage budget) in every row block"""
    g = _blocked(60_000, 20_000, 16, 8, seed=8)
    _compare(g, 8)


def test_declined_layouts_still_exact():
    rng = np.random.default_rng(6)
    n = 20_000
    u = rng.integers(0, n, 6 * n)
    v = (u + rng.integers(1, 500, u.size)) % n
    w = 0.5 + rng.random(u.size)
    gw, _ = from_edges(n, u, v, w, drop_isolated=True)  # weighted -> SELL only
    _compare(gw, 5, expect_panels=False)
    hub = np.concatenate([np.zeros(300, np.int64), u[:4 * n]])
    hv = np.concatenate([rng.choice(np.arange(1, n), 300, replace=False), v[:4 * n]])
    gh = _simple(n, hub, hv)                  # a row of > 256 entries -> SELL only
    _compare(gh, 5, expect_panels=False)
    gs = _blocked(3000, 1000, 10, 1, seed=7)   # fewer rows than one panel row block
    _compare(gs, 5, expect_panels=False)


def test_pipeline_layouts_identical():
    """fast_spectral_cluster: layout 'panels' (also the 'auto' choice at T >= 64) and 'sell'
    give bit-identical embeddings and labels"""
    from paper_2310_10939_b200 import SpectralParams, fast_spectral_cluster
    g = _blocked(120_000, 40_000, 20, 2, seed=3)
    out = {}
    for layout in ("panels", "sell", "auto"):
        res = fast_spectral_cluster(g, SpectralParams(k=3, t=70, mode="one_vector", seed=1,
                                                      layout=layout))
        out[layout] = res
    for layout in ("sell", "auto"):
        assert np.array_equal(out[layout].embedding.data, out["panels"].embedding.data)
        assert np.array_equal(out[layout].partition.labels, out["panels"].partition.labels)
