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


def test_bfs_preorder_declined():
    """a BFS pre-order renames columns out of stored order: rows would revisit panels, so the
    layout is declined (the check in k_pan_plan) and results stay exact"""
    g = _blocked(120_000, 40_000, 20, 2, seed=3)
    rng = np.random.default_rng(12)
    p = rng.permutation(g.n)  # scatter the ids so the BFS pre-order is worth applying
    rp, col = g.row_offsets, g.col_indices
    u = np.repeat(np.arange(g.n), np.diff(rp))
    gs = _simple(g.n, p[u], p[col])
    with DeviceGraph(gs, reorder="bfs", panels=True) as dg:
        assert dg.info()["panel_groups"] == 0
        x0 = dg.sample_irwin_hall(0, return_host=True)
        xT, f = dg.power_iterate(6)
    xo, fo = O.power_iterate(gs.row_offsets, gs.col_indices, None, gs.degrees, x0, 6)
    assert np.array_equal(xT, xo) and np.array_equal(f, fo)


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


@pytest.mark.parametrize("world,aligned", [(2, True), (3, True), (2, False)])
def test_shard_panels_on_one_gpu_bit_exact(world, aligned):
    """row-block shards with the panel layout (sc_graph_build_panels) over the global z space,
    the all-gather emulated by device copies: bit-exact against the single-graph oracle"""
    import torch

    from paper_2310_10939_b200 import distributed as D

    g = _blocked(150_000, 50_000, 20, 2, seed=11)
    rp, col, deg = g.row_offsets, g.col_indices.astype(np.int32), g.degrees
    starts = D.partition_rows(rp, world)
    lrps = [rp[starts[r]:starts[r + 1] + 1] - rp[starts[r]] for r in range(world)]
    # z blocks aligned to 8192 slots keep the renumbering windows inside panels; without the
    # alignment rows revisit panels and the layout is declined (SELL, still exact)
    plan = D.ShardPlan(starts, [D.sell_order(x) for x in lrps], [D.n_sell_rows(x) for x in lrps], 1,
                       align=8192 if aligned else 1)
    shards = []
    for r in range(world):
        lo, hi = int(starts[r]), int(starts[r + 1])
        s = D.CudaShard(lrps[r], plan.rename(col[rp[lo]:rp[hi]]), None, deg[lo:hi], plan, r, 0)
        built = s.build_panels()
        assert built or not aligned
        shards.append(s)
    if not aligned:
        assert not all(s_.build_panels() for s_ in shards)
    T = 9
    z = [[s.zspace(plan.ncols), s.zspace(plan.ncols)] for s in shards]
    x = [[s.zeros(s.n), s.zeros(s.n)] for s in shards]
    x0 = [s.zeros(s.n) for s in shards]

    def gather(b):
        torch.cuda.synchronize()
        for r in range(world):
            lo, hi = plan.own(0, r)
            for q in range(world):
                if q != r:
                    z[q][b][lo:hi].copy_(z[r][b][lo:hi])

    for r, s in enumerate(shards):
        s.irwin_hall(2, x0[r])
        s.scale_piece(0, x0[r], z[r][0])
    gather(0)
    for t in range(T):
        a, b = t & 1, (t & 1) ^ 1
        for r, s in enumerate(shards):
            s.step_piece(0, z[r][a], x0[r] if t == 0 else x[r][a], x[r][b], z[r][b])
        gather(b)
    torch.cuda.synchronize()
    xs = np.concatenate([s.to_original(x[r][T & 1]) for r, s in enumerate(shards)])
    fs = np.concatenate([s.to_original(s.local_z(z[r][T & 1])) for r, s in enumerate(shards)])
    x0_ref = O.irwin_hall(deg, 2)
    xT, f = O.power_iterate(rp, col, None, deg, x0_ref, T)
    assert np.array_equal(xs, xT)
    assert np.array_equal(fs, f)
    for s in shards:
        s.close()


@pytest.mark.parametrize("n", [3392, 3393, 6785])
def test_row_block_boundaries(n):
    """one full row block, a last block of a single (odd) row, and one of one row past two
    blocks: the epilogue's prefetch path and its direct-load fallback"""
    g = _blocked(n, n, 4, 0, seed=n)  # ~8 entries per row: stages fit at 1696 rows per CTA
    _compare(g, 6)


def test_long_segment_declined():
    """a row with >= 128 entries inside one panel exceeds the segment count field: declined"""
    rng = np.random.default_rng(13)
    n = 20_000
    u = rng.integers(0, n, 12 * n)
    v = (u + rng.integers(1, 2000, u.size)) % n
    hub_v = rng.choice(np.arange(1, 4000), 200, replace=False)  # 200 neighbours in panel 0
    g = _simple(n, np.concatenate([u, np.zeros(200, np.int64)]), np.concatenate([v, hub_v]))
    assert np.diff(g.row_offsets).max() <= 256
    _compare(g, 5, expect_panels=False)


@pytest.mark.parametrize("world", [2, 3])
def test_halo_shard_panels_on_one_gpu_bit_exact(world):
    """halo z spaces (lower owners' entries | own rows on an 8192 boundary | higher owners')
    keep stored column order, so every halo shard takes the panel layout; the exchange is
    emulated by packs copied into the peers' halo slots"""
    import torch

    from paper_2310_10939_b200 import distributed as D

    g = _blocked(150_000, 50_000, 20, 2, seed=17)
    rp, col, deg = g.row_offsets, g.col_indices.astype(np.int32), g.degrees
    starts = D.partition_rows(rp, world)
    lrps = [rp[starts[r]:starts[r + 1] + 1] - rp[starts[r]] for r in range(world)]
    lcols = [col[rp[starts[r]]:rp[starts[r + 1]]] for r in range(world)]
    plans = D.halo_plans_local(lrps, lcols, starts)
    shards = []
    for r in range(world):
        s = D.CudaShard(lrps[r], plans[r].rename(lcols[r]), None, deg[starts[r]:starts[r + 1]],
                        plans[r], r, 0)
        assert s.build_panels()
        shards.append(s)
    z = [[s.zspace(plans[r].ncols), s.zspace(plans[r].ncols)] for r, s in enumerate(shards)]
    x = [[s.zeros(s.n), s.zeros(s.n)] for s in shards]
    x0 = [s.zeros(s.n) for s in shards]
    idx = [[torch.from_numpy(plans[q].send_idx[r]).cuda() for r in range(world)]
           for q in range(world)]

    def exchange(b):
        for r in range(world):
            for q in range(world):
                if q == r or idx[q][r].numel() == 0:
                    continue
                buf = shards[q].zeros(idx[q][r].numel())
                shards[q].pack(z[q][b], idx[q][r], buf)
                a, e = plans[r].halo_range(q)
                z[r][b][a:e].copy_(buf)
        torch.cuda.synchronize()

    T = 8
    for r, s in enumerate(shards):
        s.irwin_hall(3, x0[r])
        s.scale_piece(0, x0[r], z[r][0])
    exchange(0)
    for t in range(T):
        a, b = t & 1, (t & 1) ^ 1
        for r, s in enumerate(shards):
            s.step_piece(0, z[r][a], x0[r] if t == 0 else x[r][a], x[r][b], z[r][b])
        exchange(b)
    xs = np.concatenate([s.to_original(x[r][T & 1]) for r, s in enumerate(shards)])
    fs = np.concatenate([s.to_original(s.local_z(z[r][T & 1])) for r, s in enumerate(shards)])
    xT, f = O.power_iterate(rp, col, None, deg, O.irwin_hall(deg, 3), T)
    assert np.array_equal(xs, xT)
    assert np.array_equal(fs, f)
    for s in shards:
        s.close()
