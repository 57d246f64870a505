"""Multi-GPU host protocol on CPU: world-size-2 gloo runs of the sharded power iteration
(partitioning, renumbering exchange, column renaming, z-slot all-gather) with the oracle as
the per-shard compute backend, checked bit for bit against the single-graph oracle."""

import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_10939_b200 import distributed as D
from paper_2310_10939_b200.generate import SbmParams, sample_sbm, sbm_rows


class OracleShard:
    """CPU stand-in for CudaShard (tests only): same renumbered layout and piece API, oracle
    arithmetic."""

    def __init__(self, rp, col_global, val, deg, plan, rank, seed_row0):
        import torch

        self.torch = torch
        self.plan, self.rank = plan, rank
        perm = plan.perms[rank]
        self.perm = perm
        self.n = perm.size
        lens = np.diff(rp)[perm]
        self.rp = np.zeros(self.n + 1, dtype=np.int64)
        np.cumsum(lens, out=self.rp[1:])
        idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in perm]) if rp[-1] else np.empty(0, int)
        self.col = plan.rename(col_global[idx])
        self.val = None if val is None else val[idx]
        self.deg_orig = deg
        self.deg = deg[perm]
        self.row0 = seed_row0

    def zeros(self, m):
        return self.torch.zeros(m, dtype=self.torch.float64)

    def irwin_hall(self, seed, x_out):
        x = O.irwin_hall(self.deg_orig, seed, row0=self.row0)
        x_out.copy_(self.torch.from_numpy(x[self.perm]))

    def _slot(self, j):
        lo, hi = (int(v) for v in self.plan.bounds[self.rank][j:j + 2])
        return lo, hi, self.plan.own(j, self.rank)[0]

    def scale_piece(self, j, x, z_full, sym=False):
        lo, hi, o = self._slot(j)
        z_full[o:o + hi - lo] = self.torch.from_numpy(x.numpy()[lo:hi] / self.deg[lo:hi])

    def step_piece(self, j, z_in, x_in, x_out, z_out, sign=1.0, sym=False):
        lo, hi, o = self._slot(j)
        rp = self.rp[lo:hi + 1] - self.rp[lo]
        col = self.col[self.rp[lo]:self.rp[hi]]
        val = None if self.val is None else self.val[self.rp[lo]:self.rp[hi]]
        y, zo = O.rw_rows(rp, col, val, self.deg[lo:hi], x_in.numpy()[lo:hi], z_in.numpy(),
                          sign=sign)
        x_out[lo:hi] = self.torch.from_numpy(y)
        z_out[o:o + hi - lo] = self.torch.from_numpy(zo)

    def pack(self, z_full, idx, out):
        out.copy_(z_full[idx.long()])

    def local_z(self, z_full):
        parts = []
        for j in range(self.plan.pieces):
            lo, hi, o = self._slot(j)
            parts.append(z_full[o:o + hi - lo].numpy())
        return np.concatenate(parts)

    def to_original(self, v):
        v = v.numpy() if hasattr(v, "numpy") else np.asarray(v)
        out = np.empty(self.n)
        out[self.perm] = v[: self.n]
        return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, graph, T, result_path, pieces=1):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rp, col, val, deg = graph
    starts = D.partition_rows(rp, world)
    lo, hi = int(starts[rank]), int(starts[rank + 1])
    lrp = rp[lo:hi + 1] - rp[lo]
    lcol = col[rp[lo]:rp[hi]]
    lval = None if val is None else val[rp[lo]:rp[hi]]
    plan = D.exchange_plan(lrp, starts, rank, world, pieces=pieces)
    shard = OracleShard(lrp, lcol, lval, deg[lo:hi], plan, rank, lo)
    xT, z = D.power_iterate_sharded(shard, plan, rank, T, seed=3)
    x_all = D.gather_to_rank0(shard.to_original(xT), plan, rank)
    f_all = D.gather_to_rank0(shard.to_original(shard.local_z(z)), plan, rank)
    if rank == 0:
        np.savez(result_path, x=x_all, f=f_all, starts=starts)
    dist.destroy_process_group()


def _halo_worker(rank, world, port, graph, T, result_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rp, col, val, deg = graph
    starts = D.partition_rows(rp, world)
    lo, hi = int(starts[rank]), int(starts[rank + 1])
    lrp = rp[lo:hi + 1] - rp[lo]
    lcol = col[rp[lo]:rp[hi]]
    lval = None if val is None else val[rp[lo]:rp[hi]]
    plan = D.exchange_halo_plan(lrp, lcol, starts, rank, world)
    shard = OracleShard(lrp, lcol, lval, deg[lo:hi], plan, rank, lo)
    runner = D.ShardedPower(shard, plan, rank, comm=D.HaloComm(shard, plan, rank))
    runner.sample(3)
    xT, z = runner.run(T)
    x_all = D.gather_to_rank0(shard.to_original(xT), plan, rank)
    f_all = D.gather_to_rank0(shard.to_original(shard.local_z(z)), plan, rank)
    if rank == 0:
        np.savez(result_path, x=x_all, f=f_all, halo=plan.n_halo, ncols=plan.ncols)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_power_iteration_bit_exact(tmp_path, world):
    """Halo exchange (only referenced remote z entries move, point to point) is bit-exact."""
    import torch.multiprocessing as mp

    g = _weighted_graph()
    graph = (g.row_offsets, g.col_indices.astype(np.int32), g.weights, g.degrees)
    T = 9
    out = str(tmp_path / "halo.npz")
    mp.start_processes(_halo_worker, args=(world, _free_port(), graph, T, out), nprocs=world,
                       join=True, start_method="spawn")
    res = np.load(out)
    x0 = O.irwin_hall(g.degrees, 3)
    xT, f = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0, T)
    assert np.array_equal(res["x"], xT)
    assert np.array_equal(res["f"], f)
    assert 0 < int(res["halo"]) < g.n


def test_halo_plans_local_match_distributed_lists():
    """halo_plans_local: every rank's send list is exactly the peer's halo request, in order."""
    g = _weighted_graph(n=2000, m=15000, seed=5)
    rp, col = g.row_offsets, g.col_indices.astype(np.int64)
    starts = D.partition_rows(rp, 3)
    lrps = [rp[starts[r]:starts[r + 1] + 1] - rp[starts[r]] for r in range(3)]
    lcols = [col[rp[starts[r]]:rp[starts[r + 1]]] for r in range(3)]
    plans = D.halo_plans_local(lrps, lcols, starts)
    for r, pl in enumerate(plans):
        ren = pl.rename(lcols[r])
        assert ren.min() >= 0 and ren.max() < pl.ncols
        # own rows start on an 8192-slot boundary and the halo blocks keep global-id order, so
        # along every row the renamed columns never go back to an earlier 4096-slot window (the
        # column-panel layout's condition)
        assert pl.base % 8192 == 0 and pl.own(0, r) == (pl.base, pl.base + pl.n)
        lr = lrps[r]
        for i in range(pl.n):
            w = ren[lr[i]:lr[i + 1]] // 4096
            assert np.all(np.diff(w) >= 0)
        for q in range(3):
            if q == r:
                continue
            # the ids q sends to r, mapped back through q's renumbering, are r's halo ids from q
            sent = plans[q].perms[q][plans[q].send_idx[r] - plans[q].base] + starts[q]
            assert np.array_equal(sent, pl.halo_ids[q])


def _weighted_graph(n=3000, m=30000, seed=11):
    from paper_2310_10939_b200 import from_edges

    rng = np.random.default_rng(seed)
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    keep = u != v
    g, _ = from_edges(n, u[keep], v[keep], 0.5 + rng.random(keep.sum()), drop_isolated=True)
    return g


@pytest.mark.parametrize("world,pieces", [(2, 1), (3, 1), (2, 4), (3, 3)])
def test_sharded_power_iteration_bit_exact(tmp_path, world, pieces):
    import torch.multiprocessing as mp

    g = _weighted_graph()
    graph = (g.row_offsets, g.col_indices.astype(np.int32), g.weights, g.degrees)
    T = 9
    out = str(tmp_path / "res.npz")
    mp.start_processes(_worker, args=(world, _free_port(), graph, T, out, pieces), nprocs=world,
                       join=True, start_method="spawn")
    res = np.load(out)
    x0 = O.irwin_hall(g.degrees, 3)
    xT, f = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0, T)
    assert np.array_equal(res["x"], xT)
    assert np.array_equal(res["f"], f)


def test_partition_rows_balanced():
    rng = np.random.default_rng(0)
    lens = rng.integers(0, 50, 10000)
    rp = np.concatenate([[0], np.cumsum(lens)])
    for world in (1, 2, 4, 8):
        s = D.partition_rows(rp, world)
        assert s[0] == 0 and s[-1] == 10000 and np.all(np.diff(s) >= 1)
        work = np.array([rp[s[r + 1]] - rp[s[r]] + s[r + 1] - s[r] for r in range(world)])
        assert work.max() <= work.mean() * 1.01 + 60


def test_plan_renaming_is_a_bijection():
    rng = np.random.default_rng(1)
    rp = np.concatenate([[0], np.cumsum(rng.integers(1, 300, 5000))])
    starts = D.partition_rows(rp, 4)
    lrps = [rp[starts[r]:starts[r + 1] + 1] - rp[starts[r]] for r in range(4)]
    perms = [D.sell_order(x) for x in lrps]
    for pieces in (1, 3):
        plan = D.ShardPlan(starts, perms, [D.n_sell_rows(x) for x in lrps], pieces)
        slots = plan.slot_of
        assert np.unique(slots).size == slots.size and slots.max() < plan.ncols
        for r in range(4):
            b = plan.bounds[r]
            assert b[0] == 0 and b[-1] == plan.sizes[r]
            for j in range(pieces):
                if b[j] < plan.n_sells[r]:
                    assert b[j] % 32 == 0
                lo, hi = plan.own(j, r)
                assert hi - lo == plan.pmax


def test_plan_alignment_keeps_windows_inside_panels():
    """ShardPlan(align=8192): every rank's z block starts on an 8192-slot boundary, so the
    4096-row renumbering windows (the only reordering of a row's columns) never straddle a
    column panel -- the condition the panel layout builder checks on the device"""
    rng = np.random.default_rng(3)
    rp = np.concatenate([[0], np.cumsum(rng.integers(1, 40, 30000))])
    starts = D.partition_rows(rp, 3)
    lrps = [rp[starts[r]:starts[r + 1] + 1] - rp[starts[r]] for r in range(3)]
    perms = [D.sell_order(x) for x in lrps]
    plan = D.ShardPlan(starts, perms, [D.n_sell_rows(x) for x in lrps], 1, align=8192)
    base = D.ShardPlan(starts, perms, [D.n_sell_rows(x) for x in lrps], 1)
    assert plan.pmax % 8192 == 0 and plan.pmax >= base.pmax
    for r in range(3):
        lo, _ = plan.own(0, r)
        assert lo % 8192 == 0
        ids = np.arange(int(starts[r]), int(starts[r + 1]))
        slots = plan.slot_of[ids]
        # original ids inside one 4096-row window of the rank stay inside one 8192 panel
        win = (ids - starts[r]) // 4096
        for w in np.unique(win):
            assert np.unique(slots[win == w] // 8192).size == 1
    assert np.unique(plan.slot_of).size == plan.slot_of.size


def test_sbm_rows_concatenate_to_sample_sbm():
    p = SbmParams(n=4000, k=8, p=0.02, q=0.002, seed=4)
    g = sample_sbm(p).graph
    assert g.n == p.n  # no isolated vertices
    parts = [sbm_rows(p, lo, hi) for lo, hi in ((0, 1000), (1000, 2500), (2500, 4000))]
    rp = np.concatenate([[0]] + [pp[0][1:] + sum(q[0][-1] for q in parts[:i])
                                 for i, pp in enumerate(parts)])
    col = np.concatenate([pp[1] for pp in parts])
    assert np.array_equal(rp, g.row_offsets)
    assert np.array_equal(col, g.col_indices)
    assert np.array_equal(np.concatenate([pp[2] for pp in parts]), g.degrees)


def test_entry_balanced_starts():
    from paper_2310_10939_b200.distributed import entry_balanced_starts

    rng = np.random.default_rng(0)
    lens = rng.integers(0, 50, 1000)
    lens[100:110] = 5000  # heavy rows
    rp = np.concatenate([[0], np.cumsum(lens)])
    for world in (1, 2, 3, 8):
        st = entry_balanced_starts(rp, world)
        assert st[0] == 0 and st[-1] == 1000 and np.all(np.diff(st) >= 1)
        loads = rp[st[1:]] - rp[st[:-1]]
        assert loads.max() - loads.min() <= 2 * lens.max()
    # every block keeps a row even when one row holds everything
    rp = np.array([0, 10**6, 10**6, 10**6, 10**6], dtype=np.int64)
    assert np.all(np.diff(entry_balanced_starts(rp, 4)) == 1)
