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
    """CPU stand-in for CudaShard (tests only): same renumbered layout, oracle arithmetic."""

    def __init__(self, rp, col_global, val, deg, plan, rank, seed_row0):
        import torch

        self.torch = torch
        self.plan, self.rank = plan, rank
        perm = plan.perms[rank]
        self.perm = perm
        self.n = perm.size
        self.off = rank * plan.n_max
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

    def scale(self, x, z_full, sym=False):
        z_full[self.off:self.off + self.n] = self.torch.from_numpy(x.numpy() / self.deg)

    def step(self, z_in, x_in, x_out, z_out, sign=1.0, sym=False):
        y, zo = O.rw_rows(self.rp, self.col, self.val, self.deg, x_in.numpy(), z_in.numpy(),
                          sign=sign)
        x_out.copy_(self.torch.from_numpy(y))
        z_out[self.off:self.off + self.n] = self.torch.from_numpy(zo)

    def to_original(self, v):
        out = np.empty(self.n)
        out[self.perm] = v[: self.n].numpy()
        return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, graph, T, result_path):
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
    plan = D.exchange_plan(lrp, starts, rank, world)
    shard = OracleShard(lrp, lcol, lval, deg[lo:hi], plan, rank, lo)
    xT, f = D.power_iterate_sharded(shard, plan, rank, T, seed=3)
    x_all = D.gather_to_rank0(shard.to_original(xT), plan, rank)
    f_all = D.gather_to_rank0(shard.to_original(f), plan, rank)
    if rank == 0:
        np.savez(result_path, x=x_all, f=f_all, starts=starts)
    dist.destroy_process_group()


def _weighted_graph(n=3000, m=30000, seed=11):
    from paper_2310_10939_b200 import from_edges

    rng = np.random.default_rng(seed)
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    keep = u != v
    g, _ = from_edges(n, u[keep], v[keep], 0.5 + rng.random(keep.sum()), drop_isolated=True)
    return g


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_power_iteration_bit_exact(tmp_path, world):
    import torch.multiprocessing as mp

    g = _weighted_graph()
    graph = (g.row_offsets, g.col_indices.astype(np.int32), g.weights, g.degrees)
    T = 9
    out = str(tmp_path / "res.npz")
    mp.start_processes(_worker, args=(world, _free_port(), graph, T, out), nprocs=world,
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
    perms = [D.sell_order(rp[starts[r]:starts[r + 1] + 1] - rp[starts[r]]) for r in range(4)]
    plan = D.ShardPlan(starts, perms)
    slots = plan.slot_of
    assert np.unique(slots).size == slots.size
    for r in range(4):
        own = slots[starts[r]:starts[r + 1]]
        assert own.min() == r * plan.n_max and own.max() < r * plan.n_max + plan.sizes[r]


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
