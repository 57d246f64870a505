"""The CUDA shard kernels (sc_shard_create / _irwin_hall / _scale / _step) for 3 row blocks
on ONE GPU, with the per-step all-gather emulated by device copies between the shards' z
buffers (no cross-rank waiting on one GPU).  Bit-exact against the single-graph oracle."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_10939_b200 import distributed as D
from paper_2310_10939_b200 import from_edges

pytestmark = pytest.mark.gpu


def _graph(n=5000, m=60000, seed=21):
    rng = np.random.default_rng(seed)
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    # a hub row longer than the SELL limit exercises the wide-row path across shards
    u = np.concatenate([u, np.zeros(700, dtype=np.int64)])
    v = np.concatenate([v, rng.integers(1, n, 700)])
    keep = u != v
    g, _ = from_edges(n, u[keep], v[keep], 0.5 + rng.random(keep.sum()), drop_isolated=True)
    return g


@pytest.mark.parametrize("world,pieces", [(1, 1), (3, 1), (1, 3), (3, 4)])
def test_shards_on_one_gpu_bit_exact(world, pieces):
    import torch

    g = _graph()
    rp, col, val, deg = g.row_offsets, g.col_indices.astype(np.int32), g.weights, g.degrees
    starts = D.partition_rows(rp, world)
    lrps = [rp[starts[r]:starts[r + 1] + 1] - rp[starts[r]] for r in range(world)]
    plan = D.ShardPlan(starts, [D.sell_order(x) for x in lrps], [D.n_sell_rows(x) for x in lrps],
                       pieces)
    shards = []
    for r in range(world):
        lo, hi = int(starts[r]), int(starts[r + 1])
        shards.append(D.CudaShard(lrps[r], plan.rename(col[rp[lo]:rp[hi]]), val[rp[lo]:rp[hi]],
                                  deg[lo:hi], plan, r, 0))
    T = 12
    z = [[s.zeros(plan.ncols), s.zeros(plan.ncols)] for s in shards]
    x = [[s.zeros(s.n), s.zeros(s.n)] for s in shards]
    x0 = [s.zeros(s.n) for s in shards]

    def gather(buf_index, j):
        torch.cuda.synchronize()
        for r in range(world):
            lo, hi = plan.own(j, r)
            for q in range(world):
                if q != r:
                    z[q][buf_index][lo:hi].copy_(z[r][buf_index][lo:hi])

    for r, s in enumerate(shards):
        s.irwin_hall(5, x0[r])
    for j in range(pieces):
        for r, s in enumerate(shards):
            s.scale_piece(j, x0[r], z[r][0])
        gather(0, j)
    for t in range(T):
        a, b = t & 1, (t & 1) ^ 1
        for j in range(pieces):
            for r, s in enumerate(shards):
                s.step_piece(j, z[r][a], x0[r] if t == 0 else x[r][a], x[r][b], z[r][b])
            gather(b, j)
    torch.cuda.synchronize()
    xs = np.concatenate([s.to_original(x[r][T & 1]) for r, s in enumerate(shards)])
    fs = np.concatenate([s.to_original(s.local_z(z[r][T & 1])) for r, s in enumerate(shards)])
    x0_ref = O.irwin_hall(deg, 5)
    x0_dev = np.concatenate([s.to_original(x0[r]) for r, s in enumerate(shards)])
    assert np.array_equal(x0_dev, x0_ref)
    xT, f = O.power_iterate(rp, col, val, deg, x0_ref, T)
    assert np.array_equal(xs, xT)
    assert np.array_equal(fs, f)
    for s in shards:
        s.close()


@pytest.mark.parametrize("world", [2, 4])
def test_halo_shards_on_one_gpu_bit_exact(world):
    """Halo layout (own rows + referenced remote entries) on the CUDA shard kernels, the
    exchange emulated by sc_gather_f64 packs copied into the peers' halo slots."""
    import torch

    g = _graph()
    rp, col, val, deg = g.row_offsets, g.col_indices.astype(np.int32), g.weights, g.degrees
    starts = D.partition_rows(rp, world)
    lrps = [rp[starts[r]:starts[r + 1] + 1] - rp[starts[r]] for r in range(world)]
    lcols = [col[rp[starts[r]]:rp[starts[r + 1]]] for r in range(world)]
    plans = D.halo_plans_local(lrps, lcols, starts)
    shards = [D.CudaShard(lrps[r], plans[r].rename(lcols[r]), val[rp[starts[r]]:rp[starts[r + 1]]],
                          deg[starts[r]:starts[r + 1]], plans[r], r, 0) for r in range(world)]
    z = [[s.zeros(plans[r].ncols), s.zeros(plans[r].ncols)] for r, s in enumerate(shards)]
    x = [[s.zeros(s.n), s.zeros(s.n)] for s in shards]
    x0 = [s.zeros(s.n) for s in shards]
    idx = [[torch.from_numpy(plans[q].send_idx[r]).cuda() for r in range(world)] for q in range(world)]

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

    T = 12
    for r, s in enumerate(shards):
        s.irwin_hall(5, x0[r])
        s.scale_piece(0, x0[r], z[r][0])
    exchange(0)
    for t in range(T):
        a, b = t & 1, (t & 1) ^ 1
        for r, s in enumerate(shards):
            s.step_piece(0, z[r][a], x0[r] if t == 0 else x[r][a], x[r][b], z[r][b])
        exchange(b)
    xs = np.concatenate([s.to_original(x[r][T & 1]) for r, s in enumerate(shards)])
    fs = np.concatenate([s.to_original(s.local_z(z[r][T & 1])) for r, s in enumerate(shards)])
    xT, f = O.power_iterate(rp, col, val, deg, O.irwin_hall(deg, 5), T)
    assert np.array_equal(xs, xT)
    assert np.array_equal(fs, f)
    assert all(p.n_halo <= p.n_global - p.n for p in plans)  # never more than an all-gather
    for s in shards:
        s.close()


def _nccl_world1_worker(rank, path, out):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"file://{path}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    g = _graph()
    rp, col, val, deg = g.row_offsets, g.col_indices.astype(np.int32), g.weights, g.degrees
    starts = D.partition_rows(rp, 1)
    plan = D.exchange_plan(rp, starts, 0, 1, pieces=3)
    shard = D.CudaShard(rp, plan.rename(col), val, deg, plan, 0, 0)
    runner = D.ShardedPower(shard, plan, 0)
    runner.sample(5)
    runner.capture(12)
    res = []
    for _ in range(2):  # replay twice: the graph reads x0 and rewrites every buffer
        xT, z = runner.run(12)
        torch.cuda.synchronize()
        res.append((shard.to_original(xT), shard.to_original(shard.local_z(z))))
    np.savez(out, x1=res[0][0], f1=res[0][1], x2=res[1][0], f2=res[1][1])
    shard.close()
    dist.destroy_process_group()


def test_nccl_pipeline_cuda_graph_bit_exact(tmp_path):
    """The NCCL path end to end (world 1, 3 pieces): side-stream all-gathers and the T-step
    sequence captured in a CUDA graph, replayed twice, bit-exact against the oracle."""
    import torch.multiprocessing as mp

    out = str(tmp_path / "r.npz")
    mp.start_processes(_nccl_world1_worker, args=(str(tmp_path / "store"), out), nprocs=1,
                       join=True, start_method="spawn")
    r = np.load(out)
    g = _graph()
    x0 = O.irwin_hall(g.degrees, 5)
    xT, f = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0, 12)
    for i in (1, 2):
        assert np.array_equal(r[f"x{i}"], xT)
        assert np.array_equal(r[f"f{i}"], f)


@pytest.mark.parametrize("world", [2, 3])
def test_fused_peer_exchange_emulated_on_one_gpu(world):
    """The fused exchange (SpMV epilogue stores every z value into the peers' z allocations,
    sc_shard_set_peers): W shards in one process on one GPU, wired with each other's
    buffers; the host serialises the shards' steps on one stream (no cross-kernel waiting, so
    the barrier kernel is not used).  Bit-exact against the single-graph oracle."""
    import torch

    g = _graph()
    rp, col, val, deg = g.row_offsets, g.col_indices.astype(np.int32), g.weights, g.degrees
    starts = D.partition_rows(rp, world)
    lrps = [rp[starts[r]:starts[r + 1] + 1] - rp[starts[r]] for r in range(world)]
    plan = D.ShardPlan(starts, [D.sell_order(x) for x in lrps], [D.n_sell_rows(x) for x in lrps])
    shards = []
    for r in range(world):
        lo, hi = int(starts[r]), int(starts[r + 1])
        shards.append(D.CudaShard(lrps[r], plan.rename(col[rp[lo]:rp[hi]]), val[rp[lo]:rp[hi]],
                                  deg[lo:hi], plan, r, 0))
    comms = [D.P2PComm(s, plan, r) for r, s in enumerate(shards)]
    D.P2PComm.link_local(comms)
    runners = [D.ShardedPower(s, plan, r, comm=c) for r, (s, c) in enumerate(zip(shards, comms))]
    T = 11
    for rn in runners:
        rn.sample(5)
    for r, rn in enumerate(runners):
        rn.shard.scale_piece(0, rn.x0, rn.z[0])
    torch.cuda.synchronize()
    for t in range(T):
        a, b = t & 1, (t & 1) ^ 1
        for rn in runners:
            rn.shard.step_piece(0, rn.z[a], rn.x0 if t == 0 else rn.x[a], rn.x[b], rn.z[b])
        torch.cuda.synchronize()
    xs = np.concatenate([rn.shard.to_original(rn.x[T & 1]) for rn in runners])
    fs = np.concatenate([rn.shard.to_original(rn.shard.local_z(rn.z[T & 1])) for rn in runners])
    # every rank holds the whole z space
    for rn in runners[1:]:
        assert np.array_equal(rn.z[T & 1].cpu().numpy(), runners[0].z[T & 1].cpu().numpy())
    x0 = O.irwin_hall(deg, 5)
    xT, f = O.power_iterate(rp, col, val, deg, x0, T)
    assert np.array_equal(xs, xT)
    assert np.array_equal(fs, f)
    for s in shards:
        s.close()


def test_peer_exchange_requires_own_buffers():
    """With peers set, a z_out outside the handle's mirrored allocation is refused."""
    from paper_2310_10939_b200.errors import SpeclusterError

    g = _graph(n=600, m=5000)
    rp, col, val, deg = g.row_offsets, g.col_indices.astype(np.int32), g.weights, g.degrees
    starts = D.partition_rows(rp, 2)
    lrps = [rp[starts[r]:starts[r + 1] + 1] - rp[starts[r]] for r in range(2)]
    plan = D.ShardPlan(starts, [D.sell_order(x) for x in lrps], [D.n_sell_rows(x) for x in lrps])
    shards = [D.CudaShard(lrps[r], plan.rename(col[rp[int(starts[r])]:rp[int(starts[r + 1])]]),
                          val[rp[int(starts[r])]:rp[int(starts[r + 1])]],
                          deg[int(starts[r]):int(starts[r + 1])], plan, r, 0) for r in range(2)]
    comms = [D.P2PComm(s, plan, r) for r, s in enumerate(shards)]
    D.P2PComm.link_local(comms)
    x = shards[0].zeros(shards[0].n)
    with pytest.raises(SpeclusterError, match="z buffers"):
        shards[0].scale_piece(0, x, shards[0].zeros(plan.ncols))
    for s in shards:
        s.close()


@pytest.mark.parametrize("world", [1, 3])
def test_shards_from_device_csr_bit_exact(world):
    """The strong-scaling setup of bench_main: every rank keeps its entry-balanced row block of
    a DEVICE-generated graph, columns renamed on the device (sc_shard_create_from_csr); a
    weighted heavy-tailed DC-SBM with wide rows, exchange emulated by device copies."""
    import torch

    from paper_2310_10939_b200.generate import DeviceCSR

    with DeviceCSR.dcsbm(120_000, 6, 3) as d:
        g = d.download().graph
        rp, col, val, deg = g.row_offsets, g.col_indices, g.weights, g.degrees
        starts = D.entry_balanced_starts(rp, world)
        lrps = [rp[starts[r]:starts[r + 1] + 1] - rp[starts[r]] for r in range(world)]
        plan = D.ShardPlan(starts, [D.sell_order(x) for x in lrps],
                           [D.n_sell_rows(x) for x in lrps], 1, 8192)
        shards = [D.CudaShard.from_device_csr(d, plan, r, 0) for r in range(world)]
    assert any(s.n > 0 for s in shards)
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
    xo, fo = O.power_iterate(rp, col, val, deg, O.irwin_hall(deg, 2), T)
    assert np.array_equal(xs, xo)
    for s in shards:
        s.close()
