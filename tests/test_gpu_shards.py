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


@pytest.mark.parametrize("world", [1, 3])
def test_shards_on_one_gpu_bit_exact(world):
    import torch

    g = _graph()
    rp, col, val, deg = g.row_offsets, g.col_indices.astype(np.int32), g.weights, g.degrees
    starts = D.partition_rows(rp, world)
    perms = [D.sell_order(rp[starts[r]:starts[r + 1] + 1] - rp[starts[r]]) for r in range(world)]
    plan = D.ShardPlan(starts, perms)
    shards = []
    for r in range(world):
        lo, hi = int(starts[r]), int(starts[r + 1])
        lrp = rp[lo:hi + 1] - rp[lo]
        shards.append(D.CudaShard(lrp, plan.rename(col[rp[lo]:rp[hi]]), val[rp[lo]:rp[hi]],
                                  deg[lo:hi], plan, r, 0))
    T = 12
    z = [[s.zeros(plan.ncols), s.zeros(plan.ncols)] for s in shards]
    x = [[s.zeros(s.n), s.zeros(s.n)] for s in shards]
    x0 = [s.zeros(s.n) for s in shards]

    def gather(buf_index):
        for r in range(world):
            src = z[r][buf_index][r * plan.n_max:(r + 1) * plan.n_max]
            for q in range(world):
                if q != r:
                    z[q][buf_index][r * plan.n_max:(r + 1) * plan.n_max].copy_(src)

    for r, s in enumerate(shards):
        s.irwin_hall(5, x0[r])
        s.scale(x0[r], z[r][0])
    torch.cuda.synchronize()
    gather(0)
    for t in range(T):
        a, b = t & 1, (t & 1) ^ 1
        for r, s in enumerate(shards):
            s.step(z[r][a], x0[r] if t == 0 else x[r][a], x[r][b], z[r][b])
        torch.cuda.synchronize()
        gather(b)
    torch.cuda.synchronize()
    xs = np.concatenate([s.to_original(x[r][T & 1]) for r, s in enumerate(shards)])
    fs = np.concatenate([s.to_original(z[r][T & 1][r * plan.n_max:]) for r, s in enumerate(shards)])
    x0_ref = O.irwin_hall(deg, 5)
    x0_dev = np.concatenate([s.to_original(x0[r]) for r, s in enumerate(shards)])
    assert np.array_equal(x0_dev, x0_ref)
    xT, f = O.power_iterate(rp, col, val, deg, x0_ref, T)
    assert np.array_equal(xs, xT)
    assert np.array_equal(fs, f)
    for s in shards:
        s.close()
