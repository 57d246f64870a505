"""Row-block sharding of the one-vector power iteration over 1/2/4/8 GPUs.

One process per GPU (``torchrun``); ``torch.distributed`` is the plumbing.  Every rank owns a
contiguous block of rows (balanced by stored entries) and its slot of the gathered vector
z = D^-1 x; per step:

    local SpMV over the shard (sc_shard_step, writes the rank's own z slot)
    all-gather of the z slots (NCCL over NVLink / NVSwitch)

The device layout renumbers each shard's rows (SELL-32-sigma, ``sc_sell_order``); every rank
learns all ranks' renumberings once and renames its columns into the global renumbered z
space, whose slot r starts at r * n_max.  Rows are never split across ranks, so every row is
still summed in scipy's order and the multi-GPU x_T / f are bit-identical to one GPU's.

The compute backend is pluggable: ``CudaShard`` (the product: libsc_b200.so on the rank's
GPU) and, in the CPU tests only, an oracle backend -- the host protocol (partitioning,
renumbering exchange, column renaming, slot layout, all-gather) is the same code.
"""

from __future__ import annotations

import ctypes
import json
import os
import time

import numpy as np

from . import _lib
from .errors import InputError


# ---------------------------------------------------------------------------
# host-side plan


def partition_rows(row_ptr: np.ndarray, world: int) -> np.ndarray:
    """Contiguous row blocks with balanced work (stored entries + 1 per row)."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    n = row_ptr.size - 1
    if world < 1 or world > n:
        raise InputError(f"cannot split {n} rows over {world} ranks")
    cost = row_ptr + np.arange(n + 1, dtype=np.int64)
    targets = (cost[-1] * np.arange(world + 1, dtype=np.float64) / world)
    starts = np.searchsorted(cost, targets, side="left").astype(np.int64)
    starts[0], starts[-1] = 0, n
    for r in range(1, world):  # every rank gets at least one row
        starts[r] = min(max(starts[r], starts[r - 1] + 1), n - (world - r))
    return starts


def sell_order(row_ptr: np.ndarray) -> np.ndarray:
    """The device renumbering of a (local) row_ptr: perm[p] = original row of row p."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    perm = np.empty(rp.size - 1, dtype=np.int32)
    _lib.check(_lib.load().sc_sell_order(_lib.ptr(rp), rp.size - 1, _lib.ptr(perm)))
    return perm


class ShardPlan:
    """Row blocks, every rank's renumbering and the global renumbered z space."""

    def __init__(self, starts, perms):
        self.starts = np.asarray(starts, dtype=np.int64)
        self.world = self.starts.size - 1
        self.sizes = np.diff(self.starts)
        self.n_global = int(self.starts[-1])
        self.n_max = int(self.sizes.max())
        self.perms = [np.asarray(p, dtype=np.int32) for p in perms]
        # z slot of every global (original) vertex id
        slot = np.empty(self.n_global, dtype=np.int64)
        for r, p in enumerate(self.perms):
            inv = np.empty(p.size, dtype=np.int64)
            inv[p] = np.arange(p.size, dtype=np.int64)
            slot[self.starts[r]:self.starts[r + 1]] = r * self.n_max + inv
        self.slot_of = slot

    @property
    def ncols(self) -> int:
        return self.world * self.n_max

    def rename(self, col_global: np.ndarray) -> np.ndarray:
        return self.slot_of[np.asarray(col_global, dtype=np.int64)].astype(np.int32)

    def owner(self, v: int) -> int:
        return int(np.searchsorted(self.starts, v, side="right") - 1)


def exchange_plan(local_row_ptr: np.ndarray, starts: np.ndarray, rank: int, world: int,
                  group=None) -> ShardPlan:
    """Every rank computes its renumbering and all-gathers it (padded to n_max)."""
    import torch
    import torch.distributed as dist

    perm = sell_order(local_row_ptr)
    n_max = int(np.diff(starts).max())
    buf = torch.full((n_max,), -1, dtype=torch.int32)
    buf[: perm.size] = torch.from_numpy(perm)
    dev = _group_device(group)
    out = [torch.empty(n_max, dtype=torch.int32, device=dev) for _ in range(world)]
    dist.all_gather(out, buf.to(dev), group=group)
    perms = [out[r][: int(starts[r + 1] - starts[r])].cpu().numpy() for r in range(world)]
    return ShardPlan(starts, perms)


def _group_device(group):
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


# ---------------------------------------------------------------------------
# backends


class CudaShard:
    """The product backend: one sc_graph shard on the rank's GPU, buffers are torch tensors
    on the same device, kernels run on torch's current stream."""

    def __init__(self, rp, col_renamed, val, deg, plan: ShardPlan, rank: int, device: int):
        import torch

        L = _lib.require_device()
        self.rank, self.plan, self.device = rank, plan, device
        self.n = int(plan.sizes[rank])
        self.off = rank * plan.n_max
        self._keep = (np.ascontiguousarray(rp, dtype=np.int64),
                      np.ascontiguousarray(col_renamed, dtype=np.int32),
                      None if val is None else np.ascontiguousarray(val, dtype=np.float64),
                      np.ascontiguousarray(deg, dtype=np.float64))
        rp_, col_, val_, deg_ = self._keep
        h = ctypes.c_void_p()
        _lib.check(L.sc_shard_create(_lib.ptr(rp_), _lib.ptr(col_), _lib.ptr(val_), _lib.ptr(deg_),
                                     self.n, int(rp_[-1]), plan.ncols, self.off,
                                     int(plan.starts[rank]), device, ctypes.byref(h)))
        self.h = h
        self.torch = torch
        self.tdev = torch.device("cuda", device)

    def close(self):
        if self.h:
            _lib.load().sc_graph_destroy(self.h)
            self.h = None

    def zeros(self, m):
        return self.torch.zeros(m, dtype=self.torch.float64, device=self.tdev)

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.tdev).cuda_stream)

    def irwin_hall(self, seed, x_out):
        from .spectral import irwin_hall_key

        k0, k1 = irwin_hall_key(seed)
        _lib.check(_lib.load().sc_shard_irwin_hall(self.h, k0, k1, ctypes.c_void_p(x_out.data_ptr()),
                                                   self._stream()))

    def scale(self, x, z_full, sym=False):
        _lib.check(_lib.load().sc_shard_scale(self.h, ctypes.c_void_p(x.data_ptr()),
                                              ctypes.c_void_p(z_full.data_ptr()),
                                              _lib.SC_SYM_VARIANT if sym else 0, self._stream()))

    def step(self, z_in, x_in, x_out, z_out, sign=1.0, sym=False):
        _lib.check(_lib.load().sc_shard_step(
            self.h, ctypes.c_void_p(z_in.data_ptr()), ctypes.c_void_p(x_in.data_ptr()),
            ctypes.c_void_p(x_out.data_ptr()), ctypes.c_void_p(z_out.data_ptr()), float(sign),
            _lib.SC_SYM_VARIANT if sym else 0, self._stream()))

    def to_original(self, v_local):
        """renumbered local vector -> numpy array in original local order"""
        perm = self.plan.perms[self.rank]
        out = np.empty(self.n)
        out[perm] = v_local[: self.n].cpu().numpy()
        return out


def allgather_slots(z_full, plan: ShardPlan, rank: int, group=None):
    """In-place all-gather of the ranks' z slots (equal slot size n_max)."""
    import torch.distributed as dist

    own = z_full[rank * plan.n_max:(rank + 1) * plan.n_max]
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(z_full, own, group=group)
    else:
        parts = [z_full[r * plan.n_max:(r + 1) * plan.n_max] for r in range(plan.world)]
        dist.all_gather(parts, own.clone(), group=group)


def power_iterate_sharded(shard, plan: ShardPlan, rank: int, T: int, *, seed: int | None = 0,
                          x0_local_renumbered=None, sign: float = 1.0, sym: bool = False,
                          group=None):
    """T steps over the shards; returns (x_T local renumbered, z_T = f local renumbered)."""
    n = int(plan.sizes[rank])
    z = [shard.zeros(plan.ncols), shard.zeros(plan.ncols)]
    x = [shard.zeros(n), shard.zeros(n)]
    x0 = shard.zeros(n)
    if x0_local_renumbered is not None:
        x0.copy_(x0_local_renumbered)
    else:
        shard.irwin_hall(seed, x0)
    off = rank * plan.n_max
    shard.scale(x0, z[0], sym)
    allgather_slots(z[0], plan, rank, group)
    for t in range(T):
        a, b = t & 1, (t & 1) ^ 1
        shard.step(z[a], x0 if t == 0 else x[a], x[b], z[b], sign, sym)
        allgather_slots(z[b], plan, rank, group)
    xT = x0 if T == 0 else x[T & 1]
    return xT, z[T & 1][off:off + n]


# ---------------------------------------------------------------------------
# multi-GPU bench (bench.py --gpus N under torchrun)


def _init_dist():
    import torch
    import torch.distributed as dist

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def bench_main(args, metric: str, unit: str):
    """Weak scaling: rank r owns one config-2 sized row block (1e6 rows, 10 SBM blocks) of an
    SBM with n = N * 1e6, k = 10 N, expected in-block degree 40 and out-of-block degree 4;
    T = 100 steps with an NCCL all-gather of z after each."""
    import torch
    import torch.distributed as dist

    from .generate import SbmParams, sbm_rows

    rank, world, local = _init_dist()
    n_loc = 10**6
    params = SbmParams(n=world * n_loc, k=10 * world, p=40 / (10**5 - 1),
                       q=4 / (world * n_loc - 10**5), seed=0)
    T = 100
    starts = np.arange(world + 1, dtype=np.int64) * n_loc
    rp, col, deg, iso = sbm_rows(params, int(starts[rank]), int(starts[rank + 1]))
    iso_t = torch.tensor([iso], device="cuda")
    dist.all_reduce(iso_t)
    if int(iso_t.item()):
        raise InputError("isolated vertices in the scaling graph; choose another seed")
    plan = exchange_plan(rp, starts, rank, world)
    shard = CudaShard(rp, plan.rename(col), None, deg, plan, rank, local)
    nnz_t = torch.tensor([int(rp[-1])], device="cuda", dtype=torch.int64)
    dist.all_reduce(nnz_t)
    nnz_total = int(nnz_t.item())
    stream = torch.cuda.current_stream()

    def one_step():
        return power_iterate_sharded(shard, plan, rank, T, seed=0)

    for _ in range(max(args.warmup, 3)):
        one_step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        one_step()
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], device="cuda", dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    tot_ms = float(ms.item())
    # all-gather alone (NVLink): T gathers of the z space
    zbuf = shard.zeros(plan.ncols)
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(stream)
    for _ in range(T):
        allgather_slots(zbuf, plan, rank)
    e1.record(stream)
    torch.cuda.synchronize()
    ag = torch.tensor([e0.elapsed_time(e1) / T], device="cuda", dtype=torch.float64)
    dist.all_reduce(ag, op=dist.ReduceOp.MAX)
    ag_ms = float(ag.item())
    recv_bytes = (world - 1) * plan.n_max * 8
    if rank == 0:
        value = nnz_total * T * args.steps / (tot_ms / 1e3) / 1e9
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config2 block per GPU (SBM n={params.n}, k={params.k})",
                       "n_per_gpu": n_loc, "nnz_total": nnz_total, "T": T,
                       "parallelism": f"row-block shards x{world}, NCCL all-gather of z per step"},
            "allgather": {"ms_per_step": ag_ms, "recv_bytes_per_gpu": recv_bytes,
                          "gbs_per_gpu": recv_bytes / (ag_ms / 1e3) / 1e9},
            "gpu_launches": args.steps * (T + 1),
        }
        print(json.dumps(line), flush=True)
    shard.close()
    dist.destroy_process_group()


def gather_to_rank0(v_local_original: np.ndarray, plan: ShardPlan, rank: int, group=None):
    """Concatenate the ranks' local vectors (original order) into the global vector on rank 0."""
    import torch
    import torch.distributed as dist

    dev = _group_device(group)
    buf = torch.zeros(plan.n_max, dtype=torch.float64)
    buf[: v_local_original.size] = torch.from_numpy(np.asarray(v_local_original, dtype=np.float64))
    out = [torch.empty(plan.n_max, dtype=torch.float64, device=dev) for _ in range(plan.world)]
    dist.all_gather(out, buf.to(dev), group=group)
    if rank != 0:
        return None
    return np.concatenate([out[r][: plan.sizes[r]].cpu().numpy() for r in range(plan.world)])


def _now() -> float:
    return time.perf_counter()
