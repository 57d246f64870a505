"""Row-block sharding of the one-vector power iteration over 1/2/4/8 GPUs.

One process per GPU (``torchrun``); ``torch.distributed`` is the plumbing.  Every rank owns a
contiguous block of rows (balanced by stored entries).  A step is pipelined over P pieces of
each rank's rows:

    for piece j:  local SpMV of piece j (sc_shard_step_range) -> writes piece j of z
                  all-gather of piece j of z over NCCL, on a second stream, while the SpMV
                  of piece j+1 runs
    the next step waits for the last gather

so only the last piece's gather is exposed.  The gathered vector is laid out piece-major --
piece j of every rank sits in one contiguous block of W * pmax entries -- so every piece is a
single in-place ``all_gather_into_tensor``.

The device layout renumbers each shard's rows (SELL-32-sigma, ``sc_sell_order``); every rank
learns all ranks' renumberings once and renames its columns into the global z space.  Rows
are never split across ranks, so every row is still summed in scipy's order and the
multi-GPU x_T / f are bit-identical to one GPU's.

The compute backend is pluggable: ``CudaShard`` (the product: libsc_b200.so on the rank's
GPU) and, in the CPU tests only, an oracle backend -- the host protocol (partitioning,
renumbering exchange, column renaming, piece layout, all-gathers) is the same code.
"""

from __future__ import annotations

import ctypes
import json
import os
import sys

import numpy as np

from . import _lib
from .errors import InputError

SELL_MAX = 256  # rows longer than this are "wide" rows (sc_graph.cu kSellMax / kExtreme)
SLICE = 32


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


def n_sell_rows(row_ptr: np.ndarray) -> int:
    """Renumbered rows laid out as SELL slices (the rest are wide rows)."""
    return int(np.count_nonzero(np.diff(np.asarray(row_ptr)) <= SELL_MAX))


def piece_bounds(n: int, n_sell: int, pieces: int) -> np.ndarray:
    """P contiguous pieces of a renumbered shard; boundaries inside the SELL rows are
    slice aligned (the kernel processes whole 32-row slices)."""
    b = np.array([j * n // pieces for j in range(pieces + 1)], dtype=np.int64)
    inside = b < n_sell
    b[inside] = (b[inside] // SLICE) * SLICE
    b[0], b[-1] = 0, n
    return np.maximum.accumulate(b)


class ShardPlan:
    """Row blocks, every rank's renumbering, the pieces and the global z space."""

    def __init__(self, starts, perms, n_sells=None, pieces: int = 1, align: int = 1):
        """``align``: round every rank's z block up to a multiple of this many slots (8192
        keeps the 4096-row renumbering windows inside 8192-column panels, so the column-panel
        layout sees every row's columns in panel order)."""
        self.starts = np.asarray(starts, dtype=np.int64)
        self.world = self.starts.size - 1
        self.sizes = np.diff(self.starts)
        self.n_global = int(self.starts[-1])
        self.perms = [np.asarray(p, dtype=np.int32) for p in perms]
        self.pieces = int(pieces)
        if n_sells is None:
            n_sells = list(self.sizes)
        self.n_sells = [int(v) for v in n_sells]
        self.bounds = [piece_bounds(int(self.sizes[r]), self.n_sells[r], self.pieces)
                       for r in range(self.world)]
        self.pmax = max(1, int(max(np.diff(b).max() for b in self.bounds)))
        self.pmax = -(-self.pmax // int(align)) * int(align)
        self.n_max = int(self.sizes.max())
        # z slot of every global (original) vertex id
        slot = np.empty(self.n_global, dtype=np.int64)
        for r, p in enumerate(self.perms):
            inv = np.empty(p.size, dtype=np.int64)
            inv[p] = np.arange(p.size, dtype=np.int64)  # original local -> renumbered
            b = self.bounds[r]
            piece = np.searchsorted(b, inv, side="right") - 1
            slot[self.starts[r]:self.starts[r + 1]] = (
                piece * self.world * self.pmax + r * self.pmax + (inv - b[piece]))
        self.slot_of = slot

    @property
    def ncols(self) -> int:
        return self.pieces * self.world * self.pmax

    def block(self, j: int) -> tuple[int, int]:
        """z range of piece j (all ranks)."""
        w = self.world * self.pmax
        return j * w, (j + 1) * w

    def own(self, j: int, rank: int) -> tuple[int, int]:
        """z range owned by `rank` in piece j (length pmax)."""
        lo = j * self.world * self.pmax + rank * self.pmax
        return lo, lo + self.pmax

    def rename(self, col_global: np.ndarray) -> np.ndarray:
        return self.slot_of[np.asarray(col_global, dtype=np.int64)].astype(np.int32)

    def owner(self, v: int) -> int:
        return int(np.searchsorted(self.starts, v, side="right") - 1)


def exchange_plan(local_row_ptr: np.ndarray, starts: np.ndarray, rank: int, world: int,
                  group=None, pieces: int = 1, align: int = 1) -> ShardPlan:
    """Every rank computes its renumbering and all-gathers it (padded to n_max)."""
    import torch
    import torch.distributed as dist

    perm = sell_order(local_row_ptr)
    n_max = int(np.diff(starts).max())
    buf = torch.full((n_max + 1,), -1, dtype=torch.int32)
    buf[: perm.size] = torch.from_numpy(perm)
    buf[n_max] = n_sell_rows(local_row_ptr)
    dev = _group_device(group)
    out = [torch.empty(n_max + 1, dtype=torch.int32, device=dev) for _ in range(world)]
    dist.all_gather(out, buf.to(dev), group=group)
    perms = [out[r][: int(starts[r + 1] - starts[r])].cpu().numpy() for r in range(world)]
    n_sells = [int(out[r][n_max].item()) for r in range(world)]
    return ShardPlan(starts, perms, n_sells, pieces, align)


class HaloPlan:
    """z space of one rank for the halo exchange (SURVEY §8(e) option 2): the remote entries
    its rows reference, grouped by owner rank and sorted by global id, with the rank's own rows
    (renumbered order) in between -- owners below the rank first, then the own rows starting on
    an 8192-slot boundary (``base``), then owners above.  That keeps every row's renamed
    columns in stored (global id) order across 8192-column panels, so the column-panel layout
    applies to halo shards too.  Per step every rank sends each peer only the own entries that
    peer references (``send_idx``: z-space slots of its own rows, in the peer's halo order) --
    at config 5 on 8 GPUs ~19 M entries per GPU instead of the 87.5 M an all-gather delivers.
    Columns are only renamed, never reordered, so results stay bit-identical.

    Exposes the ShardPlan attributes CudaShard uses (one piece)."""

    def __init__(self, starts, rank, perm, n_sell, halo_ids, send_idx):
        self.starts = np.asarray(starts, dtype=np.int64)
        self.world = self.starts.size - 1
        self.sizes = np.diff(self.starts)
        self.n_global = int(self.starts[-1])
        self.rank = rank
        n = int(self.sizes[rank])
        self.n = n
        self.perms = [None] * self.world
        self.perms[rank] = np.asarray(perm, dtype=np.int32)
        self.n_sells = [0] * self.world
        self.n_sells[rank] = int(n_sell)
        self.pieces = 1
        self.bounds = [np.array([0, int(sz)], dtype=np.int64) for sz in self.sizes]
        self.halo_ids = [np.asarray(h, dtype=np.int64) for h in halo_ids]  # per owner
        cnt = np.array([h.size for h in self.halo_ids], dtype=np.int64)
        self.n_low = int(cnt[:rank].sum())                      # halo entries of lower owners
        self.base = -(-self.n_low // 8192) * 8192               # first own slot
        off = np.concatenate([[0], np.cumsum(cnt)])
        off[rank + 1:] += self.base + n - self.n_low            # higher owners after own rows
        # owner q != rank: halo slots [off[q], off[q+1]).  off[rank] .. off[rank+1] spans the
        # alignment padding and the own rows, so it is NOT a halo range -- use halo_range(q).
        self.halo_off = off
        self.send_idx = [np.asarray(h, dtype=np.int64).astype(np.int32) + self.base
                         for h in send_idx]  # per peer, z-space slots of own rows
        self.n_halo = int(cnt.sum())
        self.pmax = n
        self.n_max = int(self.sizes.max())
        inv = np.empty(n, dtype=np.int64)
        inv[self.perms[rank]] = np.arange(n, dtype=np.int64)
        self._inv = inv
        self._halo_all = (np.concatenate(self.halo_ids) if self.halo_ids
                          else np.empty(0, dtype=np.int64))

    @property
    def ncols(self) -> int:
        return self.base + self.n + self.n_halo - self.n_low

    def halo_range(self, q: int) -> tuple[int, int]:
        """z-space slots [a, b) that receive owner q's entries (q != rank)."""
        if q == self.rank:
            raise ValueError("a rank has no halo range of its own")
        return int(self.halo_off[q]), int(self.halo_off[q + 1])

    def own(self, j: int, rank: int) -> tuple[int, int]:
        return self.base, self.base + self.n

    def rename(self, col_global: np.ndarray) -> np.ndarray:
        c = np.asarray(col_global, dtype=np.int64)
        lo, hi = int(self.starts[self.rank]), int(self.starts[self.rank + 1])
        out = np.empty(c.size, dtype=np.int64)
        mine = (c >= lo) & (c < hi)
        out[mine] = self.base + self._inv[c[mine] - lo]
        # halo ids are sorted within each owner and owners are ordered by id range, so the
        # concatenation is globally sorted; lower owners' entries sit below the own rows
        pos = np.searchsorted(self._halo_all, c[~mine])
        out[~mine] = np.where(pos < self.n_low, pos, pos - self.n_low + self.base + self.n)
        return out.astype(np.int32)


def halo_plans_local(local_row_ptrs, local_cols_global, starts) -> list:
    """All ranks' HaloPlans computed in one process (single-GPU emulation and tests): the
    same lists exchange_halo_plan builds with point-to-point messages."""
    starts = np.asarray(starts, dtype=np.int64)
    world = starts.size - 1
    perms, halos = [], []
    for r in range(world):
        lo, hi = int(starts[r]), int(starts[r + 1])
        col = np.asarray(local_cols_global[r], dtype=np.int64)
        remote = np.unique(col[(col < lo) | (col >= hi)])
        owner = np.searchsorted(starts, remote, side="right") - 1
        halos.append([remote[owner == q] for q in range(world)])
        perms.append(sell_order(local_row_ptrs[r]))
    plans = []
    for r in range(world):
        lo, hi = int(starts[r]), int(starts[r + 1])
        inv = np.empty(hi - lo, dtype=np.int64)
        inv[perms[r]] = np.arange(hi - lo, dtype=np.int64)
        send = [np.empty(0, dtype=np.int32) if q == r else inv[halos[q][r] - lo].astype(np.int32)
                for q in range(world)]
        plans.append(HaloPlan(starts, r, perms[r], n_sell_rows(local_row_ptrs[r]), halos[r], send))
    return plans


def exchange_halo_plan(local_row_ptr: np.ndarray, local_col_global: np.ndarray,
                       starts: np.ndarray, rank: int, world: int, group=None) -> HaloPlan:
    """Every rank lists the remote vertices its rows reference (per owner), sends each owner
    its list and receives the lists the peers need from it, translated to its renumbered
    local slots."""
    import torch
    import torch.distributed as dist

    starts = np.asarray(starts, dtype=np.int64)
    lo, hi = int(starts[rank]), int(starts[rank + 1])
    perm = sell_order(local_row_ptr)
    n_sell = n_sell_rows(local_row_ptr)
    col = np.asarray(local_col_global, dtype=np.int64)
    remote = np.unique(col[(col < lo) | (col >= hi)])
    owner = np.searchsorted(starts, remote, side="right") - 1
    halo_ids = [remote[owner == q] for q in range(world)]
    dev = _group_device(group)
    cnt = torch.tensor([h.size for h in halo_ids], dtype=torch.int64, device=dev)
    all_cnt = [torch.empty(world, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(all_cnt, cnt, group=group)
    need_from_me = [int(all_cnt[q][rank].item()) for q in range(world)]  # peer q asks me
    ops, recv = [], [None] * world
    for q in range(world):
        if q == rank:
            continue
        if halo_ids[q].size:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(halo_ids[q]).to(dev), q, group))
        if need_from_me[q]:
            recv[q] = torch.empty(need_from_me[q], dtype=torch.int64, device=dev)
            ops.append(dist.P2POp(dist.irecv, recv[q], q, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    inv = np.empty(hi - lo, dtype=np.int64)
    inv[perm] = np.arange(hi - lo, dtype=np.int64)
    send_idx = [np.empty(0, dtype=np.int32) if recv[q] is None
                else inv[recv[q].cpu().numpy() - lo].astype(np.int32) for q in range(world)]
    return HaloPlan(starts, rank, perm, n_sell, halo_ids, send_idx)


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
        self._keep = (np.ascontiguousarray(rp, dtype=np.int64),
                      np.ascontiguousarray(col_renamed, dtype=np.int32),
                      None if val is None else np.ascontiguousarray(val, dtype=np.float64),
                      np.ascontiguousarray(deg, dtype=np.float64))
        rp_, col_, val_, deg_ = self._keep
        h = ctypes.c_void_p()
        _lib.check(L.sc_shard_create(_lib.ptr(rp_), _lib.ptr(col_), _lib.ptr(val_), _lib.ptr(deg_),
                                     self.n, int(rp_[-1]), plan.ncols, 0, int(plan.starts[rank]),
                                     device, ctypes.byref(h)))
        self.h = h
        gi = _lib.GraphInfo()
        _lib.check(L.sc_graph_info_get(h, ctypes.byref(gi)))
        if self.n - gi.long_rows != plan.n_sells[rank]:
            raise InputError("shard layout disagrees with the plan's SELL row count")
        self.torch = torch
        self.tdev = torch.device("cuda", device)

    @classmethod
    def from_device_csr(cls, csr, plan: ShardPlan, rank: int, device: int):
        """The rank's row block straight from a device-resident CSR of the whole graph on
        `device` (sc_shard_create_from_csr): columns renamed on the device through the plan's
        slot map, nothing but row offsets and degrees of the block visits the host."""
        import torch

        L = _lib.require_device()
        self = cls.__new__(cls)
        self.rank, self.plan, self.device = rank, plan, device
        self.n = int(plan.sizes[rank])
        self._keep = ()
        slot = torch.from_numpy(plan.slot_of.astype(np.int32)).to(torch.device("cuda", device))
        lo, hi = int(plan.starts[rank]), int(plan.starts[rank + 1])
        h = ctypes.c_void_p()
        _lib.check(L.sc_shard_create_from_csr(csr.handle, lo, hi, ctypes.c_void_p(slot.data_ptr()),
                                              plan.ncols, 0, ctypes.byref(h)))
        del slot
        self.h = h
        gi = _lib.GraphInfo()
        _lib.check(L.sc_graph_info_get(h, ctypes.byref(gi)))
        if self.n - gi.long_rows != plan.n_sells[rank]:
            raise InputError("shard layout disagrees with the plan's SELL row count")
        self.torch = torch
        self.tdev = torch.device("cuda", device)
        return self

    def close(self):
        if self.h:
            _lib.load().sc_graph_destroy(self.h)
            self.h = None

    def zeros(self, m):
        return self.torch.zeros(m, dtype=self.torch.float64, device=self.tdev)

    def zspace(self, m):
        """a z-space buffer of m doubles followed by 16 zeros that are never written: the
        padding target of the column-panel layout (sc_graph_build_panels contract); the
        returned view covers the first m"""
        return self.zeros(m + 16)[:m]

    def build_panels(self) -> bool:
        """column-panel layout for full-shard steps (pieces = 1); False if declined"""
        _lib.check(_lib.load().sc_graph_build_panels(self.h))
        gi = _lib.GraphInfo()
        _lib.check(_lib.load().sc_graph_info_get(self.h, ctypes.byref(gi)))
        return gi.panel_groups > 0

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.tdev).cuda_stream)

    def _zout(self, z_full, j):
        """pointer such that z_out[row] lands in this rank's slot of piece j"""
        lo = int(self.plan.bounds[self.rank][j])
        off = int(self.plan.own(j, self.rank)[0]) - lo
        return ctypes.c_void_p(z_full.data_ptr() + 8 * off)

    def irwin_hall(self, seed, x_out):
        from .spectral import irwin_hall_key

        k0, k1 = irwin_hall_key(seed)
        _lib.check(_lib.load().sc_shard_irwin_hall(self.h, k0, k1, ctypes.c_void_p(x_out.data_ptr()),
                                                   self._stream()))

    def scale_piece(self, j, x, z_full, sym=False):
        b = self.plan.bounds[self.rank]
        _lib.check(_lib.load().sc_shard_scale_range(
            self.h, int(b[j]), int(b[j + 1]), ctypes.c_void_p(x.data_ptr()), self._zout(z_full, j),
            _lib.SC_SYM_VARIANT if sym else 0, self._stream()))

    def step_piece(self, j, z_in, x_in, x_out, z_out, sign=1.0, sym=False):
        b = self.plan.bounds[self.rank]
        _lib.check(_lib.load().sc_shard_step_range(
            self.h, int(b[j]), int(b[j + 1]), ctypes.c_void_p(z_in.data_ptr()),
            ctypes.c_void_p(x_in.data_ptr()), ctypes.c_void_p(x_out.data_ptr()),
            self._zout(z_out, j), float(sign), _lib.SC_SYM_VARIANT if sym else 0, self._stream()))

    def pack(self, z_full, idx, out):
        """out[i] = z_full[idx[i]] (idx: int32 device tensor) -- the halo send buffer"""
        _lib.check(_lib.load().sc_gather_f64(ctypes.c_void_p(z_full.data_ptr()),
                                             ctypes.c_void_p(idx.data_ptr()), int(idx.numel()),
                                             ctypes.c_void_p(out.data_ptr()), self._stream()))

    def local_z(self, z_full):
        """this rank's z entries (renumbered local order) as a host array"""
        b = self.plan.bounds[self.rank]
        parts = []
        for j in range(self.plan.pieces):
            lo = self.plan.own(j, self.rank)[0]
            parts.append(z_full[lo:lo + int(b[j + 1] - b[j])].cpu().numpy())
        return np.concatenate(parts)

    def z_views(self):
        """(z0, z1) torch views over the handle's own z allocation, and its flag array address
        (the buffers the fused peer exchange mirrors, sc_shard_buffers)."""
        zb, fl = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(_lib.load().sc_shard_buffers(self.h, ctypes.byref(zb), ctypes.byref(fl)))
        nc = self.plan.ncols
        gi = _lib.GraphInfo()
        _lib.check(_lib.load().sc_graph_info_get(self.h, ctypes.byref(gi)))
        z0 = _device_view(zb.value, nc, self.device)
        z1 = _device_view(zb.value + 8 * gi.zstride, nc, self.device)
        return z0, z1, zb.value, fl.value

    def to_original(self, v_local):
        """renumbered local vector (tensor or array) -> array in original local order"""
        v = v_local.cpu().numpy() if hasattr(v_local, "cpu") else np.asarray(v_local)
        out = np.empty(self.n)
        out[self.plan.perms[self.rank]] = v[: self.n]
        return out


def _device_view(ptr: int, count: int, device: int):
    """Zero-copy float64 torch tensor over device memory owned by the library
    (__cuda_array_interface__ import)."""
    import torch

    class _Cai:
        __cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_Cai(), device=torch.device("cuda", device))


class P2PComm:
    """Fused exchange: the step kernels store every z value straight into the peers' z
    allocations over NVLink (sc_shard_set_peers), so there is nothing to gather; ``finish``
    launches the system-scope flag barrier that ends a step.  ``link`` exchanges CUDA IPC
    handles with the other ranks; ``link_local`` wires shards living in one process (the
    single-GPU emulation used by the tests, where the host serialises the steps instead of
    a barrier)."""

    def __init__(self, shard, plan: ShardPlan, rank: int):
        import torch

        self.torch = torch
        self.shard, self.plan, self.rank = shard, plan, rank
        self.z0, self.z1, self.zbase, self.flags = shard.z_views()
        self._opened = []
        self.barrier = True

    def link(self, group=None):
        import torch.distributed as dist

        L = _lib.load()
        world = self.plan.world
        hz, hf = ctypes.create_string_buffer(64), ctypes.create_string_buffer(64)
        _lib.check(L.sc_ipc_export(ctypes.c_void_p(self.zbase), hz))
        _lib.check(L.sc_ipc_export(ctypes.c_void_p(self.flags), hf))
        handles = [None] * world
        dist.all_gather_object(handles, (hz.raw, hf.raw), group=group)
        zs, fs = [], []
        for q, (a, b) in enumerate(handles):
            if q == self.rank:
                zs.append(self.zbase)
                fs.append(self.flags)
                continue
            pz, pf = ctypes.c_void_p(), ctypes.c_void_p()
            _lib.check(L.sc_ipc_import(a, self.shard.device, ctypes.byref(pz)))
            _lib.check(L.sc_ipc_import(b, self.shard.device, ctypes.byref(pf)))
            self._opened += [pz.value, pf.value]
            zs.append(pz.value)
            fs.append(pf.value)
        self._set(zs, fs)

    @staticmethod
    def link_local(comms):
        zs = [c.zbase for c in comms]
        fs = [c.flags for c in comms]
        for c in comms:
            c._set(zs, fs)
            c.barrier = False

    def _set(self, zs, fs):
        arr = ctypes.c_void_p * len(zs)
        _lib.check(_lib.load().sc_shard_set_peers(self.shard.h, arr(*zs), arr(*fs), len(zs),
                                                  self.rank))

    def gather_piece(self, z_full, j):
        pass  # the SpMV epilogue already stored this piece into every peer

    def finish(self):
        if self.barrier:
            stream = self.torch.cuda.current_stream().cuda_stream
            _lib.check(_lib.load().sc_shard_barrier(self.shard.h, ctypes.c_void_p(stream)))

    def close(self):
        L = _lib.load()
        for p in self._opened:
            L.sc_ipc_release(ctypes.c_void_p(p))
        self._opened = []


class PieceComm:
    """All-gathers of z pieces.  NCCL: each piece's gather runs on a side stream after an
    event recorded behind that piece's SpMV, overlapping the next piece's SpMV; gloo
    (CPU tests): synchronous."""

    def __init__(self, plan: ShardPlan, rank: int, group=None):
        import torch.distributed as dist

        self.plan, self.rank, self.group = plan, rank, group
        self.nccl = dist.get_backend(group) == "nccl"
        if self.nccl:
            import torch

            self.torch = torch
            self.side = torch.cuda.Stream()

    def gather_piece(self, z_full, j):
        import torch.distributed as dist

        lo, hi = self.plan.block(j)
        own_lo, own_hi = self.plan.own(j, self.rank)
        if self.nccl:
            torch = self.torch
            main = torch.cuda.current_stream()
            self.side.wait_stream(main)
            with torch.cuda.stream(self.side):
                dist.all_gather_into_tensor(z_full[lo:hi], z_full[own_lo:own_hi], group=self.group)
        else:
            pm = self.plan.pmax
            parts = [z_full[lo + r * pm:lo + (r + 1) * pm] for r in range(self.plan.world)]
            dist.all_gather(parts, z_full[own_lo:own_hi].clone(), group=self.group)

    def finish(self):
        if self.nccl:
            self.torch.cuda.current_stream().wait_stream(self.side)


class HaloComm:
    """Halo exchange per step (SURVEY §8(e) option 2): pack the own z entries each peer
    references (sc_gather_f64) and move them with one batch of point-to-point sends/receives
    straight into the peers' halo slots.  Pieces are not used (one exchange per step)."""

    def __init__(self, shard, plan: HaloPlan, rank: int, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.shard, self.plan, self.rank, self.group = shard, plan, rank, group
        self.nccl = dist.get_backend(group) == "nccl"
        dev = _group_device(group)
        self.peers = [q for q in range(plan.world) if q != rank and
                      (plan.send_idx[q].size or plan.halo_ids[q].size)]
        self.idx = {q: torch.from_numpy(plan.send_idx[q]).to(dev) for q in self.peers}
        self.sbuf = {q: torch.empty(plan.send_idx[q].size, dtype=torch.float64, device=dev)
                     for q in self.peers}

    def gather_piece(self, z_full, j):
        dist, plan = self.dist, self.plan
        ops = []
        for q in self.peers:
            if self.sbuf[q].numel():
                self.shard.pack(z_full, self.idx[q], self.sbuf[q])
                ops.append(dist.P2POp(dist.isend, self.sbuf[q], q, self.group))
            a, b = plan.halo_range(q)
            if b > a:
                ops.append(dist.P2POp(dist.irecv, z_full[a:b], q, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def finish(self):
        pass

    def recv_bytes(self) -> int:
        return 8 * self.plan.n_halo

    def close(self):
        pass


class ShardedPower:
    """T pipelined steps over a shard with buffers allocated once.  With NCCL the whole
    T-step sequence (per-piece SpMVs, side-stream all-gathers and their event fork/joins) can
    be captured into one CUDA graph and replayed, so the pipeline is not bound by the host
    issuing 2*P launches per step."""

    def __init__(self, shard, plan: ShardPlan, rank: int, *, sign: float = 1.0,
                 sym: bool = False, group=None, comm=None):
        self.shard, self.plan, self.rank = shard, plan, rank
        self.sign, self.sym = sign, sym
        n = int(plan.sizes[rank])
        zspace = getattr(shard, "zspace", shard.zeros)
        if comm is None:
            self.comm = PieceComm(plan, rank, group)
            self.z = [zspace(plan.ncols), zspace(plan.ncols)]
        elif hasattr(comm, "z0"):  # fused peer exchange: z lives in the mirrored allocation
            self.comm = comm
            self.z = [comm.z0, comm.z1]
        else:  # halo exchange
            self.comm = comm
            self.z = [zspace(plan.ncols), zspace(plan.ncols)]
        self.x = [shard.zeros(n), shard.zeros(n)]
        self.x0 = shard.zeros(n)
        self.graph = None
        self.graph_T = None

    def _enqueue(self, T: int):
        sh, plan, comm, z, x = self.shard, self.plan, self.comm, self.z, self.x
        for j in range(plan.pieces):
            sh.scale_piece(j, self.x0, z[0], self.sym)
            comm.gather_piece(z[0], j)
        comm.finish()
        for t in range(T):
            a, b = t & 1, (t & 1) ^ 1
            xin = self.x0 if t == 0 else x[a]
            for j in range(plan.pieces):
                sh.step_piece(j, z[a], xin, x[b], z[b], self.sign, self.sym)
                comm.gather_piece(z[b], j)
            comm.finish()

    def sample(self, seed: int):
        self.shard.irwin_hall(seed, self.x0)

    def capture(self, T: int):
        """Record T steps (from the current x0 buffer) into a CUDA graph; NCCL only."""
        import torch

        if not getattr(self.comm, "nccl", True):
            raise InputError("CUDA-graph capture needs the NCCL backend or the peer exchange")
        self._enqueue(T)  # warm: communicator and side-stream setup outside the capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._enqueue(T)
        torch.cuda.synchronize()
        self.graph, self.graph_T = g, T

    def run(self, T: int):
        """T steps from x0; returns (x_T local renumbered, z space of step T)."""
        if self.graph is not None and self.graph_T == T:
            self.graph.replay()
        else:
            self._enqueue(T)
        return (self.x0 if T == 0 else self.x[T & 1]), self.z[T & 1]


def power_iterate_sharded(shard, plan: ShardPlan, rank: int, T: int, *, seed: int | None = 0,
                          x0_local_renumbered=None, sign: float = 1.0, sym: bool = False,
                          group=None):
    """T steps over the shards; returns (x_T local renumbered, z space of step T)."""
    p = ShardedPower(shard, plan, rank, sign=sign, sym=sym, group=group)
    if x0_local_renumbered is not None:
        p.x0.copy_(x0_local_renumbered)
    else:
        p.sample(seed)
    return p.run(T)


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
        # NCCL writes its debug output (the version banner under NCCL_DEBUG=VERSION/INFO) to
        # stdout by default; the bench prints exactly one JSON line there
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def entry_balanced_starts(row_ptr: np.ndarray, world: int) -> np.ndarray:
    """Row-block starts balancing stored entries (the multi-GPU handle's rule): block w starts
    at the first row whose offset reaches w * nnz / world (each block keeps >= 1 row)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    n, nnz = rp.size - 1, int(rp[-1])
    st = np.zeros(world + 1, dtype=np.int64)
    st[world] = n
    for w in range(1, world):
        r = int(np.searchsorted(rp, nnz * w // world, side="left"))
        st[w] = min(max(r, st[w - 1] + 1), n - (world - w))
    return st


def bench_main(args, metric: str, unit: str):
    """Default (the driver's scaling run): WEAK scaling -- rank r owns one config-2 sized row
    block (1e6 rows, 10 SBM blocks) of an SBM with n = N * 1e6, k = 10 N, expected in-block
    degree 40 and out-of-block degree 4; T = 100 steps, each pipelined over P pieces with an
    NCCL all-gather per piece.  `--config 3|4|5`: STRONG scaling of that BASELINE config --
    every rank generates the whole graph on its own GPU with the device generator, keeps its
    entry-balanced row block (columns renamed on the device, sc_shard_create_from_csr) and
    frees the rest; the total work is fixed as N grows."""
    import torch
    import torch.distributed as dist

    from .generate import SbmParams, sbm_rows

    rank, world, local = _init_dist()
    strong = int(getattr(args, "config", 2)) in (3, 4, 5)
    n_loc = 10**6
    params = SbmParams(n=world * n_loc, k=10 * world, p=40 / (10**5 - 1),
                       q=4 / (world * n_loc - 10**5), seed=0)
    T = 100
    p2p = getattr(args, "comm", "nccl") == "p2p"
    halo = getattr(args, "comm", "nccl") == "halo"
    if strong and halo:
        raise InputError("the strong-scaling configs use the all-gather or the peer exchange")
    # Splitting a step into P pieces costs ~12 us per extra piece on one B200 (smaller grids,
    # one more collective) and hides up to (P-1)/P of the all-gather, which moves
    # (W-1) * 8 MB per GPU per step (~12 us at W = 2, ~80 us at W = 8 over NVLink): only
    # worth it for the widest runs.
    default_pieces = 2 if world >= 8 else 1
    pieces = 1 if (p2p or halo) else int(getattr(args, "pieces", 0) or default_pieces)
    if strong:
        from .generate import CONFIG_T, config_device_csr

        cfg = int(args.config)
        T = CONFIG_T[cfg]
        with config_device_csr(cfg, 0, local) as dcsr:
            rp_all = np.empty(dcsr.n + 1, dtype=np.int64)
            _lib.check(_lib.load().sc_csr_download(dcsr.handle, _lib.ptr(rp_all), None, None, None))
            starts = entry_balanced_starts(rp_all, world)
            rp = rp_all[starts[rank]:starts[rank + 1] + 1] - rp_all[starts[rank]]
            plan = exchange_plan(rp, starts, rank, world, pieces=pieces,
                                 align=8192 if pieces == 1 else 1)
            shard = CudaShard.from_device_csr(dcsr, plan, rank, local)
            n_total, weighted = int(dcsr.n), bool(dcsr.weighted)
        del rp_all
    else:
        starts = np.arange(world + 1, dtype=np.int64) * n_loc
        rp, col, deg, iso = sbm_rows(params, int(starts[rank]), int(starts[rank + 1]))
        iso_t = torch.tensor([iso], device="cuda")
        dist.all_reduce(iso_t)
        if int(iso_t.item()):
            raise InputError("isolated vertices in the scaling graph; choose another seed")
        if halo:
            plan = exchange_halo_plan(rp, col, starts, rank, world)
        else:
            plan = exchange_plan(rp, starts, rank, world, pieces=pieces,
                                 align=8192 if pieces == 1 else 1)
        shard = CudaShard(rp, plan.rename(col), None, deg, plan, rank, local)
        n_total, weighted = int(params.n), False
    # column panels for whole-shard steps (as the single-GPU pipeline at T >= 64); the peer
    # exchange and multi-piece steps stay on SELL
    panels = False
    if not p2p and pieces == 1 and not getattr(args, "sell", False):
        ok_t = torch.tensor([1 if shard.build_panels() else 0], device="cuda", dtype=torch.int32)
        dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
        panels = bool(ok_t.item())
    nnz_t = torch.tensor([int(rp[-1])], device="cuda", dtype=torch.int64)
    dist.all_reduce(nnz_t)
    nnz_total = int(nnz_t.item())
    stream = torch.cuda.current_stream()
    comm = None
    if p2p:
        comm = P2PComm(shard, plan, rank)
        comm.link()
    elif halo:
        comm = HaloComm(shard, plan, rank)
    runner = ShardedPower(shard, plan, rank, comm=comm)
    use_graph = not getattr(args, "no_graph", False)

    def one_step():
        runner.sample(0)
        return runner.run(T)

    runner.sample(0)
    if use_graph:
        # every rank must take the same path: capture, agree on success, else launch per step
        ok = torch.tensor([1], device="cuda", dtype=torch.int32)
        try:
            runner.capture(T)
        except Exception as exc:  # noqa: BLE001 -- e.g. a NCCL build that cannot be captured
            print(f"[rank {rank}] CUDA-graph capture failed ({exc}); launching per step",
                  file=sys.stderr, flush=True)
            ok.zero_()
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if not int(ok.item()):
            runner.graph = None
            use_graph = False
    for _ in range(max(args.warmup, 3)):
        one_step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    from .clocks import ClockSampler

    clk = ClockSampler(torch.cuda.current_device())
    with clk:
        e0.record(stream)
        for _ in range(args.steps):
            one_step()
        e1.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], device="cuda", dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    tot_ms = float(ms.item())
    # the exchange alone (NVLink): T steps x P pieces
    zbuf = shard.zeros(plan.ncols)
    agc = comm if halo else PieceComm(plan, rank)
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(stream)
    for _ in range(T):
        for j in range(plan.pieces):
            agc.gather_piece(zbuf, j)
        agc.finish()
    e1.record(stream)
    torch.cuda.synchronize()
    ag = torch.tensor([e0.elapsed_time(e1) / T], device="cuda", dtype=torch.float64)
    dist.all_reduce(ag, op=dist.ReduceOp.MAX)
    ag_ms = float(ag.item())
    recv_bytes = comm.recv_bytes() if halo else (world - 1) * plan.pieces * plan.pmax * 8
    # end-to-end leg through the drop-in's multi-GPU call (weak-scaling workload only), in a
    # subprocess of rank 0 while the other ranks wait
    e2e = None
    if not strong and not getattr(args, "no_e2e", False):
        from datetime import timedelta

        dist.barrier()
        torch.cuda.synchronize()
        # the other ranks wait on the HOST (store key), not in a collective: a spinning NCCL
        # kernel on their GPUs would be time-sliced against the subprocess's kernels
        store = dist.distributed_c10d._get_default_store()
        if rank == 0:
            e2e = _inprocess_e2e(world, T)
            store.set("sc_e2e_done", "1")
        else:
            try:
                store.wait(["sc_e2e_done"], timedelta(seconds=420))
            except Exception:  # noqa: BLE001 -- rank 0 prints the line either way
                pass
    if rank == 0:
        value = nnz_total * T * args.steps / (tot_ms / 1e3) / 1e9
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": (f"config{args.config} (whole graph, row blocks balanced by "
                                    "entries)" if strong else
                                    f"config2 block per GPU (SBM n={params.n}, k={params.k})"),
                       "n_per_gpu": int(plan.n_max) if strong else n_loc,
                       "nnz_total": nnz_total, "T": T, "pieces": plan.pieces,
                       "spmv_layout": "panels" if panels else "sell",
                       "cuda_graph": use_graph,
                       "comm": "p2p" if p2p else "halo" if halo else "nccl",
                       "parallelism": (f"row-block shards x{world}, z stored into the peers' "
                                       "buffers by the SpMV epilogue + flag barrier"
                                       if p2p else
                                       f"row-block shards x{world}, halo exchange (packed "
                                       "referenced entries, NCCL send/recv)"
                                       if halo else
                                       f"row-block shards x{world}, pipelined NCCL all-gather "
                                       f"of z ({plan.pieces} pieces per step)")},
            "exchange": {"kind": "halo send/recv" if halo else "all-gather",
                         "ms_per_step": ag_ms, "recv_bytes_per_gpu": recv_bytes,
                         "gbs_per_gpu": recv_bytes / (ag_ms / 1e3) / 1e9 if world > 1 else 0.0},
            "roofline": _shard_roofline(nnz_total, n_total, weighted, tot_ms / (args.steps * T), world),
            "clocks": clk.summary(),
            "gpu_launches": args.steps * (1 + (T + 1) * plan.pieces
                                          + ((T + 1) if p2p and world > 1 else 0)
                                          + ((T + 1) * sum(1 for q in comm.peers
                                                           if comm.sbuf[q].numel())
                                             if halo else 0)),
        }
        if e2e is not None:
            line["e2e"] = e2e
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    shard.close()
    dist.destroy_process_group()


_E2E_CODE = r"""
import json, sys, time
sys.path.insert(0, %r)
import numpy as np
from paper_2310_10939_b200 import SpectralParams, fast_spectral_cluster
from paper_2310_10939_b200.generate import DeviceCSR, SbmParams
world, T = int(sys.argv[1]), int(sys.argv[2])
n_loc = 10**6
p = SbmParams(n=world * n_loc, k=10 * world, p=40 / (10**5 - 1), q=4 / (world * n_loc - 10**5), seed=0)
with DeviceCSR(p, 0) as d:
    g = d.download(pinned=True).graph
ms = []
for rep in range(3):
    t0 = time.perf_counter()
    res = fast_spectral_cluster(g, SpectralParams(k=p.k, t=T, mode="one_vector", seed=0, gpus=world))
    ms.append(1e3 * (time.perf_counter() - t0))
print(json.dumps({"cluster_ms": min(ms[1:]), "n": g.n, "nnz": g.nnz,
                  "h2d": int(g.row_offsets.nbytes + 4 * g.nnz + g.degrees.nbytes),
                  "d2h": int(16 * g.n), "sizes": int(np.bincount(res.partition.labels).size)}))
"""


def _inprocess_e2e(world: int, T: int, timeout_s: int = 240):
    """End to end at `world` GPUs through the drop-in call (fast_spectral_cluster with
    SpectralParams(gpus=world): ONE process over all GPUs) on a graph of the weak-scaling law,
    run in a fresh subprocess of rank 0 so that nothing it does (an unsupported peer mapping, a
    timeout) can take the torchrun bench line down.  Returns the e2e object or None."""
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT",
                        "TORCHELASTIC_RUN_ID", "GROUP_RANK", "ROLE_RANK", "LOCAL_WORLD_SIZE")}
    try:
        r = subprocess.run([sys.executable, "-c", _E2E_CODE % root, str(world), str(T)],
                           capture_output=True, text=True, timeout=timeout_s, env=env, cwd=root)
        if r.returncode:
            return {"unavailable": (r.stderr.strip().splitlines() or ["failed"])[-1][:200]}
        d = json.loads(r.stdout.strip().splitlines()[-1])
        return {"value": d["nnz"] * T / (d["cluster_ms"] / 1e3) / 1e9, "unit": "GNNZ/s",
                "h2d_bytes_per_step": d["h2d"], "d2h_bytes_per_step": d["d2h"],
                "cluster_ms": d["cluster_ms"],
                "path": f"fast_spectral_cluster(SpectralParams(gpus={world})) in one process over "
                        f"{world} GPU(s), graph of the weak-scaling law (n={d['n']}, device "
                        "generator) in pinned host memory -> labels + f on host"}
    except Exception as e:  # noqa: BLE001 -- the extra leg never fails the bench line
        return {"unavailable": f"{type(e).__name__}: {e}"[:200]}


def _shard_roofline(nnz_total: int, n_total: int, weighted: bool, step_ms: float, world: int) -> dict:
    """Whole-job HBM roofline of one sharded step (SURVEY.md §8(d) byte formula over all ranks
    against world x the measured per-GPU peak; the all-gather's bytes are reported separately
    under "exchange")."""
    peak, kind = 6650.0, "fallback"
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            peak, kind = float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        pass
    idx_val = 12 if weighted else 4
    alg = nnz_total * idx_val + 16 * n_total
    achieved = alg / (step_ms / 1e3) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peak * world, "unit": "GB/s",
            "frac": achieved / (peak * world), "traffic": None, "peak_kind": kind,
            "alg_bytes_per_launch": alg,
            "alg_bytes_formula": f"nnz*{idx_val} + 16n over all {world} ranks"
                                 + (" (idx+val)" if weighted else " (unit weights: val elided)"),
            "kernel_ms": step_ms}


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
