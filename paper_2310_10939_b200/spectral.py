"""Device-resident operators, the Irwin-Hall start vector and the power method.

Mirrors the operator half of specluster/spectral.py:
  * ``rng_for``            spectral.py:32-36 (SeedSequence([seed, *tags]) -> PCG64)
  * ``SignlessLaplacianOp`` spectral.py:39-64 -- same ``.n`` / ``.matvec`` protocol,
    executed by the sm_100a kernel with the symmetric variant flag
  * ``RandomWalkOp``        the one-vector operator M x = 0.5 x +/- 0.5 A D^-1 x
    (PAPER.md:19 with the '+' sign of PAPER.md:109,134,162)
  * ``power_method``       spectral.py:87-102 -- T fused steps on the GPU
  * ``EmbeddingMatrix``    spectral.py:109-135
  * ``sample_irwin_hall``  x0(u) ~ IW(deg u); counter-based Philox4x64-10,
    stream tag 6 (tags 1-5 are taken: spectral.py:28-29, pipeline.py:47-48, generate.py:22)

Everything numeric runs in libsc_b200.so; this module only moves arrays and keys.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InputError
from .graph import Graph, as_graph

TAG_IRWIN_HALL = 6
GENERATOR_NAME = "philox4x64-10-irwin-hall"


def rng_for(seed: int, *tags: int) -> np.random.Generator:
    if seed < 0:
        raise InputError(f"seed must be a nonnegative integer, got {seed}")
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, *tags])))


def irwin_hall_key(seed: int) -> tuple[int, int]:
    """Philox key of the Irwin-Hall stream: SeedSequence([seed, 6]) -> two u64 words."""
    if seed < 0:
        raise InputError(f"seed must be a nonnegative integer, got {seed}")
    k = np.random.SeedSequence([seed, TAG_IRWIN_HALL]).generate_state(2, np.uint64)
    return int(k[0]), int(k[1])


@dataclass
class EmbeddingMatrix:
    """n x l block, one vertex per row (spectral.py:109-135)."""

    data: np.ndarray
    scaled: bool
    seed: int = 0

    def __post_init__(self):
        self.data = np.ascontiguousarray(self.data, dtype=np.float64)
        if self.data.ndim != 2 or self.data.shape[1] < 1:
            raise InputError("embedding must be a 2-D array with at least one column")
        if not np.all(np.isfinite(self.data)):
            raise InputError("embedding contains NaN or Inf")

    @property
    def n(self) -> int:
        return self.data.shape[0]

    @property
    def l(self) -> int:
        return self.data.shape[1]


def _check_shapes(g: Graph) -> None:
    n = int(g.n)
    if n < 1:
        raise InputError(f"graph must have n >= 1 vertices, got {n}")
    if np.shape(g.row_offsets) != (n + 1,) or np.shape(g.degrees) != (n,):
        raise InputError("row_offsets must have length n+1 and degrees length n")
    nnz = int(g.row_offsets[-1])
    if np.shape(g.col_indices) != (nnz,):
        raise InputError("col_indices length must equal row_offsets[-1]")
    if g.weights is not None and np.shape(g.weights) != (nnz,):
        raise InputError("weights length must equal row_offsets[-1]")


LOCALITY_THRESHOLD = 0.15


def id_locality(g, samples: int = 256) -> float:
    """Mean |col - row| / n over the entries of a fixed sample of rows: ~0.33 for ids that
    carry no locality (uniformly scattered neighbours), a few percent for block- or
    space-ordered ids (the reference SBM numbering: 0.06 at config 2)."""
    n = int(g.n)
    rp = np.asarray(g.row_offsets)
    if n < 2 or rp[-1] == 0:
        return 0.0
    rows = np.random.default_rng(12345).integers(0, n, min(samples, n))
    starts = rp[rows]
    lens = rp[rows + 1] - starts
    total = int(lens.sum())
    if total == 0:
        return 0.0
    first = np.repeat(np.cumsum(lens) - lens, lens)
    idx = np.repeat(starts, lens) + (np.arange(total) - first)
    c = np.asarray(g.col_indices)[idx].astype(np.int64)
    return float(np.abs(c - np.repeat(rows, lens)).sum()) / (total * n)


class DeviceGraph:
    """Owns an ``sc_graph`` handle: the CSR uploaded once to one GPU (graph.py:28-45
    layout; degrees copied verbatim, never recomputed)."""

    def __init__(self, graph, device: int = 0, keep_weights: bool = False,
                 fp32_values: bool = False, reorder: str | None = None, panels: bool = False,
                 gpus: int = 1, devices=None, windows: bool = False):
        """``panels``: also build the column-panel layout (sc_panel.cuh; unit weights and rows
        of <= 256 entries only, declined silently otherwise -- see ``info()['panel_groups']``);
        whole-graph steps then stage heavily referenced column ranges in shared memory.
        ``windows``: also try the row-window layout (sc_window.cuh; any weights): for graphs
        whose renumbered rows reference mostly their own 4096-row neighbourhood (k-NN /
        geometric graphs after the BFS pre-order) each CTA stages its z panel and its
        out-of-panel z values in shared memory and streams 16-bit indices; declined silently
        otherwise (``info()['window_items']``).
        ``fp32_values``: store the weights as fp32 (the optional fp32-value variant:
        half the weight bytes, results within 1e-5 relative of fp64; unit-weight graphs are
        unaffected).  ``reorder="bfs"``: renumber the vertices by a multi-source BFS before the
        SELL layout (locality for graphs whose ids carry none; results unchanged).
        ``gpus`` / ``devices``: one handle over several GPUs in this process
        (sc_graph_create_multi): row blocks balanced by entries, one shard per GPU (``devices``
        lists them, default ``device .. device + gpus - 1``; a device may repeat), z exchanged
        by peer stores from the SpMV epilogue; results bit-identical to one GPU.  Multi-GPU
        handles keep the shards' own order (no BFS pre-order)."""
        if reorder not in (None, "bfs", "auto"):
            raise InputError(f"reorder must be None, 'bfs' or 'auto', got {reorder!r}")
        g = as_graph(graph)
        _check_shapes(g)  # content (ranges, monotonicity, degrees) is validated by the C-ABI
        if devices is not None:
            devices = [int(d) for d in devices]
            gpus = len(devices)
        elif gpus > 1:
            devices = list(range(device, device + gpus))
        if gpus < 1:
            raise InputError(f"gpus must be >= 1, got {gpus}")
        multi = gpus > 1
        if multi:
            if reorder == "bfs":
                raise InputError("the BFS pre-order applies to single-GPU handles")
            reorder = None
        if reorder == "auto":
            reorder = "bfs" if id_locality(g) > LOCALITY_THRESHOLD else None
        self.reorder = reorder
        self.gpus = gpus
        self.devices = devices if multi else [device]
        L = _lib.require_device()
        self.graph = g
        self.n = g.n
        self.nnz = g.nnz
        self._rp = np.ascontiguousarray(g.row_offsets, dtype=np.int64)
        self._col = np.ascontiguousarray(g.col_indices, dtype=np.int32)
        self._deg = np.ascontiguousarray(g.degrees, dtype=np.float64)
        if keep_weights:
            # benchmark/diagnostic mode: stream the weight array even if it is all ones
            w = (np.ones(g.nnz) if g.weights is None
                 else np.ascontiguousarray(g.weights, dtype=np.float64))
        else:
            w = None if (g.weights is None or g.unit_weights()) else np.ascontiguousarray(
                g.weights, dtype=np.float64)
        h = ctypes.c_void_p()
        cflags = ((_lib.SC_CREATE_KEEP_WEIGHTS if keep_weights else 0)
                  | (_lib.SC_CREATE_FP32_VALUES if fp32_values else 0)
                  | (_lib.SC_CREATE_REORDER_BFS if reorder == "bfs" else 0)
                  | (_lib.SC_CREATE_PANELS if panels else 0)
                  | (_lib.SC_CREATE_WINDOWS if windows else 0))
        if multi:
            dv = np.ascontiguousarray(devices, dtype=np.int32)
            _lib.check(L.sc_graph_create_multi(_lib.ptr(self._rp), _lib.ptr(self._col),
                                               _lib.ptr(w), _lib.ptr(self._deg), g.n, g.nnz,
                                               gpus, _lib.ptr(dv), cflags, ctypes.byref(h)))
        else:
            _lib.check(L.sc_graph_create_ex(_lib.ptr(self._rp), _lib.ptr(self._col), _lib.ptr(w),
                                            _lib.ptr(self._deg), g.n, g.nnz, device, cflags,
                                            ctypes.byref(h)))
        self._h = h
        self.device = self.devices[0]
        self.last_timing = None

    @classmethod
    def from_device_csr(cls, csr, keep_weights: bool = False, panels: bool = False,
                        reorder: str | None = None, windows: bool = False,
                        fp32_values: bool = False) -> "DeviceGraph":
        """Graph handle straight from a device-resident CSR (``generate.DeviceCSR``): the
        column array never visits the host (sc_graph_create_from_csr)."""
        L = _lib.require_device()
        self = cls.__new__(cls)
        h = ctypes.c_void_p()
        _lib.check(L.sc_graph_create_from_csr(csr.handle,
                                              (_lib.SC_CREATE_KEEP_WEIGHTS if keep_weights else 0)
                                              | (_lib.SC_CREATE_PANELS if panels else 0)
                                              | (_lib.SC_CREATE_REORDER_BFS if reorder == "bfs" else 0)
                                              | (_lib.SC_CREATE_WINDOWS if windows else 0)
                                              | (_lib.SC_CREATE_FP32_VALUES if fp32_values else 0),
                                              ctypes.byref(h)))
        self._h = h
        self.graph = None
        self.reorder = reorder
        self.gpus, self.devices = 1, [csr.device]
        self.n, self.nnz = csr.n, csr.nnz
        self.device = csr.device
        self.last_timing = None
        return self

    # -- lifecycle
    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.load().sc_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        if not self._h:
            raise InputError("device graph is closed")
        return self._h

    def info(self) -> dict:
        gi = _lib.GraphInfo()
        _lib.check(_lib.load().sc_graph_info_get(self.handle, ctypes.byref(gi)))
        return {f: getattr(gi, f) for f, _ in gi._fields_ }

    def shard_layout(self) -> list:
        """multi-GPU handles: per shard (row0, rows, z offset, device)"""
        out = []
        for w in range(self.gpus if self.gpus > 1 else 0):
            r0, nr, zo, dv = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
            _lib.check(_lib.load().sc_graph_shard_layout(self.handle, w, ctypes.byref(r0),
                                                         ctypes.byref(nr), ctypes.byref(zo),
                                                         ctypes.byref(dv)))
            out.append((r0.value, nr.value, zo.value, dv.value))
        return out

    # -- start vector
    def sample_irwin_hall(self, seed: int, return_host: bool = False):
        k0, k1 = irwin_hall_key(seed)
        out = np.empty(self.n) if return_host else None
        _lib.check(_lib.load().sc_sample_irwin_hall(self.handle, k0, k1, _lib.ptr(out)))
        return out

    def set_x0(self, x0) -> None:
        x = np.ascontiguousarray(x0, dtype=np.float64)
        if x.shape != (self.n,):
            raise InputError(f"x0 has shape {x.shape}, expected ({self.n},)")
        if not np.all(np.isfinite(x)):
            raise InputError("x0 contains NaN or Inf")
        _lib.check(_lib.load().sc_set_x0(self.handle, _lib.ptr(x)))

    # -- power iteration
    def power_iterate(self, t: int, *, sign: float = 1.0, sym: bool = False,
                      want_x: bool = True, want_f: bool = True, cuda_graph: bool = True,
                      l2_persist: bool = False, force_weighted: bool = False,
                      force_sell: bool = False):
        if t < 0:
            raise InputError(f"power method step count must be >= 0, got {t}")
        flags = ((_lib.SC_SYM_VARIANT if sym else 0) | (0 if cuda_graph else _lib.SC_NO_CUDA_GRAPH)
                 | (_lib.SC_L2_PERSIST if l2_persist else 0)
                 | (_lib.SC_FORCE_WEIGHTED if force_weighted else 0)
                 | (_lib.SC_FORCE_SELL if force_sell else 0))
        xT = np.empty(self.n) if want_x else None
        f = np.empty(self.n) if want_f else None
        tm = _lib.Timing()
        _lib.check(_lib.load().sc_power_iterate(self.handle, int(t), float(sign), flags,
                                                 _lib.ptr(xT), _lib.ptr(f), ctypes.byref(tm)))
        self.last_timing = {"power_ms": tm.power_ms, "kernel_ms": tm.kernel_ms,
                            "d2h_ms": tm.d2h_ms}
        return xT, f

    def download_f(self) -> np.ndarray:
        """f = D^-1 x_T of the last power_iterate, original vertex order (host copy)"""
        f = np.empty(self.n)
        _lib.check(_lib.load().sc_graph_download_f(self.handle, _lib.ptr(f)))
        return f

    def power_iterate_block(self, x0: np.ndarray, t: int, *, want_raw: bool = True):
        """t steps of the signless operator on an (n, L) block (pm_log_k's embedding,
        pipeline.py:144-147); returns (raw = M^t x0, scaled = raw * d^-1/2)."""
        x = np.ascontiguousarray(x0, dtype=np.float64)
        if x.ndim != 2 or x.shape[0] != self.n:
            raise InputError(f"block must be ({self.n}, L), got {x.shape}")
        if t < 0:
            raise InputError(f"power method step count must be >= 0, got {t}")
        raw = np.empty_like(x) if want_raw else None
        scaled = np.empty_like(x)
        tm = _lib.Timing()
        _lib.check(_lib.load().sc_power_iterate_block(self.handle, int(t), x.shape[1], _lib.ptr(x),
                                                       _lib.ptr(raw), _lib.ptr(scaled),
                                                       ctypes.byref(tm)))
        self.last_timing = {"power_ms": tm.power_ms, "kernel_ms": tm.kernel_ms}
        return raw, scaled


class _DeviceOp:
    """Operator protocol of spectral.py:52-59/71-79 (``.n``, ``.matvec``) backed by a
    DeviceGraph; ``power(x0, t)`` runs t fused steps without host round trips."""

    _sym = False

    def __init__(self, graph, device: int = 0, sign: float = 1.0):
        self.dev = graph if isinstance(graph, DeviceGraph) else DeviceGraph(graph, device)
        self.graph = self.dev.graph
        self.n = self.dev.n
        self.sign = sign

    def power(self, x0: np.ndarray, t: int) -> np.ndarray:
        x0 = np.asarray(x0, dtype=np.float64)
        if x0.shape[0] != self.n:
            raise InputError(f"operand has {x0.shape[0]} rows, operator expects {self.n}")
        if x0.ndim == 1:
            self.dev.set_x0(x0)
            xT, _ = self.dev.power_iterate(t, sign=self.sign, sym=self._sym, want_f=False)
            return xT
        if self._sym and self.sign == 1.0 and 1 <= x0.shape[1] <= 16:
            return self.dev.power_iterate_block(x0, t)[0]  # all columns in one pass
        cols = [self.power(x0[:, i], t) for i in range(x0.shape[1])]
        return np.stack(cols, axis=1)

    def matvec(self, x: np.ndarray) -> np.ndarray:
        return self.power(x, 1)

    __call__ = matvec


class RandomWalkOp(_DeviceOp):
    """M x = 0.5 x + sign * 0.5 * A (x / d): the one-vector lazy random walk."""


class SignlessLaplacianOp(_DeviceOp):
    """M x = 0.5 x + 0.5 s (A (s x)), s = deg^-1/2 (spectral.py:39-57), on the GPU."""

    _sym = True

    @property
    def inv_sqrt_degrees(self) -> np.ndarray:
        return 1.0 / np.sqrt(self.graph.degrees)


def power_method(op, x0: np.ndarray, t: int) -> np.ndarray:
    """M^t x0, no normalisation (spectral.py:87-102).  Device operators run t fused
    steps on the GPU; a plain callable is the caller's own operator and is applied t
    times as given (nothing here computes on the CPU on its behalf)."""
    if t < 0:
        raise InputError(f"power method step count must be >= 0, got {t}")
    if isinstance(op, _DeviceOp):
        return op.power(x0, int(t))
    if isinstance(op, (Graph,)):
        return RandomWalkOp(op).power(x0, int(t))
    if callable(op) and not isinstance(op, np.ndarray):
        x = np.array(x0, dtype=np.float64, copy=True)
        for _ in range(int(t)):
            x = op(x)
        return x
    raise InputError(f"cannot interpret {type(op).__name__} as a device operator; wrap the "
                     "graph in RandomWalkOp or SignlessLaplacianOp")


TAG_GAUSSIAN_COLUMN = 1  # spectral.py:28


def sample_gaussian_vectors(n: int, l: int, seed: int) -> EmbeddingMatrix:
    """Algorithm 2's start block (spectral.py:183-195): column i is
    rng_for(seed, 1, i).standard_normal(n) -- the same numpy calls, so the same bits."""
    if n < 1 or l < 1:
        raise InputError(f"need n >= 1 and l >= 1, got n={n}, l={l}")
    data = np.empty((n, l), dtype=np.float64)

    def column(i):
        data[:, i] = rng_for(seed, TAG_GAUSSIAN_COLUMN, i).standard_normal(n)

    if l > 1 and n >= 100_000:  # independent streams: fill the columns concurrently
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(min(l, 8)) as ex:
            list(ex.map(column, range(l)))
    else:
        for i in range(l):
            column(i)
    return EmbeddingMatrix(data=data, scaled=False, seed=seed)


def sample_irwin_hall(graph, seed: int, device: int = 0) -> EmbeddingMatrix:
    """x0(u) ~ IW(deg u) drawn on the GPU, returned as an n x 1 EmbeddingMatrix."""
    dev = graph if isinstance(graph, DeviceGraph) else DeviceGraph(graph, device)
    x0 = dev.sample_irwin_hall(seed, return_host=True)
    return EmbeddingMatrix(data=x0[:, None], scaled=False, seed=seed)


def release_device_memory(device: int = -1) -> int:
    """Free the device buffers that destroyed graphs left in the library's reuse cache
    (all devices by default); returns the bytes released."""
    return int(_lib.load().sc_release_cached_memory(int(device)))
