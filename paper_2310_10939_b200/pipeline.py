"""``fast_spectral_cluster`` -- the drop-in entry point (specluster/pipeline.py:127-178).

Same signature ``fast_spectral_cluster(g, params) -> PipelineResult`` and the same
``SpectralParams`` / ``PipelineResult`` fields (pipeline.py:55-120), with one more mode
in ``MODES``: ``"one_vector"`` -- the method of PAPER.md:12-253:

    x0(u) ~ IW(deg u)                      (GPU Philox sampler, or params.x0)
    x_T  = M^T x0,  M = 0.5 (I + s A D^-1)  (fused sm_100a SpMV, T steps, s = +1 / -1)
    f    = D^-1 x_T                         (fused into the last step's epilogue)
    labels = lloyd(f, k, seed=_kmeans_seed(seed))   (bit-exact GPU replica)

Timings keep the reference keys {embed, scale, kmeans, total} in milliseconds
(pipeline.py:163-168).  ``"pm_log_k"`` (the reference's default Algorithm-2 embedding,
pipeline.py:144-147) also runs on the device: the reference's own Gaussian start block
(host numpy, same calls), the block power method of the signless operator (bit-exact,
csrc sc_power_iterate_block), the d^-1/2 row scaling fused into the last step, and the
d-dimensional k-means.  pm_k and the eigs_* modes raise InputError.
"""

from __future__ import annotations

import concurrent.futures
import math
import time
from dataclasses import dataclass

import numpy as np

from .errors import InputError
from .graph import as_graph
from .kmeans import KMeans1D, Partition
from .spectral import DeviceGraph, EmbeddingMatrix, sample_gaussian_vectors

MODES = ("pm_log_k", "pm_k", "eigs_k", "eigs_log_k", "one_vector")
DEVICE_MODES = ("one_vector", "pm_log_k")

_TAG_KMEANS = 2  # pipeline.py:47


@dataclass
class SpectralParams:
    """pipeline.py:55-105, plus optional one-vector knobs (defaults keep old call sites)."""

    k: int
    epsilon: float | None = None
    l: int | None = None
    t: int | None = None
    mode: str = "pm_log_k"
    seed: int = 0
    # one_vector extensions
    walk_sign: int = 1           # M = 0.5 (I + walk_sign * A D^-1)
    x0: np.ndarray | None = None  # caller-supplied start vector (else Irwin-Hall)
    device: int = 0
    restarts: int = 10
    max_iters: int = 100
    tol: float = 1e-6
    kmeans: str = "exact"        # "exact" (bit-exact replica) or "sorted" (approximate:
                                 # labels may differ from the reference's)
    cost_assert: bool | None = None  # kmeans.py:206's assert; None: on unless python -O
    reorder: str | None = "auto"  # device-layout pre-order: "auto", "bfs" or None (exact)
    layout: str = "auto"         # SpMV layout: "auto" (column panels, else row windows, for
                                 # T >= 64 when the graph qualifies), "panels", "windows"
                                 # or "sell"; results identical
    gpus: int = 1                # row-block shards over this many GPUs of this process
    devices: tuple | None = None  # explicit shard devices (overrides gpus; may repeat)

    def __post_init__(self):
        if self.mode not in MODES:
            raise InputError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.k < 2:
            raise InputError(f"need k >= 2, got k={self.k}")
        if self.epsilon is not None and not 0.0 < self.epsilon <= 1.0:
            raise InputError(f"epsilon must lie in (0, 1], got {self.epsilon}")
        if self.l is not None and self.l < 1:
            raise InputError(f"l must be >= 1, got {self.l}")
        if self.t is not None and self.t < 0:
            raise InputError(f"t must be >= 0, got {self.t}")
        if self.seed < 0:
            raise InputError(f"seed must be nonnegative, got {self.seed}")
        if self.walk_sign not in (1, -1):
            raise InputError(f"walk_sign must be +1 or -1, got {self.walk_sign}")
        if self.kmeans not in ("exact", "sorted"):
            raise InputError(f"kmeans must be 'exact' or 'sorted', got {self.kmeans!r}")
        if self.gpus < 1 or (self.devices is not None and len(self.devices) < 1):
            raise InputError(f"gpus must be >= 1, got {self.gpus}")
        if self.layout not in ("auto", "panels", "windows", "sell"):
            raise InputError(f"layout must be 'auto', 'panels', 'windows' or 'sell', "
                             f"got {self.layout!r}")

    def num_columns(self, n: int) -> int:
        if self.mode == "one_vector":
            return 1
        if self.l is not None:
            return self.l
        log_k = max(1, math.ceil(math.log2(self.k)))
        if self.mode in ("pm_k", "eigs_k"):
            return self.k
        if self.mode == "pm_log_k" and self.epsilon is not None:
            return min(self.k, math.ceil((math.log2(self.k) + math.log2(1.0 / self.epsilon))
                                         / self.epsilon**2))
        return log_k

    def num_steps(self, n: int) -> int:
        if self.t is not None:
            return self.t
        if self.epsilon is not None:
            c3 = 1.0 / (2.0 * math.log(2.0))
            return int(math.ceil(c3 * math.log(24.0 * n / (self.epsilon**2 * self.k))))
        return int(math.ceil(10.0 * math.log(max(2.0, n / self.k))))


@dataclass
class PipelineResult:
    partition: Partition
    embedding: EmbeddingMatrix
    timings: dict
    mode: str
    l: int
    t: int | None
    eigs_converged: bool | None = None
    eigs_iterations: int | None = None
    x_T: np.ndarray | None = None
    device_timings: dict | None = None

    def __iter__(self):
        return iter((self.partition, self.embedding, self.timings))


def _kmeans_seed(seed: int) -> int:
    """pipeline.py:123-124."""
    return int(np.random.SeedSequence([seed, _TAG_KMEANS]).generate_state(1)[0])


PANEL_MIN_STEPS = 64
_POOL = concurrent.futures.ThreadPoolExecutor(max_workers=1, thread_name_prefix="sc-download")


def fast_spectral_cluster(g, params: SpectralParams, *, device_graph: DeviceGraph | None = None,
                          keep_x: bool = False) -> PipelineResult:
    """Cluster the graph's vertices into k parts (pipeline.py:127-178 contract).

    ``device_graph`` lets a caller reuse an uploaded graph across calls; by default the
    CSR is uploaded here (that upload is inside ``total``)."""
    if params.mode not in DEVICE_MODES:
        raise InputError(f"mode {params.mode!r} is the reference's Algorithm-2 embedding; the "
                         f"B200 path implements {DEVICE_MODES}")
    graph = as_graph(g) if device_graph is None else device_graph.graph
    n = graph.n
    if params.k > n:
        raise InputError(f"k={params.k} exceeds the vertex count n={n}")
    steps = params.num_steps(n)
    if params.mode == "pm_log_k":
        return _pm_log_k(graph, params, steps, device_graph)
    t_start = time.perf_counter()
    # the panel layout costs about a dozen SELL steps to build (device, ~1.7 ms at config 2)
    # and saves ~13 % per step where it applies
    panels = params.layout == "panels" or (params.layout == "auto" and steps >= PANEL_MIN_STEPS)
    # the row-window layout (one pass over the columns to decide, ~2 SELL steps to build) is
    # tried when the handle has no panel layout
    windows = params.layout == "windows" or (params.layout == "auto" and steps >= PANEL_MIN_STEPS)
    dev = device_graph if device_graph is not None else DeviceGraph(
        graph, params.device, reorder=params.reorder, panels=panels, gpus=params.gpus,
        devices=params.devices, windows=windows)
    try:
        t0 = time.perf_counter()
        if params.x0 is not None:
            dev.set_x0(params.x0)
        else:
            dev.sample_irwin_hall(params.seed)
        x_t, _ = dev.power_iterate(steps, sign=float(params.walk_sign), want_x=keep_x,
                                   want_f=False)
        t1 = time.perf_counter()
        # the k-means context copies f on the device; the host copy of f (and its validation,
        # spectral.py:123) overlaps the Lloyd iterations on a helper thread (both C calls
        # release the GIL; they use different handles and streams)
        with KMeans1D(graph=dev) as km:
            emb = _POOL.submit(lambda: EmbeddingMatrix(data=dev.download_f()[:, None], scaled=True,
                                                       seed=params.seed))
            t2 = time.perf_counter()
            try:
                part = km.lloyd(params.k, _kmeans_seed(params.seed), max_iters=params.max_iters,
                                tol=params.tol, restarts=params.restarts, method=params.kmeans,
                                assert_cost=params.cost_assert)
            finally:
                embedding = emb.result()
            km_info = dict(km.last)
        t3 = time.perf_counter()
    finally:
        if device_graph is None:
            dev.close()
    timings = {
        "embed": (t1 - t0) * 1e3,
        "scale": (t2 - t1) * 1e3,
        "kmeans": (t3 - t2) * 1e3,
        "total": (t3 - t0) * 1e3,
    }
    dt = dict(dev.last_timing or {})
    dt["upload_ms"] = (t0 - t_start) * 1e3
    dt["kmeans_costs"] = km_info.get("costs")
    dt["kmeans_iters"] = km_info.get("iters")
    dt["kmeans_best_restart"] = km_info.get("best_restart")
    return PipelineResult(partition=part, embedding=embedding, timings=timings,
                          mode=params.mode, l=1, t=steps, x_T=x_t, device_timings=dt)


def _pm_log_k(graph, params: SpectralParams, steps: int, device_graph) -> PipelineResult:
    """pipeline.py:140-178 for mode pm_log_k, on the device."""
    n = graph.n
    cols = params.num_columns(n)
    if cols > n:
        raise InputError(f"embedding width l={cols} exceeds n={n}")
    if cols > 16:
        raise InputError(f"the device block power method handles l <= 16 columns, got {cols}")
    t_start = time.perf_counter()
    dev = device_graph if device_graph is not None else DeviceGraph(graph, params.device)
    try:
        t0 = time.perf_counter()
        x0 = sample_gaussian_vectors(n, cols, params.seed).data
        _, scaled = dev.power_iterate_block(x0, steps, want_raw=False)
        t1 = time.perf_counter()
        embedding = EmbeddingMatrix(data=scaled, scaled=True, seed=params.seed)
        t2 = time.perf_counter()
        with KMeans1D(scaled, device=params.device) as km:
            part = km.lloyd(params.k, _kmeans_seed(params.seed), max_iters=params.max_iters,
                            tol=params.tol, restarts=params.restarts)
            km_info = dict(km.last)
        t3 = time.perf_counter()
    finally:
        if device_graph is None:
            dev.close()
    timings = {"embed": (t1 - t0) * 1e3, "scale": (t2 - t1) * 1e3, "kmeans": (t3 - t2) * 1e3,
               "total": (t3 - t0) * 1e3}
    dt = dict(dev.last_timing or {})
    dt["upload_ms"] = (t0 - t_start) * 1e3
    dt["kmeans_costs"] = km_info.get("costs")
    dt["kmeans_iters"] = km_info.get("iters")
    return PipelineResult(partition=part, embedding=embedding, timings=timings,
                          mode=params.mode, l=cols, t=steps, device_timings=dt)
