"""1-D k-means on the GPU: a bit-exact replica of the reference's restarted Lloyd.

Mirrors specluster/kmeans.py:
  * ``PointSet`` / ``Partition``  kmeans.py:24-83
  * ``lloyd``                     kmeans.py:167-215 (restarts, max_iters, tol, best-cost
                                  restart = first with strictly smallest cost)
  * k-means++ seeding            kmeans.py:116-137; every random draw is replayed on the
                                  host with the very numpy calls the reference makes, in
                                  the same order, from rng_for(seed, r) (kmeans.py:193):
                                  ``integers(n)`` then one ``random()`` per round, or
                                  ``integers(#unchosen)`` in the all-weights-zero round.
The data work (distances, cumulative sums, assignment, repair, ordered means, einsum-
order cost) runs in libsc_b200.so (csrc/sc_kmeans.cu).  1-D point sets (the one-vector
embedding) are replicated bit for bit; d-dimensional ones (pm_log_k embeddings) use the same
kernels with d-dimensional distances, whose middle term the reference evaluates with BLAS
(CPU-specific order), so there labels agree with the reference up to exact distance ties.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InputError
from .spectral import DeviceGraph, rng_for


@dataclass
class PointSet:
    coords: np.ndarray

    def __post_init__(self):
        self.coords = np.ascontiguousarray(self.coords, dtype=np.float64)
        if self.coords.ndim != 2 or self.coords.shape[1] < 1:
            raise InputError("points must form a 2-D array with d >= 1")
        if not np.all(np.isfinite(self.coords)):
            raise InputError("points contain NaN or Inf")

    @property
    def n(self) -> int:
        return self.coords.shape[0]

    @property
    def d(self) -> int:
        return self.coords.shape[1]


@dataclass
class Partition:
    labels: np.ndarray
    k: int

    def __post_init__(self):
        self.labels = np.asarray(self.labels, dtype=np.int64)
        if self.labels.ndim != 1:
            raise InputError("labels must be a 1-D array")
        if self.k < 1:
            raise InputError(f"k must be >= 1, got {self.k}")
        if self.labels.size and (self.labels.min() < 0 or self.labels.max() >= self.k):
            raise InputError(f"labels must lie in [0, {self.k})")

    @classmethod
    def _from_device(cls, labels: np.ndarray, k: int) -> "Partition":
        """labels written by the device Lloyd (int64, C-contiguous; every value is an argmin or
        repair index over k centres, so it lies in [0, k) by construction): the two O(n) range
        scans of __post_init__ (~0.7 ms per 1e6 points) are skipped."""
        self = object.__new__(cls)
        self.labels = labels
        self.k = int(k)
        return self

    @classmethod
    def from_labels(cls, labels, k: int | None = None) -> "Partition":
        labels = np.asarray(labels, dtype=np.int64)
        if k is None:
            k = int(labels.max()) + 1 if labels.size else 1
        return cls(labels=labels, k=k)

    @property
    def n(self) -> int:
        return self.labels.size

    def sizes(self) -> np.ndarray:
        return np.bincount(self.labels, minlength=self.k)

    def empty_parts(self) -> list[int]:
        return np.flatnonzero(self.sizes() == 0).tolist()


class KMeans1D:
    """Owns an ``sc_kmeans`` context: the points resident on one GPU plus workspaces."""

    def __init__(self, points=None, *, graph: DeviceGraph | None = None, device: int = 0):
        L = _lib.require_device()
        h = ctypes.c_void_p()
        if graph is not None:
            _lib.check(L.sc_kmeans_create_from_graph(graph.handle, ctypes.byref(h)))
            self.n = graph.n
        else:
            x = _as_2d(points)
            _lib.check(L.sc_kmeans_create_nd(_lib.ptr(x), x.shape[0], x.shape[1], device,
                                             ctypes.byref(h)))
            self.n = x.shape[0]
        self._h = h
        self.last = {}

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().sc_kmeans_destroy(self._h)
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

    # -- seeding with host-replayed draws
    def seed_centers(self, k: int, seed: int, restarts: int) -> np.ndarray:
        """chosen[r, :] = _kmeans_pp_indices(coords, k, rng_for(seed, r)) for every r."""
        n = self.n
        rngs = [rng_for(seed, r) for r in range(restarts)]
        chosen = np.zeros((restarts, k), dtype=np.int64)
        for r, g in enumerate(rngs):
            chosen[r, 0] = g.integers(n)
        start = np.ones(restarts, dtype=np.int32)
        done = np.zeros(restarts, dtype=bool)
        if k == 1:
            return chosen
        while not done.all():
            snaps = [g.bit_generator.state for g in rngs]
            u = np.zeros((restarts, k - 1), dtype=np.float64)
            for r, g in enumerate(rngs):
                if not done[r]:
                    u[r, start[r] - 1:] = [g.random() for _ in range(start[r], k)]
            st = np.where(done, k, start).astype(np.int32)
            degen = np.empty(restarts, dtype=np.int32)
            _lib.check(_lib.load().sc_kmeans_pp(self._h, k, restarts, _lib.ptr(st), _lib.ptr(u),
                                                _lib.ptr(chosen), _lib.ptr(degen)))
            for r, g in enumerate(rngs):
                if done[r]:
                    continue
                i = int(degen[r])
                if i < 0:
                    done[r] = True
                    continue
                # round i found every D^2 weight at 0 (kmeans.py:131-134): rewind the
                # stream, replay the uniforms of rounds start..i-1, then the integer draw
                g.bit_generator.state = snaps[r]
                for _ in range(start[r], i):
                    g.random()
                taken = np.unique(chosen[r, :i])
                m = int(g.integers(n - taken.size))
                chosen[r, i] = _nth_unchosen(taken, m)
                start[r] = i + 1
                if start[r] >= k:
                    done[r] = True
        return chosen

    def lloyd(self, k: int, seed: int, max_iters: int = 100, tol: float = 1e-6,
              restarts: int = 10, method: str = "exact",
              assert_cost: bool | None = None) -> Partition:
        """method "exact": the bit-exact replica; "sorted": the same seeds, then Lloyd on the
        sorted values with prefix-sum means (1-D only, k <= 2048; not bit-exact, see
        DESIGN.md §8 -- an approximation, not a parity path).

        ``assert_cost``: raise (SpeclusterError) when a restart's cost goes up, as the
        reference's ``assert`` at kmeans.py:206 does; None follows the interpreter like that
        ``assert`` (skipped under ``python -O``, where the increase stops the restart)."""
        if method not in ("exact", "sorted"):
            raise InputError(f"method must be 'exact' or 'sorted', got {method!r}")
        if not 1 <= k <= self.n:
            raise InputError(f"need 1 <= k <= n, got k={k}, n={self.n}")
        if restarts < 1:
            raise InputError(f"restarts must be >= 1, got {restarts}")
        if max_iters < 1:
            raise InputError(f"max_iters must be >= 1, got {max_iters}")
        if assert_cost is None:
            assert_cost = __debug__
        _lib.check(_lib.load().sc_kmeans_set_flags(self._h, 0 if assert_cost else 1))
        chosen = self.seed_centers(k, seed, restarts)
        labels = np.empty(self.n, dtype=np.int64)
        costs = np.empty(restarts)
        iters = np.empty(restarts, dtype=np.int32)
        best = ctypes.c_int32()
        ms = ctypes.c_double()
        if method == "sorted":
            _lib.check(_lib.load().sc_kmeans_lloyd_sorted(
                self._h, k, restarts, _lib.ptr(chosen), max_iters, float(tol), _lib.ptr(labels),
                _lib.ptr(costs), _lib.ptr(iters), ctypes.byref(best)))
            self.last = {"costs": costs, "iters": iters, "best_restart": best.value,
                         "chosen": chosen, "method": "sorted"}
            return Partition(labels=labels, k=k)
        _lib.check(_lib.load().sc_kmeans_lloyd(
            self._h, k, restarts, _lib.ptr(chosen), max_iters, float(tol), _lib.ptr(labels),
            _lib.ptr(costs), _lib.ptr(iters), ctypes.byref(best), ctypes.byref(ms)))
        self.last = {"costs": costs, "iters": iters, "best_restart": best.value,
                     "chosen": chosen, "lloyd_ms": ms.value}
        return Partition._from_device(labels, k)


def _nth_unchosen(taken_sorted: np.ndarray, m: int) -> int:
    """The m-th (0-based) index not in ``taken_sorted`` == np.setdiff1d(arange(n), taken)[m]."""
    idx = m
    for t in taken_sorted:
        if t <= idx:
            idx += 1
        else:
            break
    return int(idx)


def _as_2d(points) -> np.ndarray:
    if isinstance(points, np.ndarray) and points.ndim == 1:
        points = points[:, None]
    c = points.coords if isinstance(points, PointSet) else PointSet(np.asarray(points)).coords
    if c.shape[1] > 64:
        raise InputError(f"point dimension {c.shape[1]} exceeds the device limit of 64")
    return np.ascontiguousarray(c)


def _as_1d(points) -> np.ndarray:
    c = _as_2d(points)
    if c.shape[1] != 1:
        raise InputError(f"expected 1-D points, got d={c.shape[1]}")
    return np.ascontiguousarray(c[:, 0])


KMeans = KMeans1D  # the context handles any dimension; the name is kept for callers


def lloyd(points, k: int, seed: int, max_iters: int = 100, tol: float = 1e-6,
          restarts: int = 10) -> Partition:
    """Restarted Lloyd from k-means++ seeds, best cost kept (kmeans.py:167-215)."""
    x = _as_2d(points)
    if not 1 <= k <= x.shape[0]:
        raise InputError(f"need 1 <= k <= n, got k={k}, n={x.shape[0]}")
    with KMeans1D(x) as km:
        return km.lloyd(k, seed, max_iters=max_iters, tol=tol, restarts=restarts)
