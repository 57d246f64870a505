"""Weighted undirected graph in CSR form -- the hot path's input layout.

Mirrors ``specluster.graph.Graph`` (graph.py:28-95) field for field, so a reference
``Graph`` instance and this one are interchangeable at the ``fast_spectral_cluster``
boundary.  Differences are storage-only: ``col_indices`` may be int32 (the device
layout) and ``row_offsets`` is int64.

``from_edges`` restates graph.py:98-184 (symmetrise, sum duplicates, sort columns,
weighted degrees as ``np.add.reduceat`` of each row -- the same call scipy's
``csr.sum(axis=1)`` makes, graph.py:152 -- isolated/self-loop policy) in numpy without
scipy, so the GPU box can build inputs without the reference.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import InputError


@dataclass
class Graph:
    n: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    weights: np.ndarray | None
    degrees: np.ndarray
    self_loop_weights: np.ndarray | None = None
    _unit: bool | None = field(default=None, repr=False, compare=False)

    @property
    def nnz(self) -> int:
        return int(self.col_indices.size)

    @property
    def num_edges(self) -> int:
        return self.nnz // 2

    @property
    def total_volume(self) -> float:
        return float(self.degrees.sum())

    def unit_weights(self) -> bool:
        """True when every stored weight is exactly 1.0 (or weights is None)."""
        if self._unit is None:
            w = self.weights
            object.__setattr__(self, "_unit", w is None or bool(np.all(w == 1.0)))
        return bool(self._unit)

    def validate(self) -> None:
        """Structural checks needed by the device path (graph.py:72-95 subset)."""
        validate_csr(self.n, self.row_offsets, self.col_indices, self.weights, self.degrees)


def validate_csr(n, row_offsets, col_indices, weights, degrees) -> None:
    if n < 1:
        raise InputError(f"graph must have n >= 1 vertices, got {n}")
    rp = np.asarray(row_offsets)
    if rp.shape != (n + 1,):
        raise InputError("row_offsets must have length n+1")
    if rp[0] != 0 or np.any(np.diff(rp) < 0):
        raise InputError("row_offsets must start at 0 and be nondecreasing")
    nnz = int(rp[-1])
    if np.asarray(col_indices).shape != (nnz,):
        raise InputError("col_indices length must equal row_offsets[-1]")
    if weights is not None and np.asarray(weights).shape != (nnz,):
        raise InputError("weights length must equal row_offsets[-1]")
    d = np.asarray(degrees)
    if d.shape != (n,):
        raise InputError("degrees must have length n")
    if not np.all(d > 0) or not np.all(np.isfinite(d)):
        raise InputError("degrees must be positive and finite (isolated vertices are not allowed)")
    if nnz:
        c = np.asarray(col_indices)
        if c.min() < 0 or c.max() >= n:
            raise InputError("col_indices out of range [0, n)")


def from_csr(n, row_offsets, col_indices, weights=None, degrees=None) -> Graph:
    """Wrap CSR arrays; degrees default to per-row weight sums (np.add.reduceat)."""
    rp = np.ascontiguousarray(row_offsets, dtype=np.int64)
    col = np.ascontiguousarray(col_indices, dtype=np.int32 if n < 2**31 else np.int64)
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    if degrees is None:
        degrees = row_weight_sums(rp, w, n)
    g = Graph(n=int(n), row_offsets=rp, col_indices=col, weights=w,
              degrees=np.ascontiguousarray(degrees, dtype=np.float64))
    return g


def row_weight_sums(rp: np.ndarray, w: np.ndarray | None, n: int) -> np.ndarray:
    counts = np.diff(rp)
    if w is None:
        return counts.astype(np.float64)
    out = np.zeros(n, dtype=np.float64)
    nz = counts > 0
    if w.size:
        # scipy's csr.sum(axis=1) is np.add.reduceat(data, indptr[:-1]) (probe-verified);
        # reduceat on an empty row would return the next element, hence the mask.
        out[nz] = np.add.reduceat(w, rp[:-1][nz])
    return out


def from_edges(n: int, u, v, w=None, *, allow_self_loops: bool = False,
               drop_isolated: bool = False) -> tuple[Graph, list[int]]:
    """Build a Graph from an undirected edge list (graph.py:98-184 semantics)."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    w = np.ones(u.size) if w is None else np.asarray(w, dtype=np.float64)
    unit = bool(np.all(w == 1.0))
    if not (u.size == v.size == w.size):
        raise InputError("edge arrays u, v, w must have equal length")
    if u.size and (min(u.min(), v.min()) < 0 or max(u.max(), v.max()) >= n):
        raise InputError(f"vertex id out of range [0, {n})")
    if np.any(w <= 0) or not np.all(np.isfinite(w)):
        raise InputError("edge weights must be strictly positive and finite")
    loops = u == v
    self_loops = None
    if np.any(loops):
        if not allow_self_loops:
            raise InputError(f"self-loops present at vertices {np.unique(u[loops])[:8].tolist()}")
        self_loops = np.zeros(n)
        np.add.at(self_loops, u[loops], w[loops])
        u, v, w = u[~loops], v[~loops], w[~loops]

    rows = np.concatenate([u, v])
    cols = np.concatenate([v, u])
    key = rows * np.int64(n) + cols
    if unit:
        key, counts = np.unique(key, return_counts=True)  # sorted by (row, col)
        vals = None if np.all(counts == 1) else counts.astype(np.float64)
    else:
        order = np.argsort(key, kind="stable")
        ks = key[order]
        ws = np.concatenate([w, w])[order]
        key, start = np.unique(ks, return_index=True)
        # duplicates are summed in their (stable) input order
        vals = np.add.reduceat(ws, start) if ws.size else ws
    r = key // n
    c = key % n
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=rp[1:])
    deg = row_weight_sums(rp, vals, n)
    if self_loops is not None:
        deg = deg + self_loops
    dropped: list[int] = []
    iso = deg == 0
    if np.any(iso):
        if not drop_isolated:
            raise InputError(f"isolated vertices present: {np.flatnonzero(iso)[:8].tolist()}")
        dropped = np.flatnonzero(iso).tolist()
        keep = ~iso
        newid = np.cumsum(keep) - 1
        # isolated rows have no entries and no vertex points at them
        c = newid[c]
        counts = np.diff(rp)[keep]
        n = int(keep.sum())
        if n == 0:
            raise InputError("graph is empty after dropping isolated vertices")
        rp = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=rp[1:])
        deg = deg[keep]
        if self_loops is not None:
            self_loops = self_loops[keep]
    g = Graph(n=n, row_offsets=rp, col_indices=c.astype(np.int32 if n < 2**31 else np.int64),
              weights=None if vals is None else vals, degrees=deg, self_loop_weights=self_loops)
    return g, dropped


def as_graph(g) -> Graph:
    """Accept this package's Graph or any object with the reference Graph's fields."""
    if isinstance(g, Graph):
        return g
    for attr in ("n", "row_offsets", "col_indices", "weights", "degrees"):
        if not hasattr(g, attr):
            raise InputError(f"object of type {type(g).__name__} is not a Graph (missing {attr})")
    w = np.asarray(g.weights, dtype=np.float64) if g.weights is not None else None
    return Graph(n=int(g.n), row_offsets=np.ascontiguousarray(g.row_offsets, dtype=np.int64),
                 col_indices=np.ascontiguousarray(g.col_indices, dtype=np.int32),
                 weights=w, degrees=np.ascontiguousarray(g.degrees, dtype=np.float64),
                 self_loop_weights=getattr(g, "self_loop_weights", None))
