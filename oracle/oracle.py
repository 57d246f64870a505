"""CPU oracle for the one-vector hot path.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs
(``cpu_baseline``, ``--impl reference``) may import this module.  The product package
``paper_2310_10939_b200`` never imports it, and has no CPU fallback.

Two layers, each pinned against golden vectors made by running the reference package
itself (``tests/golden/make_golden.py``):

* ``liboracle`` -- ctypes bindings to ``sc_oracle.c`` (bit-exact C restatement; fast
  enough for configs 1-2 and the CPU baseline).
* ``np_*`` -- numpy/scipy restatements that call the *same* third-party numerics the
  reference calls (scipy ``csr_matvec``, ``np.add.at``, ``np.cumsum``, ``np.einsum``),
  used at small sizes to cross-check the C layer.

Reference anchors (``/root/reference/pkg/src/specluster``):
  rng_for                 spectral.py:32-36
  power_method            spectral.py:87-102  (rw callable: SURVEY.md CS2)
  SignlessLaplacianOp     spectral.py:46-57
  _kmeans_seed            pipeline.py:123-124
  _kmeans_pp_indices      kmeans.py:121-137  (+ _weighted_index :116-118)
  lloyd                   kmeans.py:167-215
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libsc_oracle.so")

TAG_KMEANS = 2  # pipeline.py:47
TAG_IRWIN_HALL = 6  # first unused stream tag (spectral.py:28-29, pipeline.py:47-48, generate.py:22)

_lib = None


def build() -> str:
    """Compile sc_oracle.c with its Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, i32, f64, u64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_uint64
        L.orc_philox4x64_10.argtypes = [P, P, P]
        L.orc_irwin_hall.argtypes = [i64, P, u64, u64, P, i32, i64]
        L.orc_power_iterate.argtypes = [i64, P, P, P, P, P, i32, i32, f64, P, P, i32]
        L.orc_einsum_sumsq.argtypes = [i64, P]
        L.orc_einsum_sumsq.restype = f64
        L.orc_kmeanspp.argtypes = [i64, P, i32, i32, P, P]
        L.orc_kmeanspp.restype = i32
        L.orc_lloyd_restart.argtypes = [i64, P, i32, P, i32, f64, P, P]
        L.orc_lloyd_restart.restype = i32
        L.orc_rw_rows.argtypes = [i64, P, P, P, P, P, P, i32, f64, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


# ---------------------------------------------------------------------------
# seeds (host conventions shared with the product)


def rng_for(seed: int, *tags: int) -> np.random.Generator:
    """spectral.py:32-36: Generator(PCG64(SeedSequence([seed, *tags])))."""
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, *tags])))


def kmeans_seed(seed: int) -> int:
    """pipeline.py:123-124."""
    return int(np.random.SeedSequence([seed, TAG_KMEANS]).generate_state(1)[0])


def irwin_hall_key(seed: int) -> tuple[int, int]:
    k = np.random.SeedSequence([seed, TAG_IRWIN_HALL]).generate_state(2, np.uint64)
    return int(k[0]), int(k[1])


# ---------------------------------------------------------------------------
# C layer


def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint64)
    k = np.ascontiguousarray(key, dtype=np.uint64)
    out = np.empty(4, dtype=np.uint64)
    lib().orc_philox4x64_10(_p(c), _p(k), _p(out))
    return out


def irwin_hall(degrees: np.ndarray, seed: int, threads: int = 1, row0: int = 0) -> np.ndarray:
    """x0 for vertices row0 .. row0+len(degrees)-1 (global ids)."""
    d = np.ascontiguousarray(degrees, dtype=np.float64)
    k0, k1 = irwin_hall_key(seed)
    x0 = np.empty_like(d)
    lib().orc_irwin_hall(d.size, _p(d), k0, k1, _p(x0), threads, int(row0))
    return x0


def power_iterate(row_offsets, col_indices, weights, degrees, x0, t: int, *, variant: str = "rw",
                  sign: float = 1.0, threads: int = 1):
    """Returns (x_T, f).  weights=None means unit weights."""
    rp = np.ascontiguousarray(row_offsets, dtype=np.int64)
    col = np.ascontiguousarray(col_indices, dtype=np.int32)
    val = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    deg = np.ascontiguousarray(degrees, dtype=np.float64)
    x = np.ascontiguousarray(x0, dtype=np.float64)
    n = deg.size
    xT = np.empty(n)
    f = np.empty(n)
    lib().orc_power_iterate(n, _p(rp), _p(col), _p(val), _p(deg), _p(x), int(t),
                            0 if variant == "rw" else 1, float(sign), _p(xT), _p(f), threads)
    return xT, f


def rw_rows(row_offsets, col_indices, weights, degrees, x, z, *, variant="rw", sign=1.0):
    """One step for a block of rows given the full gathered z; returns (y, z_out)."""
    rp = np.ascontiguousarray(row_offsets, dtype=np.int64)
    col = np.ascontiguousarray(col_indices, dtype=np.int32)
    val = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    deg = np.ascontiguousarray(degrees, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    z = np.ascontiguousarray(z, dtype=np.float64)
    n = deg.size
    y = np.empty(n)
    zo = np.empty(n)
    lib().orc_rw_rows(n, _p(rp), _p(col), _p(val), _p(deg), _p(x), _p(z),
                      0 if variant == "rw" else 1, float(sign), _p(y), _p(zo))
    return y, zo


def einsum_sumsq(v: np.ndarray) -> float:
    v = np.ascontiguousarray(v, dtype=np.float64)
    return float(lib().orc_einsum_sumsq(v.size, _p(v)))


def kmeanspp_indices(x: np.ndarray, k: int, rng: np.random.Generator) -> np.ndarray:
    """_kmeans_pp_indices (kmeans.py:121-137) with the C replica doing the data work and
    the host issuing the very same rng calls in the same order."""
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    n = x.size
    chosen = np.zeros(k, dtype=np.int64)
    chosen[0] = rng.integers(n)
    start = 1
    while start < k:
        snap = rng.bit_generator.state
        u = np.array([rng.random() for _ in range(start, k)], dtype=np.float64)
        draws = np.zeros(max(k - 1, 1))
        draws[start - 1:k - 1] = u
        ret = lib().orc_kmeanspp(n, _p(x), k, start, _p(draws), _p(chosen))
        if ret < 0:
            break
        # degenerate round `ret`: rewind, replay the uniform draws of rounds start..ret-1,
        # then the uniform-over-unchosen integer draw (kmeans.py:131-134)
        rng.bit_generator.state = snap
        for _ in range(start, ret):
            rng.random()
        unchosen = np.setdiff1d(np.arange(n), chosen[:ret])
        chosen[ret] = int(unchosen[rng.integers(unchosen.size)])
        start = ret + 1
    return chosen


def lloyd(x: np.ndarray, k: int, seed: int, max_iters: int = 100, tol: float = 1e-6,
          restarts: int = 10, threads: int = 0,
          assert_cost: bool = True) -> tuple[np.ndarray, float]:
    """lloyd (kmeans.py:167-215) on 1-D points; returns (labels int64, best cost).  Restarts
    are independent (rng_for(seed, r) each) and run on `threads` host threads (0 = all cores;
    the C calls release the GIL); the best is picked in restart order exactly as the loop does.
    assert_cost=False is the reference under `python -O` (kmeans.py:206's assert skipped: a
    cost increase ends the restart through the small-gain test, with that cost and labels)."""
    import concurrent.futures as cf
    import os

    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    n = x.size

    def one(r):
        rng = rng_for(seed, r)
        centers = x[kmeanspp_indices(x, k, rng)].copy()
        cost = ctypes.c_double()
        labels = np.empty(n, dtype=np.int64)
        it = lib().orc_lloyd_restart(n, _p(x), k, _p(centers), max_iters, tol, _p(labels),
                                     ctypes.byref(cost))
        return labels, cost.value, it

    nt = min(restarts, threads or os.cpu_count() or 1)
    if nt <= 1:
        results = [one(r) for r in range(restarts)]
    else:
        with cf.ThreadPoolExecutor(nt) as ex:
            results = list(ex.map(one, range(restarts)))
    best_labels, best_cost = None, np.inf
    for r, (labels, cost, it) in enumerate(results):
        if it < 0 and assert_cost:  # `assert cost <= prev_cost*(1+1e-12)+1e-12` (kmeans.py:206)
            raise AssertionError(f"k-means cost increased (restart {r}, iteration {-it - 1})")
        if cost < best_cost:
            best_cost, best_labels = cost, labels
    return best_labels, best_cost


# ---------------------------------------------------------------------------
# numpy / scipy layer (same third-party numerics as the reference; small sizes)


def np_irwin_hall(degrees: np.ndarray, seed: int) -> np.ndarray:
    """Per-vertex numpy Philox streams; slow (one Generator per vertex)."""
    key = np.array(irwin_hall_key(seed), dtype=np.uint64)
    out = np.empty(len(degrees))
    for u, d in enumerate(np.asarray(degrees, dtype=np.float64)):
        m = int(np.floor(d))
        frac = d - np.floor(d)
        g = np.random.Generator(np.random.Philox(key=key, counter=[0, u, 0, 0]))
        us = g.random(m + (1 if frac > 0 else 0))
        s = 0.0
        for v in us[:m]:
            s += float(v)
        if frac > 0:
            s += float(frac * us[m])
        out[u] = s
    return out


def np_power_iterate(row_offsets, col_indices, weights, degrees, x0, t: int, variant="rw"):
    import scipy.sparse as sp

    n = len(degrees)
    w = np.ones(len(col_indices)) if weights is None else np.asarray(weights, dtype=np.float64)
    a = sp.csr_matrix((w, np.asarray(col_indices), np.asarray(row_offsets)), shape=(n, n))
    d = np.asarray(degrees, dtype=np.float64)
    x = np.array(x0, dtype=np.float64, copy=True)
    if variant == "rw":
        for _ in range(t):
            x = 0.5 * x + 0.5 * (a @ (x / d))
        return x, x / d
    s = 1.0 / np.sqrt(d)
    for _ in range(t):
        x = 0.5 * x + 0.5 * (s * (a @ (s * x)))
    return x, x * s


def np_sq_dists(x: np.ndarray, c: np.ndarray) -> np.ndarray:
    """(n,k) expanded-form distances for 1-D points, kmeans.py:106-113 order."""
    xx = (x * x)[:, None]
    return np.maximum((xx - (2.0 * x)[:, None] * c[None, :]) + (c * c)[None, :], 0.0)


def np_lloyd(x: np.ndarray, k: int, seed: int, max_iters=100, tol=1e-6, restarts=10):
    """numpy restatement of lloyd for 1-D points (kmeans.py:167-215)."""
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    n = x.size
    best, best_cost = None, np.inf
    for r in range(restarts):
        rng = rng_for(seed, r)
        # seeding (kmeans.py:121-137)
        chosen = [int(rng.integers(n))]
        near = np_sq_dists(x, x[chosen[:1]])[:, 0]
        while len(chosen) < k:
            if near.sum() > 0:
                cum = np.cumsum(near)
                pick = int(np.searchsorted(cum, rng.random() * cum[-1], side="right").clip(0, n - 1))
            else:
                rest = np.setdiff1d(np.arange(n), chosen)
                pick = int(rest[rng.integers(rest.size)])
            chosen.append(pick)
            near = np.minimum(near, np_sq_dists(x, x[[pick]])[:, 0])
        centers = x[chosen].copy()
        labels = np.zeros(n, dtype=np.int64)
        prev = np.inf
        for _ in range(max_iters):
            dist = np_sq_dists(x, centers)
            lab = np.argmin(dist, axis=1)
            own = dist[np.arange(n), lab]
            cnt = np.bincount(lab, minlength=k)
            for e in np.flatnonzero(cnt == 0):
                j = int(np.argmax(own))
                cnt[lab[j]] -= 1
                lab[j] = e
                cnt[e] = 1
                own[j] = 0.0
            same = bool(np.array_equal(lab, labels)) and np.isfinite(prev)
            labels = lab
            sums = np.zeros((k, 1))
            np.add.at(sums, labels, x[:, None])
            cnt = np.bincount(labels, minlength=k).astype(np.float64)
            centers = sums[:, 0].copy()
            centers[cnt > 0] = sums[cnt > 0, 0] / cnt[cnt > 0]
            diff = (x - centers[labels])[:, None]
            cost = float(np.einsum("ij,ij->", diff, diff))
            assert cost <= prev * (1 + 1e-12) + 1e-12, "k-means cost increased"  # kmeans.py:206
            stop = same or (np.isfinite(prev) and prev - cost <= tol * max(prev, 1e-300))
            prev = cost
            if stop:
                break
        if prev < best_cost:
            best_cost, best = prev, labels
    return best, best_cost


def canonical_labels(labels: np.ndarray) -> np.ndarray:
    """Relabel clusters in order of first appearance (labels equal up to permutation
    <=> canonical forms equal)."""
    labels = np.asarray(labels, dtype=np.int64)
    _, first = np.unique(labels, return_index=True)
    order = np.argsort(first)
    remap = np.empty(labels.max() + 1 if labels.size else 0, dtype=np.int64)
    remap[np.unique(labels)[order]] = np.arange(order.size)
    return remap[labels]


# ---------------------------------------------------------------------------
# the device SBM generator's law, restated (sc_generate.cu; not a reference algorithm -- the
# reference's per-block-pair streams cannot be replayed at config-5 scale -- so it is pinned
# by restating the generator's own counter/skip convention in numpy, op for op)

DEVICE_SBM_TAG = 0x5BD1E995


def np_sc_log(x: np.ndarray) -> np.ndarray:
    """sc_generate.cu sc_log: the same IEEE operation sequence (numpy rounds every op)."""
    x = np.asarray(x, dtype=np.float64)
    b = x.view(np.uint64)
    e = ((b >> np.uint64(52)) & np.uint64(0x7FF)).astype(np.int64) - 1023
    m = ((b & np.uint64(0x000FFFFFFFFFFFFF)) | np.uint64(0x3FF0000000000000)).view(np.float64)
    big = m > 1.4142135623730951
    m = np.where(big, m * 0.5, m)
    e = np.where(big, e + 1, e)
    t = (m - 1.0) / (m + 1.0)
    t2 = t * t
    p = np.full_like(t, 1.0 / 25.0)
    for d in (23.0, 21.0, 19.0, 17.0, 15.0, 13.0, 11.0, 9.0, 7.0, 5.0, 3.0):
        p = p * t2 + 1.0 / d
    p = p * t2 + 1.0
    return e.astype(np.float64) * 0.6931471805599453 + 2.0 * t * p


def device_sbm(n: int, k: int, p: float, q: float, seed: int):
    """Rows of the device generator's graph, built on the host (small n only).  Returns
    (row_ptr, col, deg, orig_ids) with isolated vertices dropped and ids compacted."""
    import math

    key = np.array(np.random.SeedSequence([seed, 9]).generate_state(2, np.uint64))
    inv_p = 0.0 if p <= 0 else (-0.0 if p >= 1 else 1.0 / math.log1p(-p))
    inv_q = 0.0 if q <= 0 else (-0.0 if q >= 1 else 1.0 / math.log1p(-q))
    s = n // k
    has_p, has_q = p > 0 and s > 1, q > 0 and k > 1
    us, vs = [], []
    for u in range(n):
        bg = np.random.Philox(key=key, counter=[0, u, DEVICE_SBM_TAG, 0])
        buf, pos = np.empty(0, dtype=np.uint64), 0

        def skip(inv):
            nonlocal buf, pos
            if pos == buf.size:
                buf, pos = bg.random_raw(64), 0
            raw = buf[pos]
            pos += 1
            U = float((int(raw) >> 11) + 1) * 1.1102230246251565e-16
            g = math.floor(float(np_sc_log(np.array([U]))[0] * inv))
            return (1 << 62) if g >= 4.0e18 else 1 + g

        hi = (u // s + 1) * s
        if has_p:
            v = u + skip(inv_p)
            while v < hi:
                us.append(u)
                vs.append(v)
                v += skip(inv_p)
        if has_q:
            v = hi - 1 + skip(inv_q)
            while v < n:
                us.append(u)
                vs.append(v)
                v += skip(inv_q)
    u = np.array(us, dtype=np.int64)
    v = np.array(vs, dtype=np.int64)
    r = np.concatenate([u, v])
    c = np.concatenate([v, u])
    order = np.lexsort((c, r))
    r, c = r[order], c[order]
    deg = np.bincount(r, minlength=n)
    keep = deg > 0
    newid = np.cumsum(keep) - 1
    rp = np.zeros(int(keep.sum()) + 1, dtype=np.int64)
    np.cumsum(deg[keep], out=rp[1:])
    return rp, newid[c].astype(np.int32), deg[keep].astype(np.float64), np.flatnonzero(keep)


# ---------------------------------------------------------------------------
# the weighted device generators' laws (sc_generate_wt.cu, configs 3 and 4), restated op for op
# in numpy; small n only.  Ours, not reference algorithms (the reference has no generator for
# either graph), so they are pinned by this restatement.

KNN_TAG_CENTRES, KNN_TAG_POINTS = 0x43454E54, 0x504F494E
DC_TAG_DEGREES, DC_TAG_STUBS = 0x44454752, 0x53545542
DBL_MIN = 2.2250738585072014e-308


def np_sc_exp(y: np.ndarray) -> np.ndarray:
    """sc_genmath.cuh sc_exp: Cody-Waite reduction, degree-14 Taylor, exact 2^q scaling."""
    y = np.asarray(y, dtype=np.float64)
    q = np.rint(y * 1.4426950408889634)
    r = (y - q * 0.6931471803691238) - q * 1.9082149292705877e-10
    fact = [87178291200.0, 6227020800.0, 479001600.0, 39916800.0, 3628800.0, 362880.0, 40320.0,
            5040.0, 720.0, 120.0, 24.0, 6.0]
    p = np.full_like(r, 1.0 / fact[0])
    for f in fact[1:]:
        p = p * r + 1.0 / f
    p = p * r + 0.5
    p = p * r + 1.0
    p = p * r + 1.0
    qi = np.clip(q, -1000, 1000).astype(np.int64)
    scale = ((qi + 1023).astype(np.uint64) << np.uint64(52)).view(np.float64)
    out = p * scale
    out = np.where(y > -700.0, out, 0.0)
    return np.where(y > 700.0, np.inf, out)


def _u53(raw: np.ndarray) -> np.ndarray:
    return (raw >> np.uint64(11)).astype(np.float64) * 1.1102230246251565e-16


def _words(key, ident: int, tag: int, count: int) -> np.ndarray:
    return np.random.Philox(key=key, counter=[0, ident, tag, 0]).random_raw(count)


def _seq_row_sums(rp: np.ndarray, val: np.ndarray) -> np.ndarray:
    """Each row's weights summed left to right (one rounded add per entry, column order)."""
    n = rp.size - 1
    lens = np.diff(rp)
    deg = np.zeros(n)
    for t in range(int(lens.max()) if n else 0):
        rows = np.flatnonzero(lens > t)
        deg[rows] = deg[rows] + val[rp[rows] + t]
    return deg


def _csr_from_pairs(n: int, r: np.ndarray, c: np.ndarray, w: np.ndarray):
    """Unique symmetric (r, c, w) -> (row_ptr, col, val, deg, orig) with empty rows dropped."""
    order = np.lexsort((c, r))
    r, c, w = r[order], c[order], w[order]
    lens = np.bincount(r, minlength=n)
    keep = lens > 0
    newid = np.cumsum(keep) - 1
    rp = np.zeros(int(keep.sum()) + 1, dtype=np.int64)
    np.cumsum(lens[keep], out=rp[1:])
    val = w.astype(np.float64)
    return rp, newid[c].astype(np.int32), val, _seq_row_sums(rp, val), np.flatnonzero(keep)


def device_knn3d_points(n: int, k: int, sigma: float, seed: int):
    key = np.array(np.random.SeedSequence([seed, 10]).generate_state(2, np.uint64))
    cen = np.array([_u53(_words(key, j, KNN_TAG_CENTRES, 3)) for j in range(k)])
    pts = np.empty((n, 3))
    lab = np.empty(n, dtype=np.int64)
    for i in range(n):
        u = _u53(_words(key, i, KNN_TAG_POINTS, 37))
        lb = min(int(np.floor(u[0] * float(k))), k - 1)
        lab[i] = lb
        for c in range(3):
            acc = 0.0
            for t in range(12):
                acc = acc + float(u[1 + 12 * c + t])
            pts[i, c] = float(cen[lb, c]) + sigma * (acc - 6.0)
    return pts, lab


def device_knn3d(n: int, k: int, sigma: float, knn: int, scale: float, seed: int):
    """sc_generate_knn3d restated: (row_ptr, col, val, deg, orig, points, labels)."""
    pts, lab = device_knn3d_points(n, k, sigma, seed)
    rs, cs, ws = [], [], []
    idx = np.arange(n)
    for i0 in range(0, n, 256):
        blk = pts[i0:i0 + 256]
        dx = blk[:, 0:1] - pts[None, :, 0]
        dy = blk[:, 1:2] - pts[None, :, 1]
        dz = blk[:, 2:3] - pts[None, :, 2]
        d2 = (dx * dx + dy * dy) + dz * dz
        for t in range(blk.shape[0]):
            i = i0 + t
            row = d2[t].copy()
            row[i] = np.inf
            order = np.lexsort((idx, row))[:knn]
            rs.append(np.full(knn, i))
            cs.append(order)
            ws.append(np.maximum(np_sc_exp(-(row[order] / scale)), DBL_MIN))
    r = np.concatenate(rs)
    c = np.concatenate(cs)
    w = np.concatenate(ws)
    key = np.concatenate([r * n + c, c * n + r])
    ww = np.concatenate([w, w])
    key, first = np.unique(key, return_index=True)
    rp, col, val, deg, orig = _csr_from_pairs(n, key // n, key % n, ww[first])
    return rp, col, val, deg, orig, pts, lab


def device_dcsbm(n: int, offsets, A: float, B: float, inv_a: float, dmin: int, dmax: int,
                 mix: float, wlo: float, whi: float, seed: int):
    """sc_generate_dcsbm restated: (row_ptr, col, val, deg, orig)."""
    key = np.array(np.random.SeedSequence([seed, 11]).generate_state(2, np.uint64))
    offsets = np.asarray(offsets, dtype=np.int64)
    d = np.empty(n, dtype=np.int64)
    m = np.empty(n, dtype=np.int64)
    for i in range(n):
        u = _u53(_words(key, i, DC_TAG_DEGREES, 2))
        x = np_sc_exp(np_sc_log(np.array([A + u[0] * (B - A)])) * inv_a)[0]
        fl = min(max(float(np.floor(x)), float(dmin)), float(dmax))
        d[i] = int(fl)
        m[i] = d[i] // 2 + (1 if (d[i] & 1) and u[1] < 0.5 else 0)
    cum = np.cumsum(d)
    W = int(cum[-1])
    blk = np.searchsorted(offsets, np.arange(n), side="right") - 1
    keys, ws = [], []
    for i in range(n):
        if m[i] == 0:
            continue
        u = _u53(_words(key, i, DC_TAG_STUBS, 3 * int(m[i]))).reshape(-1, 3)
        b0, b1 = int(offsets[blk[i]]), int(offsets[blk[i] + 1])
        before = int(cum[b0 - 1]) if b0 > 0 else 0
        Wb = int(cum[b1 - 1]) - before
        for ua, ub, uc in u:
            if ua >= mix:
                t = before + int(np.floor(ub * float(Wb)))
                p = b0 + int(np.searchsorted(cum[b0:b1], t, side="right"))
            else:
                t = int(np.floor(ub * float(W)))
                p = int(np.searchsorted(cum, t, side="right"))
            w = wlo + (whi - wlo) * uc
            if p == i:
                continue
            keys.append(min(i, p) * n + max(i, p))
            ws.append(w)
    keys = np.array(keys, dtype=np.int64)
    ws = np.array(ws)
    uk, first = np.unique(keys, return_index=True)  # first occurrence = first stub
    a, b = uk // n, uk % n
    w = ws[first]
    return _csr_from_pairs(n, np.concatenate([a, b]), np.concatenate([b, a]), np.concatenate([w, w]))
