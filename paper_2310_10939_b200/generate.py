"""Seeded synthetic inputs for the hot path (host side, numpy).

``sample_sbm`` restates the reference's planted-partition sampler
(specluster/generate.py:58-149): per block pair (bi <= bj) its own stream
``rng_for(seed, 4, bi, bj)`` (:125), geometric skip-sampling of the Bernoulli pair
positions with the same batch sizes and the same ``rng.geometric`` calls (:58-73),
strict-upper-triangle decoding for diagonal blocks (:76-83), then CSR assembly with
isolated vertices dropped (:137).  Same seed => the same edges as the reference, so
config 1 and config 2 of BASELINE.json can be rebuilt on a GPU box that has no
reference installed (graph hashes pinned in tests/golden/golden.json).

``sample_dcsbm`` / ``sample_weighted_rgg`` build configs 3 and 4, which the
reference cannot generate; their construction is ours and stated in
DESIGN.md.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InputError
from .graph import Graph, from_csr, from_edges

TAG_SBM_BLOCK = 4  # generate.py:22
TAG_DCSBM = 7
TAG_RGG = 8
TAG_DEVICE_SBM = 9


def rng_for(seed: int, *tags: int) -> np.random.Generator:
    """spectral.py:32-36."""
    if seed < 0:
        raise InputError(f"seed must be a nonnegative integer, got {seed}")
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, *tags])))


@dataclass
class SbmParams:
    n: int
    k: int
    p: float
    q: float
    seed: int

    def __post_init__(self):
        if self.k < 1 or self.n < 1:
            raise InputError(f"need n >= 1 and k >= 1, got n={self.n}, k={self.k}")
        if self.n % self.k:
            raise InputError(f"k must divide n, got n={self.n}, k={self.k}")
        if not 0.0 <= self.q <= self.p <= 1.0:
            raise InputError(f"need 0 <= q <= p <= 1, got p={self.p}, q={self.q}")
        if self.seed < 0:
            raise InputError(f"seed must be nonnegative, got {self.seed}")

    @property
    def block_size(self) -> int:
        return self.n // self.k


@dataclass
class SbmSample:
    graph: Graph
    planted: np.ndarray
    dropped: list
    params: SbmParams

    def __iter__(self):
        return iter((self.graph, self.planted))


def _skip_sample(rng: np.random.Generator, trials: int, prob: float) -> np.ndarray:
    """0-based success positions among `trials` Bernoulli(prob) trials, drawn as
    geometric gaps in batches sized exactly as generate.py:64-71 sizes them."""
    if trials <= 0 or prob <= 0.0:
        return np.empty(0, dtype=np.int64)
    if prob >= 1.0:
        return np.arange(trials, dtype=np.int64)
    parts = []
    reached = 0
    while reached <= trials:
        want = max(int((trials - reached) * prob * 1.1) + 16, 16)
        steps = np.cumsum(rng.geometric(prob, size=want).astype(np.int64)) + reached
        reached = int(steps[-1])
        parts.append(steps)
    pos = np.concatenate(parts)
    return pos[pos <= trials] - 1


def _triu_pairs(pos: np.ndarray, s: int) -> tuple[np.ndarray, np.ndarray]:
    """Row-major strict-upper-triangle index -> (row, col), row < col."""
    r = np.arange(s, dtype=np.int64)
    first = r * s - r * (r + 1) // 2
    row = np.searchsorted(first, pos, side="right") - 1
    return row, pos - first[row] + row + 1


def sbm_edges(params: SbmParams) -> tuple[np.ndarray, np.ndarray]:
    s = params.block_size
    us, vs = [], []
    for bi in range(params.k):
        for bj in range(bi, params.k):
            rng = rng_for(params.seed, TAG_SBM_BLOCK, bi, bj)
            if bi == bj:
                row, col = _triu_pairs(_skip_sample(rng, s * (s - 1) // 2, params.p), s)
                us.append(row + bi * s)
                vs.append(col + bi * s)
            else:
                pos = _skip_sample(rng, s * s, params.q)
                us.append(pos // s + bi * s)
                vs.append(pos % s + bj * s)
    u = np.concatenate(us) if us else np.empty(0, dtype=np.int64)
    v = np.concatenate(vs) if vs else np.empty(0, dtype=np.int64)
    return u, v


def sample_sbm(params: SbmParams) -> SbmSample:
    u, v = sbm_edges(params)
    g, dropped = from_edges(params.n, u, v, None, drop_isolated=True)
    planted = np.repeat(np.arange(params.k, dtype=np.int64), params.block_size)
    if dropped:
        keep = np.ones(params.n, dtype=bool)
        keep[dropped] = False
        planted = planted[keep]
    return SbmSample(graph=g, planted=planted, dropped=dropped, params=params)


def sbm_rows(params: SbmParams, lo: int, hi: int):
    """Rows [lo, hi) of the SBM of ``params`` (global column ids), generating only the block
    pairs that touch those rows with the very streams ``sample_sbm`` uses -- so the shards of
    all ranks concatenate to ``sample_sbm(params).graph`` whenever no vertex is isolated
    (which sample_sbm would drop and compact).  Returns (row_ptr int64, col int32,
    degrees float64, isolated count)."""
    s = params.block_size
    b_lo, b_hi = lo // s, (hi - 1) // s
    rows, cols = [], []
    for bi in range(params.k):
        for bj in range(bi, params.k):
            if not (b_lo <= bi <= b_hi or b_lo <= bj <= b_hi):
                continue
            rng = rng_for(params.seed, TAG_SBM_BLOCK, bi, bj)
            if bi == bj:
                r, c = _triu_pairs(_skip_sample(rng, s * (s - 1) // 2, params.p), s)
                u, v = r + bi * s, c + bi * s
            else:
                pos = _skip_sample(rng, s * s, params.q)
                u, v = pos // s + bi * s, pos % s + bj * s
            for a, b in ((u, v), (v, u)):
                m = (a >= lo) & (a < hi)
                rows.append(a[m] - lo)
                cols.append(b[m])
    n = hi - lo
    r = np.concatenate(rows) if rows else np.empty(0, dtype=np.int64)
    c = np.concatenate(cols) if cols else np.empty(0, dtype=np.int64)
    key = np.unique(r * np.int64(params.n) + c)
    r, c = key // params.n, key % params.n
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=rp[1:])
    deg = np.diff(rp).astype(np.float64)
    return rp, c.astype(np.int32), deg, int(np.count_nonzero(deg == 0))


# ---------------------------------------------------------------------------
# BASELINE.json configurations


def config_sbm(cfg: int, seed: int = 0) -> SbmParams:
    """Configs 1, 2 (and 5) as SbmParams."""
    if cfg == 1:
        return SbmParams(n=1000, k=5, p=0.3, q=0.01, seed=seed)
    if cfg == 2:
        return SbmParams(n=10**6, k=10, p=40 / (10**5 - 1), q=4 / (9 * 10**5), seed=seed)
    if cfg == 5:
        return SbmParams(n=10**8, k=1000, p=16 / (10**5 - 1), q=2 / (10**8 - 10**5), seed=seed)
    raise InputError(f"config {cfg} is not an SBM config")


CONFIG_T = {1: 50, 2: 100, 3: 200, 4: 300, 5: 100}
CONFIG_K = {1: 5, 2: 10, 3: 50, 4: 100, 5: 1000}


def sample_dcsbm(n: int, k: int, seed: int, *, alpha: float = 2.0, gamma: float = 2.5,
                 dmin: float = 5.0, dmax: float = 5000.0, mix: float = 0.1,
                 wlo: float = 0.5, whi: float = 1.5) -> SbmSample:
    """Degree-corrected SBM (config 3 shape): Dirichlet(alpha) block sizes, expected
    degrees from a truncated power law d^-gamma on [dmin, dmax], a fraction `mix` of
    each vertex's stubs leaving its block, Chung-Lu style pairing by weighted sampling
    (multi-edges summed), weights Uniform(wlo, whi), symmetrised.  Our construction --
    the reference has no DC-SBM."""
    rng = rng_for(seed, TAG_DCSBM)
    sizes = np.maximum(1, np.round(rng.dirichlet(np.full(k, alpha)) * n).astype(np.int64))
    sizes[-1] += n - sizes.sum()
    if sizes[-1] < 1:
        raise InputError("dirichlet block sizes degenerate; choose another seed")
    block = np.repeat(np.arange(k), sizes)
    # inverse-CDF of the truncated power law
    a = 1.0 - gamma
    u = rng.random(n)
    deg = (dmin**a + u * (dmax**a - dmin**a)) ** (1.0 / a)
    stubs = rng.poisson(deg / 2.0)
    m = int(stubs.sum())
    src = np.repeat(np.arange(n, dtype=np.int64), stubs)
    inside = rng.random(m) >= mix
    starts = np.concatenate([[0], np.cumsum(sizes)])
    # pick partners proportional to expected degree, inside the block or anywhere
    cdf_all = np.cumsum(deg)
    dst = np.searchsorted(cdf_all, rng.random(m) * cdf_all[-1], side="right").clip(0, n - 1)
    b = block[src[inside]]
    lo = np.where(starts[b] > 0, cdf_all[starts[b] - 1], 0.0)
    hi = cdf_all[starts[b + 1] - 1]
    dst_in = np.searchsorted(cdf_all, lo + rng.random(b.size) * (hi - lo), side="right")
    dst[inside] = np.minimum(np.maximum(dst_in, starts[b]), starts[b + 1] - 1)
    w = wlo + (whi - wlo) * rng.random(m)
    keep = src != dst
    g, dropped = from_edges(n, src[keep], dst[keep], w[keep], drop_isolated=True)
    planted = block
    if dropped:
        mask = np.ones(n, dtype=bool)
        mask[dropped] = False
        planted = planted[mask]
    return SbmSample(graph=g, planted=planted, dropped=dropped,
                     params=SbmParams(n=n, k=1, p=0.0, q=0.0, seed=seed))


def sample_weighted_rgg(n: int, k: int, seed: int, *, sigma: float = 0.05, knn: int = 16,
                        scale: float = 0.01) -> SbmSample:
    """Weighted random geometric cluster graph (config 4 shape): k Gaussian centres
    Uniform[0,1]^3, sigma, each point joined to its `knn` nearest neighbours with weight
    exp(-d^2/scale), symmetrised as a union (a mutual pair is one edge).  Exact kNN with
    scipy's cKDTree on all host cores.  Our construction (the reference's kNN builder is
    brute force, unit weights and refuses n > 50,000: generate.py:178,199-200)."""
    from scipy.spatial import cKDTree

    rng = rng_for(seed, TAG_RGG)
    centres = rng.random((k, 3))
    lab = rng.integers(0, k, size=n)
    pts = centres[lab] + sigma * rng.standard_normal((n, 3))
    dist, nb = cKDTree(pts).query(pts, k=knn + 1, workers=-1)
    src = np.repeat(np.arange(n, dtype=np.int64), knn)
    dst = nb[:, 1:].ravel().astype(np.int64)
    d2 = dist[:, 1:].ravel() ** 2
    keep = src != dst  # duplicate points can displace self from column 0
    src, dst, d2 = src[keep], dst[keep], d2[keep]
    a, b = np.minimum(src, dst), np.maximum(src, dst)
    key, first = np.unique(a * np.int64(n) + b, return_index=True)
    w = np.maximum(np.exp(-d2[first] / scale), np.finfo(np.float64).tiny)
    g, dropped = from_edges(n, key // n, key % n, w, drop_isolated=True)
    planted = lab
    if dropped:
        mask = np.ones(n, dtype=bool)
        mask[dropped] = False
        planted = planted[mask]
    return SbmSample(graph=g, planted=planted, dropped=dropped,
                     params=SbmParams(n=n, k=1, p=0.0, q=0.0, seed=seed))


# ---------------------------------------------------------------------------
# device generator (sc_generate.cu): the same SBM law, realised on the GPU for sizes the
# host cannot build (config 5: n = 1e8, ~1.8e9 stored entries)


TAG_DEVICE_KNN = 10
TAG_DEVICE_DCSBM = 11


def device_key(seed: int, tag: int) -> tuple[int, int]:
    """Philox key SeedSequence([seed, tag]) of a device generator."""
    if seed < 0:
        raise InputError(f"seed must be a nonnegative integer, got {seed}")
    k = np.random.SeedSequence([seed, tag]).generate_state(2, np.uint64)
    return int(k[0]), int(k[1])


def dcsbm_block_offsets(n: int, k: int, seed: int, alpha: float = 2.0) -> np.ndarray:
    """Block offsets of the device DC-SBM: Dirichlet(alpha) sizes (host numpy, stream
    rng_for(seed, 11)), rounded, the last block taking the remainder."""
    rng = rng_for(seed, TAG_DEVICE_DCSBM)
    sizes = np.maximum(1, np.round(rng.dirichlet(np.full(k, alpha)) * n).astype(np.int64))
    sizes[-1] += n - sizes.sum()
    if sizes[-1] < 1:
        raise InputError("dirichlet block sizes degenerate; choose another seed")
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def dcsbm_power_law(gamma: float = 2.5, dmin: int = 5, dmax: int = 5000):
    """(dmin^a, dmax^a, 1/a), a = 1 - gamma: the inverse-CDF constants of the degree law."""
    a = 1.0 - gamma
    return float(dmin) ** a, float(dmax) ** a, 1.0 / a


def device_sbm_key(seed: int) -> tuple[int, int]:
    """Philox key of the device generator: SeedSequence([seed, 9]) (tag 9 unused by the
    reference, spectral.py:26-29)."""
    if seed < 0:
        raise InputError(f"seed must be a nonnegative integer, got {seed}")
    k = np.random.SeedSequence([seed, TAG_DEVICE_SBM]).generate_state(2, np.uint64)
    return int(k[0]), int(k[1])


def inv_log1m(prob: float) -> float:
    """1 / log1p(-prob), the geometric-skip scale handed to the generator (-0.0 at prob 1)."""
    import math

    if prob <= 0.0:
        return 0.0
    if prob >= 1.0:
        return -0.0
    return 1.0 / math.log1p(-prob)


class DeviceCSR:
    """A CSR generated and kept on one GPU (``sc_csr`` handle): the SBM law (configs 1, 2, 5;
    ``DeviceCSR(params)``), the degree-corrected SBM of config 3 (``DeviceCSR.dcsbm``) or the
    weighted 3-D kNN cluster graph of config 4 (``DeviceCSR.knn3d``)."""

    def __init__(self, params: SbmParams | None, device: int = 0, *, _handle=None,
                 weighted: bool = False, planted_of=None):
        import ctypes

        from . import _lib

        L = _lib.require_device()
        if _handle is None:
            k0, k1 = device_sbm_key(params.seed)
            h = ctypes.c_void_p()
            _lib.check(L.sc_generate_sbm(params.n, params.k, params.p, params.q,
                                         inv_log1m(params.p), inv_log1m(params.q), k0, k1, device,
                                         ctypes.byref(h)))
            planted_of = lambda orig: (orig // params.block_size).astype(np.int64)  # noqa: E731
        else:
            h = _handle
        self._h, self.params, self.device = h, params, device
        self.weighted = weighted
        self._planted_of = planted_of
        n, nnz, ng = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(L.sc_csr_info(h, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(ng)))
        self.n, self.nnz, self.n_generated = n.value, nnz.value, ng.value

    @classmethod
    def knn3d(cls, n: int, k: int, seed: int, *, sigma: float = 0.05, knn: int = 16,
              scale: float = 0.01, device: int = 0) -> "DeviceCSR":
        """Config 4's law on the device (sc_generate_knn3d; oracle.device_knn3d restates it)."""
        import ctypes

        from . import _lib

        L = _lib.require_device()
        k0, k1 = device_key(seed, TAG_DEVICE_KNN)
        h = ctypes.c_void_p()
        _lib.check(L.sc_generate_knn3d(n, k, float(sigma), knn, float(scale), k0, k1, device,
                                       ctypes.byref(h)))
        return cls(None, device, _handle=h, weighted=True)

    @classmethod
    def dcsbm(cls, n: int, k: int, seed: int, *, alpha: float = 2.0, gamma: float = 2.5,
              dmin: int = 5, dmax: int = 5000, mix: float = 0.1, wlo: float = 0.5,
              whi: float = 1.5, device: int = 0) -> "DeviceCSR":
        """Config 3's law on the device (sc_generate_dcsbm; oracle.device_dcsbm restates it)."""
        import ctypes

        from . import _lib

        L = _lib.require_device()
        offs = dcsbm_block_offsets(n, k, seed, alpha)
        A, B, inv_a = dcsbm_power_law(gamma, dmin, dmax)
        k0, k1 = device_key(seed, TAG_DEVICE_DCSBM)
        h = ctypes.c_void_p()
        _lib.check(L.sc_generate_dcsbm(n, _lib.ptr(offs), k, A, B, inv_a, dmin, dmax, float(mix),
                                       float(wlo), float(whi), k0, k1, device, ctypes.byref(h)))
        planted_of = lambda orig: (np.searchsorted(offs, orig, side="right") - 1).astype(np.int64)  # noqa: E731
        return cls(None, device, _handle=h, weighted=True, planted_of=planted_of)

    @property
    def handle(self):
        if not self._h:
            raise InputError("device CSR is closed")
        return self._h

    def download(self, pinned: bool = False) -> SbmSample:
        """Copy to host arrays (optionally page-locked, for fast re-upload) -> SbmSample with
        the planted labels of the kept vertices."""
        from . import _lib

        def empty(count, dtype):
            if pinned:  # the array's base keeps the page-locked tensor alive
                import torch

                tdt = {np.int64: torch.int64, np.int32: torch.int32, np.float64: torch.float64}
                return torch.empty(count, dtype=tdt[dtype], pin_memory=True).numpy()
            return np.empty(count, dtype=dtype)

        rp, col = empty(self.n + 1, np.int64), empty(self.nnz, np.int32)
        deg, orig = empty(self.n, np.float64), np.empty(self.n, dtype=np.int32)
        _lib.check(_lib.load().sc_csr_download(self.handle, _lib.ptr(rp), _lib.ptr(col),
                                               _lib.ptr(deg), _lib.ptr(orig)))
        val = None
        if self.weighted:
            val = empty(self.nnz, np.float64)
            _lib.check(_lib.load().sc_csr_download_weights(self.handle, _lib.ptr(val)))
        g = Graph(n=self.n, row_offsets=rp, col_indices=col, weights=val, degrees=deg)
        planted = self._planted_of(orig) if self._planted_of else None
        kept = np.zeros(self.n_generated, dtype=bool)
        kept[orig] = True
        return SbmSample(graph=g, planted=planted, dropped=list(np.flatnonzero(~kept)),
                         params=self.params)

    def close(self) -> None:
        if getattr(self, "_h", None):
            from . import _lib

            _lib.load().sc_csr_destroy(self._h)
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


def config_device_csr(cfg: int, seed: int = 0, device: int = 0) -> DeviceCSR:
    """BASELINE.json configs 3, 4 and 5 generated on the device."""
    if cfg == 3:
        return DeviceCSR.dcsbm(4_000_000, 50, seed, device=device)
    if cfg == 4:
        return DeviceCSR.knn3d(10_000_000, 100, seed, device=device)
    if cfg == 5:
        return DeviceCSR(config_sbm(5, seed), device)
    raise InputError(f"config {cfg} has no device generator (configs 1 and 2 use sample_sbm)")


def sample_sbm_device(params: SbmParams, device: int = 0, pinned: bool = False) -> SbmSample:
    with DeviceCSR(params, device) as d:
        return d.download(pinned=pinned)
