"""The persistent exact Lloyd (csrc/sc_kmeans_fused.cu: 1-D points of one sign, k <= 32) must
reproduce the reference's restarted Lloyd (kmeans.py:167-215) bit for bit: labels against the
C oracle replica, and labels, exact einsum-order costs and iteration counts against the
general batched path (SC_KMEANS_NO_FUSED) on the same seeds.  The inputs stress what the
fused kernel does differently: chunk boundaries (n around 1024), empty-cluster repairs,
binade crossings and ties to even in the exact sums, negative inputs (run on -x), mixed signs
(fallback to the general path), restarts up to 64, max_iters 1 and 2."""

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_10939_b200 import KMeans1D

pytestmark = pytest.mark.gpu


def _run(x, k, seed, fused, **kw):
    if fused:
        os.environ.pop("SC_KMEANS_NO_FUSED", None)
    else:
        os.environ["SC_KMEANS_NO_FUSED"] = "1"
    try:
        with KMeans1D(np.ascontiguousarray(x, dtype=np.float64)) as km:
            part = km.lloyd(k, seed, **kw)
            return part.labels, km.last["costs"].copy(), km.last["iters"].copy()
    finally:
        os.environ.pop("SC_KMEANS_NO_FUSED", None)


def _cases():
    rng = np.random.default_rng(2024)
    yield "band_c2_like", 0.4999 + 1e-6 * rng.standard_normal(300_000), 10, {}
    yield "chunk_1023", rng.random(1023), 5, {}
    yield "chunk_1025", rng.random(1025), 5, {}
    yield "n_33", rng.random(33), 4, {}
    yield "n_5_k5", rng.random(5), 5, {}
    yield "k1", rng.random(5000), 1, {}
    yield "k32", rng.random(40_000) ** 3, 32, {}
    yield "restarts64", rng.random(20_000), 16, {"restarts": 64}
    yield "max_iters1", rng.random(10_000), 6, {"max_iters": 1}
    yield "max_iters2", rng.random(10_000), 6, {"max_iters": 2}
    yield "negative", -np.exp(rng.normal(0, 3, 50_000)), 8, {}
    yield "nonpositive_zeros", -np.where(rng.random(30_000) < 0.2, 0.0, rng.random(30_000)), 7, {}
    yield "duplicates_repair", np.repeat(rng.random(9), 400)[rng.permutation(3600)], 12, {"max_iters": 8}
    yield "dyadic_ties", rng.integers(0, 4096, 60_000) * 0.125, 7, {}
    yield "wide_range", np.exp(rng.normal(0, 12, 40_000)), 9, {}
    yield "subnormal", rng.random(8000) * 1e-300, 4, {}
    yield "zeros_and_ones", (rng.random(20_000) < 0.5).astype(float), 3, {}
    yield "sorted_blocks", np.sort(rng.random(200_000)), 10, {}


@pytest.mark.parametrize("name,x,k,kw", list(_cases()), ids=[c[0] for c in _cases()])
def test_fused_lloyd_matches_oracle_and_general_path(name, x, k, kw):
    lab_f, cost_f, it_f = _run(x, k, 31, True, **kw)
    lab_g, cost_g, it_g = _run(x, k, 31, False, **kw)
    assert np.array_equal(lab_f, lab_g), name
    assert np.array_equal(cost_f, cost_g), name
    assert np.array_equal(it_f, it_g), name
    lab_o, cost_o = O.lloyd(x, k, 31, **kw)
    assert np.array_equal(lab_f, lab_o), name
    assert cost_f.min() == cost_o, name


def test_mixed_signs_fall_back():
    rng = np.random.default_rng(3)
    x = rng.standard_normal(20_000)
    lab_f, cost_f, _ = _run(x, 6, 5, True)
    lab_o, cost_o = O.lloyd(x, 6, 5)
    assert np.array_equal(lab_f, lab_o)
    assert cost_f.min() == cost_o
