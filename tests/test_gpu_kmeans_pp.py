"""k-means++ seeding (kmeans.py:121-137) on the device against the oracle's own k-means++
(oracle/sc_oracle.c orc_kmeanspp with the host replaying the same numpy draws), for the
paths the library picks by size: the one-CTA-per-restart small path (n <= 4096), the one-pass
round (update + speculative chunk maps + fix-up + super-chunk walk + super search) and the
classic per-round pipeline (SC_KPP_CLASSIC).  Inputs include narrow bands (the shape of the
embeddings at configs 2-5, where most weights become exact zeros and rounding noise decides
the draws), padding at the end of the weight stride, and duplicate points (degenerate rounds
replayed on the host)."""

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_10939_b200 import KMeans1D
from paper_2310_10939_b200.generate import rng_for

pytestmark = pytest.mark.gpu


def _oracle_seeds(x, k, seed, R):
    return np.stack([O.kmeanspp_indices(x, k, rng_for(seed, r)) for r in range(R)])


CASES = {
    "small_band": (lambda r: 0.5 + 1e-9 * r.standard_normal(3000), 20),
    "band_300k": (lambda r: 0.5 + 1e-9 * r.standard_normal(300_001), 40),
    "wide_band_300k": (lambda r: 0.4999 + 1e-6 * r.standard_normal(300_000), 40),
    "uniform_1m": (lambda r: r.random(1_000_003), 30),
    "negative_500k": (lambda r: -1.0 - r.random(500_000) ** 3, 25),
    "duplicates": (lambda r: np.repeat(r.random(40), 2500), 60),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("classic", [False, True])
def test_kmeanspp_matches_oracle(case, classic, monkeypatch):
    make, k = CASES[case]
    x = make(np.random.default_rng(11))
    if classic:
        monkeypatch.setenv("SC_KPP_CLASSIC", "1")
    with KMeans1D(x) as km:
        ch = km.seed_centers(k, 5, 10)
    assert np.array_equal(ch, _oracle_seeds(x, k, 5, 10))


def test_kmeanspp_restart_counts():
    # 1 and 64 restarts (the one-pass round keeps per-restart state for up to 64)
    x = 0.25 + 1e-7 * np.random.default_rng(3).standard_normal(200_000)
    for R in (1, 64):
        with KMeans1D(x) as km:
            ch = km.seed_centers(12, 9, R)
        assert np.array_equal(ch, _oracle_seeds(x, 12, 9, R))


@pytest.mark.parametrize("case", ["band_300k", "uniform_1m", "negative_500k", "duplicates",
                                  "wide_band_300k"])
@pytest.mark.parametrize("mode", ["nofast", "scale_1e4", "scale_1e7", "scale_1e12"])
def test_certified_fast_draw_and_fallback(case, mode, monkeypatch):
    """the certified fast draw (k_kpp_fast: tree-order prefix sums with a rigorous bound against
    the reference's sequential cumsum) against the exact pipeline: off, and with its margin
    widened so that a growing share of the draws is NOT certified and falls back to the exact
    pipeline within the same round (1e12: every draw) -- the seeds never change"""
    make, k = CASES[case]
    x = make(np.random.default_rng(11))
    if mode == "nofast":
        monkeypatch.setenv("SC_KPP_NOFAST", "1")
    else:
        monkeypatch.setenv("SC_KPP_EPS_SCALE", mode.split("_")[1])
    with KMeans1D(x) as km:
        ch = km.seed_centers(k, 5, 10)
    assert np.array_equal(ch, _oracle_seeds(x, k, 5, 10))
