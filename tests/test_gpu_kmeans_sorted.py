"""The sorted-centers assignment (k >= 16) must reproduce the brute-force argmin of the
reference's rounded distance bit for bit: adversarial 1-D inputs (exact duplicates,
near-ties at the rounding level, 12 decades of magnitude, k up to 4096) against the C
oracle's brute-force Lloyd."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_10939_b200 import KMeans1D

pytestmark = pytest.mark.gpu


def _cases():
    rng = np.random.default_rng(42)
    yield "duplicates", np.repeat(rng.random(300), 7)[rng.permutation(2100)], 64
    yield "near_ties", 1.0 + 1e-13 * rng.integers(0, 50, 5000).astype(float), 40
    yield "ulp_grid", np.nextafter(1.0, 2.0) ** 0 + np.arange(3000) * 2.0**-52, 100
    yield "decades", 10.0 ** rng.uniform(-6, 6, 20000), 1000
    yield "clustered", np.concatenate([c + 1e-9 * rng.standard_normal(400)
                                       for c in rng.random(50)]), 300
    yield "big_k", rng.random(30000) * 1e-3 + 5.0, 4096


@pytest.mark.parametrize("name,x,k", list(_cases()), ids=[c[0] for c in _cases()])
def test_sorted_assignment_matches_bruteforce(name, x, k):
    x = np.ascontiguousarray(x, dtype=np.float64)
    with KMeans1D(x) as km:
        part = km.lloyd(k, 11, restarts=2)
    lab, _ = O.lloyd(x, k, 11, restarts=2)
    assert np.array_equal(part.labels, lab)


def test_cooperative_repair_matches_oracle():
    """n >= 200k takes the grid-wide (cooperative) empty-cluster repair; heavy duplication
    with k above the number of distinct values forces degenerate seeding rounds and repeated
    repairs, including the all-zero-distance argmax corner.  Labels vs the C oracle."""
    rng = np.random.default_rng(7)
    vals = rng.random(60)
    x = vals[rng.integers(0, 60, 300_000)]
    with KMeans1D(x) as km:
        part = km.lloyd(90, 3, restarts=2, max_iters=6)
    lab, _ = O.lloyd(x, 90, 3, restarts=2, max_iters=6)
    assert np.array_equal(part.labels, lab)
    x2 = np.concatenate([rng.random(250_000), np.full(50_000, 0.5)])
    with KMeans1D(x2) as km:
        part = km.lloyd(40, 5, restarts=3, max_iters=8)
    lab, _ = O.lloyd(x2, 40, 5, restarts=3, max_iters=8)
    assert np.array_equal(part.labels, lab)
