"""The exact sequential-sum engine behind the k-means replica (sc_seqsum) against
np.cumsum, on inputs built to hit every path: ties to even, binade crossings, zero and
subnormal prefixes, spikes, wide dynamic range, many segments."""

import numpy as np
import pytest

from paper_2310_10939_b200 import _lib

pytestmark = pytest.mark.gpu


def run(vals, offs):
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    offs = np.asarray(offs, dtype=np.int64)
    tot = np.empty(len(offs) - 1)
    nch = int(sum((offs[i + 1] - offs[i] + 255) // 256 for i in range(len(offs) - 1)))
    cs = np.empty(max(nch, 1))
    _lib.check(_lib.load().sc_seqsum(_lib.ptr(vals), len(offs) - 1, _lib.ptr(offs), 0,
                                     _lib.ptr(tot), _lib.ptr(cs)))
    return tot, cs


def cases():
    rng = np.random.default_rng(0)
    return {
        "uniform": rng.random(100000),
        "wide": np.exp(rng.normal(0, 12, 20000)),
        "wide2": np.exp(rng.normal(0, 40, 20000)),
        "dyadic": rng.integers(0, 4096, 50000) * 0.125,
        "ints": rng.integers(0, 3, 70000).astype(float),
        "zeros_then": np.concatenate([np.zeros(1000), rng.random(5000)]),
        "subnormal": rng.random(3000) * 1e-310,
        "spiky": np.where(rng.random(50000) < 0.001, 1e30, rng.random(50000)),
        "d2like": (rng.random(20000) - 0.5) ** 2 * np.exp(rng.normal(0, 10, 20000)),
        "above_2p53": rng.random(20000) * 2.0**60,
        "single": np.array([3.5]),
    }


@pytest.mark.parametrize("name", list(cases()))
def test_seqsum_matches_cumsum(name):
    a = cases()[name]
    tot, cs = run(a, [0, a.size])
    cum = np.concatenate([[0.0], np.cumsum(a)])
    assert tot[0] == cum[-1]
    starts = cum[np.arange(0, a.size, 256)]
    assert np.array_equal(cs[: starts.size], starts)


def test_seqsum_segments_and_negatives():
    rng = np.random.default_rng(1)
    a = np.exp(rng.normal(0, 8, 200000))
    a[5000:5100] *= -1.0  # a segment with negative values takes the plain path
    offs = [0] + np.sort(rng.choice(np.arange(1, a.size), 99, replace=False)).tolist() + [a.size]
    tot, _ = run(a, offs)
    ref = np.array([np.cumsum(a[offs[i]:offs[i + 1]])[-1] for i in range(len(offs) - 1)])
    assert np.array_equal(tot, ref)


@pytest.mark.parametrize("name", ["uniform", "wide", "dyadic", "spiky", "above_2p53"])
def test_seqsum_all_nonpositive_segments(name):
    """Segments whose elements are all <= 0 are summed as negated nonnegative sums (the
    rounding is symmetric); totals and chunk starts must still equal np.cumsum's."""
    a = -cases()[name]
    a[::97] = -0.0
    tot, cs = run(a, [0, a.size])
    cum = np.concatenate([[0.0], np.cumsum(a)])
    assert tot[0] == cum[-1]
    starts = cum[np.arange(0, a.size, 256)]
    assert np.array_equal(cs[: starts.size], starts)


def test_seqsum_mixed_sign_segments_batch():
    """Many segments: nonnegative, nonpositive and mixed-sign ones side by side."""
    rng = np.random.default_rng(9)
    a = np.exp(rng.normal(0, 6, 300000))
    offs = [0] + np.sort(rng.choice(np.arange(1, a.size), 199, replace=False)).tolist() + [a.size]
    for i in range(0, 200, 3):  # every third segment all negative
        a[offs[i]:offs[i + 1]] *= -1.0
    for i in range(1, 200, 7):  # some mixed
        a[offs[i]:offs[i + 1]:5] *= -1.0
    tot, _ = run(a, offs)
    ref = np.array([np.cumsum(a[offs[i]:offs[i + 1]])[-1] if offs[i + 1] > offs[i] else 0.0
                    for i in range(len(offs) - 1)])
    assert np.array_equal(tot, ref)
