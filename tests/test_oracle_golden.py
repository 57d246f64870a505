"""Pin the CPU oracle against golden vectors produced by the reference package itself
(tests/golden/make_golden.py).  No GPU needed."""

import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(GOLD, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def c1():
    return dict(np.load(os.path.join(GOLD, "c1.npz")))


@pytest.fixture(scope="module")
def wg():
    return dict(np.load(os.path.join(GOLD, "weighted.npz")))


def test_philox_known_answers(meta):
    for case in meta["philox_known_answers"].values():
        key = np.array([int(v) for v in case["key"]], dtype=np.uint64)
        ctr = [int(v) for v in case["counter"]]
        raw = []
        c = list(ctr)
        for _ in range(2):
            # numpy increments the 256-bit counter before each block
            c[0] = (c[0] + 1) % 2**64
            if c[0] == 0:
                c[1] = (c[1] + 1) % 2**64
            raw.extend(int(v) for v in O.philox(np.array(c, dtype=np.uint64), key))
        assert raw == [int(v) for v in case["raw8"]]


def test_irwin_hall_c1_matches_numpy_philox(c1):
    x0 = O.irwin_hall(c1["deg"], 0)
    assert np.array_equal(x0, c1["x0"])
    # numpy's own Philox generator draws the same uniforms (spot check 50 vertices)
    sub = O.np_irwin_hall(c1["deg"][:50], 0)
    assert np.array_equal(sub, x0[:50])


def test_irwin_hall_noninteger_degrees(wg):
    assert np.any(wg["deg"] != np.floor(wg["deg"]))
    x0 = O.irwin_hall(wg["deg"], 3, threads=4)
    assert np.array_equal(x0, wg["x0"])


def test_irwin_hall_moments():
    deg = np.full(20000, 37.0)
    x0 = O.irwin_hall(deg, 5, threads=4)
    assert abs(x0.mean() - 18.5) < 0.05
    assert abs(x0.var() - 37 / 12) < 0.15
    frac = np.full(20000, 10.25)
    y = O.irwin_hall(frac, 5)
    assert abs(y.mean() - 10.25 / 2) < 0.05


def test_power_rw_c1_bit_exact(c1):
    xT, f = O.power_iterate(c1["rp"], c1["col"], None, c1["deg"], c1["x0"], 50, threads=3)
    assert np.array_equal(xT, c1["xT"])
    assert np.array_equal(f, c1["f"])


def test_power_minus_sign_c1(c1):
    xT, _ = O.power_iterate(c1["rp"], c1["col"], None, c1["deg"], c1["x0"], 10, sign=-1.0)
    assert np.array_equal(xT, c1["xT_minus10"])


def test_power_sym_c1(c1):
    xT, _ = O.power_iterate(c1["rp"], c1["col"], None, c1["deg"], c1["x0"], 50, variant="sym")
    assert np.array_equal(xT, c1["xT_sym"])


def test_power_weighted_bit_exact(wg):
    xT, f = O.power_iterate(wg["rp"], wg["col"], wg["w"], wg["deg"], wg["x0"], 40, threads=2)
    assert np.array_equal(xT, wg["xT"])
    assert np.array_equal(f, wg["f"])
    xm, _ = O.power_iterate(wg["rp"], wg["col"], wg["w"], wg["deg"], wg["x0"], 12, sign=-1.0)
    assert np.array_equal(xm, wg["xT_minus12"])


def test_numpy_restatement_matches_c(wg):
    a, fa = O.np_power_iterate(wg["rp"], wg["col"], wg["w"], wg["deg"], wg["x0"], 7)
    b, fb = O.power_iterate(wg["rp"], wg["col"], wg["w"], wg["deg"], wg["x0"], 7)
    assert np.array_equal(a, b) and np.array_equal(fa, fb)


def test_lloyd_c1(c1, meta):
    assert O.kmeans_seed(0) == meta["kmeans_seed_0"]
    lab, _ = O.lloyd(c1["f"], 5, O.kmeans_seed(0))
    assert np.array_equal(lab, c1["labels"])


def test_lloyd_weighted(wg):
    lab, _ = O.lloyd(wg["f"], 4, O.kmeans_seed(3))
    assert np.array_equal(lab, wg["labels"])


def test_lloyd_edge_cases(meta):
    arr = np.load(os.path.join(GOLD, "kmeans_cases.npz"))
    for name, case in meta["kmeans_cases"].items():
        x = arr[name.split("__")[0] + "__x"]
        lab, _ = O.lloyd(x, case["k"], case["seed"])
        assert np.array_equal(lab, arr[name]), name
        if x.size <= 3000:
            lab2, _ = O.np_lloyd(x, case["k"], case["seed"])
            assert np.array_equal(lab2, arr[name]), name


def test_einsum_order(meta):
    rng = np.random.default_rng(99)
    # sizes in generation order (golden.json keys are sorted as strings)
    for nn in (1, 7, 8, 9, 17, 8191, 8192, 8193, 20000, 100003):
        dd = (rng.random((nn, 1)) - 0.5) * 1e-4
        assert O.einsum_sumsq(dd[:, 0]) == meta["einsum_known_answers"][str(nn)]["value"], nn


def test_canonical_labels():
    a = np.array([3, 3, 1, 0, 1, 2])
    b = np.array([0, 0, 2, 1, 2, 3])
    assert np.array_equal(O.canonical_labels(a), O.canonical_labels(b))
    assert O.canonical_labels(a).tolist() == [0, 0, 1, 2, 1, 3]
