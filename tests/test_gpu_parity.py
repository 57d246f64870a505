"""GPU parity: the sm_100a path (through the C-ABI) against the reference's golden
vectors and the CPU oracle.  Bar: bit-exact for x0, x_T, f and labels (the labels are
compared exactly, which implies equality up to permutation)."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_10939_b200 import (DeviceGraph, KMeans1D, RandomWalkOp, SignlessLaplacianOp,
                                   SpectralParams, fast_spectral_cluster, from_csr, lloyd,
                                   power_method)
from paper_2310_10939_b200.generate import config_sbm, sample_sbm

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(GOLD, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def c1():
    d = dict(np.load(os.path.join(GOLD, "c1.npz")))
    d["graph"] = from_csr(len(d["deg"]), d["rp"], d["col"], None, d["deg"])
    return d


@pytest.fixture(scope="module")
def wg():
    d = dict(np.load(os.path.join(GOLD, "weighted.npz")))
    d["graph"] = from_csr(len(d["deg"]), d["rp"], d["col"], d["w"], d["deg"])
    return d


def test_irwin_hall_c1(c1):
    with DeviceGraph(c1["graph"]) as dg:
        assert np.array_equal(dg.sample_irwin_hall(0, return_host=True), c1["x0"])


def test_irwin_hall_weighted_noninteger(wg):
    with DeviceGraph(wg["graph"]) as dg:
        assert np.array_equal(dg.sample_irwin_hall(3, return_host=True), wg["x0"])


@pytest.mark.parametrize("cuda_graph", [True, False])
def test_power_rw_c1(c1, cuda_graph):
    with DeviceGraph(c1["graph"]) as dg:
        dg.sample_irwin_hall(0)
        xT, f = dg.power_iterate(50, cuda_graph=cuda_graph)
        assert np.array_equal(xT, c1["xT"])
        assert np.array_equal(f, c1["f"])
        # repeat from the same x0: the cached CUDA graph replays identically
        xT2, _ = dg.power_iterate(50, cuda_graph=cuda_graph, l2_persist=True)
        assert np.array_equal(xT2, c1["xT"])


def test_power_variants_c1(c1):
    with DeviceGraph(c1["graph"]) as dg:
        dg.set_x0(c1["x0"])
        xm, _ = dg.power_iterate(10, sign=-1.0)
        assert np.array_equal(xm, c1["xT_minus10"])
        xs, fs = dg.power_iterate(50, sym=True)
        assert np.array_equal(xs, c1["xT_sym"])
        x0, f0 = dg.power_iterate(0)
        assert np.array_equal(x0, c1["x0"]) and np.array_equal(f0, c1["x0"] / c1["deg"])


def test_power_weighted(wg):
    with DeviceGraph(wg["graph"]) as dg:
        dg.set_x0(wg["x0"])
        xT, f = dg.power_iterate(40)
        assert np.array_equal(xT, wg["xT"]) and np.array_equal(f, wg["f"])
        xm, _ = dg.power_iterate(12, sign=-1.0)
        assert np.array_equal(xm, wg["xT_minus12"])


def test_unit_vs_forced_weighted_kernel(c1):
    g = c1["graph"]
    gw = from_csr(g.n, g.row_offsets, g.col_indices, np.ones(g.nnz), g.degrees)
    with DeviceGraph(gw) as dg:
        assert dg.info()["unit_weights"] == 1
        dg.set_x0(c1["x0"])
        a, _ = dg.power_iterate(20)
        b, _ = dg.power_iterate(20, force_weighted=True)
        assert np.array_equal(a, b)


def test_composition_bitwise(wg):
    """power_method(t1+t2) == power_method(power_method(t1), t2) (test_spectral.py:115-122)."""
    op = RandomWalkOp(wg["graph"])
    a = power_method(op, wg["x0"], 17)
    b = power_method(op, power_method(op, wg["x0"], 9), 8)
    assert np.array_equal(a, b)
    sym = SignlessLaplacianOp(wg["graph"])
    xs = sym.matvec(wg["x0"])
    xo, _ = O.power_iterate(wg["rp"], wg["col"], wg["w"], wg["deg"], wg["x0"], 1, variant="sym")
    assert np.array_equal(xs, xo)


def test_long_rows_and_tiles():
    """Star + clique graph: one row longer than a shared-memory chunk, many tiny rows."""
    rng = np.random.default_rng(1)
    n = 6000
    hub = np.zeros(n - 1, dtype=np.int64)
    leaves = np.arange(1, n)
    u = np.concatenate([hub, rng.integers(1, n, 20000)])
    v = np.concatenate([leaves, rng.integers(1, n, 20000)])
    keep = u != v
    from paper_2310_10939_b200 import from_edges
    g, _ = from_edges(n, u[keep], v[keep], 0.5 + rng.random(keep.sum()), drop_isolated=True)
    x0 = O.irwin_hall(g.degrees, 9)
    xo, fo = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0, 25)
    with DeviceGraph(g) as dg:
        assert dg.info()["long_rows"] >= 1
        assert np.array_equal(dg.sample_irwin_hall(9, return_host=True), x0)
        xT, f = dg.power_iterate(25)
        assert np.array_equal(xT, xo) and np.array_equal(f, fo)


def test_lloyd_c1(c1):
    part = lloyd(c1["f"][:, None], 5, seed=O.kmeans_seed(0))
    assert np.array_equal(part.labels, c1["labels"])


def test_lloyd_weighted(wg):
    part = lloyd(wg["f"][:, None], 4, seed=O.kmeans_seed(3))
    assert np.array_equal(part.labels, wg["labels"])


def test_lloyd_edge_cases(meta):
    arr = np.load(os.path.join(GOLD, "kmeans_cases.npz"))
    for name, case in meta["kmeans_cases"].items():
        x = arr[name.split("__")[0] + "__x"]
        part = lloyd(x[:, None], case["k"], seed=case["seed"])
        assert np.array_equal(part.labels, arr[name]), name


def test_pipeline_c1(c1):
    res = fast_spectral_cluster(c1["graph"], SpectralParams(k=5, t=50, mode="one_vector", seed=0),
                                keep_x=True)
    assert np.array_equal(res.x_T, c1["xT"])
    assert np.array_equal(res.embedding.data[:, 0], c1["f"])
    assert np.array_equal(res.partition.labels, c1["labels"])
    assert set(res.timings) == {"embed", "scale", "kmeans", "total"}
    assert res.l == 1 and res.t == 50


def test_pipeline_supplied_x0(wg):
    res = fast_spectral_cluster(wg["graph"], SpectralParams(k=4, t=40, mode="one_vector", seed=3,
                                                             x0=wg["x0"]))
    assert np.array_equal(res.partition.labels, wg["labels"])


def test_determinism(wg):
    p = SpectralParams(k=4, t=40, mode="one_vector", seed=3)
    a = fast_spectral_cluster(wg["graph"], p)
    b = fast_spectral_cluster(wg["graph"], p)
    assert np.array_equal(a.partition.labels, b.partition.labels)
    assert np.array_equal(a.embedding.data, b.embedding.data)


@pytest.fixture(scope="module")
def c2_graph(meta):
    g = sample_sbm(config_sbm(2)).graph
    h = hashlib.sha256()
    h.update(g.row_offsets.astype(np.int64).tobytes())
    h.update(g.col_indices.astype(np.int32).tobytes())
    h.update(g.degrees.astype(np.float64).tobytes())
    assert h.hexdigest() == meta["configs"]["c2"]["graph_sha"], "config-2 graph differs"
    return g


def test_pipeline_c2_matches_reference(c2_graph, meta):
    """Config 2 (n=1e6, nnz=44M, T=100, k=10): x0, x_T, f and labels bit-identical to
    the reference's power_method / lloyd (hashes frozen by make_golden.py)."""
    ref = meta["configs"]["c2"]
    res = fast_spectral_cluster(c2_graph, SpectralParams(k=10, t=100, mode="one_vector", seed=0),
                                keep_x=True)
    assert sha(res.x_T) == ref["xT_sha"]
    assert sha(res.embedding.data[:, 0]) == ref["f_sha"]
    assert sha(O.canonical_labels(res.partition.labels)) == ref["labels_canon_sha"]
    assert sha(res.partition.labels.astype(np.int64)) == ref["labels_sha"]


def test_c2_properties(c2_graph):
    """Size-independent properties at config 2: mass conservation 1^T M = 1^T and
    nonnegativity of the lazy walk; the x0 hash."""
    with DeviceGraph(c2_graph) as dg:
        x0 = dg.sample_irwin_hall(0, return_host=True)
        xT, f = dg.power_iterate(100)
    assert np.all(xT >= 0)
    assert abs(xT.sum() - x0.sum()) <= 1e-9 * x0.sum()
    assert np.array_equal(f, xT / c2_graph.degrees)


@pytest.mark.parametrize("case", ["dyadic", "integers", "wide_range", "tiny_subnormal", "big_n"])
def test_lloyd_exact_sums_stress(case):
    """Inputs that stress the exact sequential-sum machinery (ties to even, many binade
    crossings, subnormals, long segments) against the C oracle replica."""
    rng = np.random.default_rng(5)
    if case == "dyadic":
        x, k = rng.integers(0, 4096, 30000) * 0.125, 7
    elif case == "integers":
        x, k = rng.integers(0, 50, 20000).astype(np.float64), 5
    elif case == "wide_range":
        x, k = np.exp(rng.normal(0, 12, 20000)), 9
    elif case == "tiny_subnormal":
        x, k = rng.random(5000) * 1e-300, 4
    else:
        x, k = rng.random(300000) * 1e-3 + 0.5, 20
    lab_o, cost_o = O.lloyd(x, k, 77)
    part = lloyd(x[:, None], k, seed=77)
    assert np.array_equal(part.labels, lab_o), case


def test_recycled_buffers_partial_last_slice(wg, c1):
    """Graph buffers are recycled across handles; the lanes past n in the last SELL slice
    must be padding, not stale column indices of the previous graph (which once read out of
    bounds).  A bigger weighted graph first, then config 1 (n = 1000: a partial slice)."""
    for _ in range(2):
        with DeviceGraph(wg["graph"], keep_weights=True) as dg:
            dg.set_x0(wg["x0"])
            dg.power_iterate(3)
        with DeviceGraph(c1["graph"]) as dg:
            dg.set_x0(c1["x0"])
            xT, _ = dg.power_iterate(50, cuda_graph=False)
            assert np.array_equal(xT, c1["xT"])


def test_device_column_range_check():
    """Column arrays of >= 2^20 entries are range-checked on the device during the upload;
    a bad index still surfaces as an InputError naming it, and nothing leaks."""
    from paper_2310_10939_b200.errors import InputError

    n, per = 1 << 15, 40
    rng = np.random.default_rng(3)
    rp = np.arange(n + 1, dtype=np.int64) * per
    col = rng.integers(0, n, n * per).astype(np.int32)
    col[777_777] = n + 5
    g = from_csr(n, rp, col, None, np.full(n, float(per)))
    with pytest.raises(InputError, match=r"col_indices\[777777\]"):
        DeviceGraph(g)
    col[777_777] = 3
    with DeviceGraph(from_csr(n, rp, col, None, np.full(n, float(per)))) as dg:
        assert dg.info()["nnz"] == n * per


def test_release_cached_device_memory(c1):
    """Destroyed handles park their buffers in the reuse cache; release_device_memory frees
    them (and a second call finds nothing)."""
    from paper_2310_10939_b200.spectral import release_device_memory

    with DeviceGraph(c1["graph"]) as dg:
        dg.sample_irwin_hall(0)
    assert release_device_memory() > 0
    assert release_device_memory() == 0
