"""The host-numerics contracts the device replica pins, re-checked ON THE GPU BOX's host (these
run with `-m gpu`, i.e. where the reference would actually run beside the GPU):

* numpy's einsum("ij,ij->") summation order (kmeans.py:96-103's cost) on this machine's numpy
  build equals the golden known answers the replica's cost order was pinned to in the build
  container (a different SIMD dispatch would change the order, and with it costs and stop
  decisions);
* when the unmodified reference package is present in baseline/_ref (bench.py's reference
  baseline), its own kmeans_cost and its own power_method + lloyd on config 1 agree with the
  device path bit for bit on this host."""

import json
import os
import sys

import numpy as np
import pytest

from paper_2310_10939_b200 import SpectralParams, fast_spectral_cluster, from_csr

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(GOLD, "golden.json")) as fh:
        return json.load(fh)


def _einsum_inputs():
    rng = np.random.default_rng(99)
    for nn in (1, 7, 8, 9, 17, 8191, 8192, 8193, 20000, 100003):
        yield nn, (rng.random((nn, 1)) - 0.5) * 1e-4


def test_box_numpy_einsum_order(meta):
    for nn, dd in _einsum_inputs():
        assert float(np.einsum("ij,ij->", dd, dd)) == meta["einsum_known_answers"][str(nn)]["value"], nn


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "specluster")):
        pytest.skip("reference package not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import specluster.kmeans as K
    import specluster.pipeline as P
    import specluster.spectral as S

    return K, S, P


def test_box_reference_kmeans_cost(ref):
    """the reference's own kmeans_cost on this host == the replica's einsum-order restatement"""
    from oracle import oracle as O

    K, _, _ = ref
    rng = np.random.default_rng(5)
    for nn in (1, 9, 8191, 8193, 100003):
        pts = 0.3 + 1e-6 * rng.standard_normal((nn, 1))
        labels = rng.integers(0, 3, nn)
        labels[:3] = [0, 1, 2][: min(3, nn)]
        part = K.Partition(labels=labels, k=3)
        means = K.cluster_means(pts, part.labels, 3)
        diff = (pts - means[part.labels])[:, 0]
        assert K.kmeans_cost(pts, part) == O.einsum_sumsq(np.ascontiguousarray(diff)), nn


def test_box_reference_pipeline_c1(ref):
    K, S, P = ref
    d = dict(np.load(os.path.join(GOLD, "c1.npz")))
    g = from_csr(len(d["deg"]), d["rp"], d["col"], None, d["deg"])
    res = fast_spectral_cluster(g, SpectralParams(k=5, t=50, mode="one_vector", seed=0), keep_x=True)
    from specluster.graph import Graph as RGraph

    rg = RGraph(g.n, g.row_offsets, g.col_indices, np.ones(g.nnz), g.degrees)
    A, deg = rg.adjacency_csr(), g.degrees
    xT = S.power_method(lambda x: 0.5 * x + 0.5 * (A @ (x / deg)), d["x0"], 50)
    assert np.array_equal(xT, res.x_T)
    f = xT / deg
    assert np.array_equal(f, res.embedding.data[:, 0])
    part = K.lloyd(K.PointSet(f[:, None]), 5, P._kmeans_seed(0))
    assert np.array_equal(part.labels, res.partition.labels)
