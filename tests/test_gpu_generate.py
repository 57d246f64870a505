"""Device SBM generator (sc_generate.cu): bit-exact against the numpy restatement of its
law at small sizes (incl. isolated-vertex compaction), graphs built straight from the device
CSR equal graphs uploaded from the host, and the config-5 law at scale."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_10939_b200 import DeviceGraph
from paper_2310_10939_b200.generate import DeviceCSR, SbmParams, sample_sbm_device

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,k,p,q,seed", [(3000, 3, 0.01, 0.001, 1),
                                           (2000, 10, 0.002, 0.0002, 2),  # many isolated
                                           (1200, 1, 0.02, 0.0, 3),
                                           (1000, 1000, 1.0, 0.004, 4)])
def test_device_sbm_matches_restated_law(n, k, p, q, seed):
    s = sample_sbm_device(SbmParams(n=n, k=k, p=p, q=q, seed=seed))
    rp, col, deg, orig = O.device_sbm(n, k, p, q, seed)
    g = s.graph
    assert np.array_equal(g.row_offsets, rp)
    assert np.array_equal(g.col_indices, col)
    assert np.array_equal(g.degrees, deg)
    assert np.array_equal(s.planted, orig // (n // k))
    assert len(s.dropped) == n - orig.size


def test_graph_from_device_csr_equals_host_upload():
    params = SbmParams(n=200_000, k=4, p=30 / 49_999, q=3 / 150_000, seed=7)
    with DeviceCSR(params) as d:
        host = d.download()
        with DeviceGraph.from_device_csr(d) as dg1, DeviceGraph(host.graph) as dg2:
            dg1.sample_irwin_hall(3)
            dg2.sample_irwin_hall(3)
            a, fa = dg1.power_iterate(20)
            b, fb = dg2.power_iterate(20)
            assert dg1.info()["nnz"] == host.graph.nnz
    assert np.array_equal(a, b) and np.array_equal(fa, fb)


def test_config5_law_at_scale():
    """Config 5's law (blocks of 1e5, expected degree 16 in / 2 out) at n = 5e6: symmetric,
    sorted rows without self loops, degree mean and in-block fraction as the law says."""
    n = 5_000_000
    params = SbmParams(n=n, k=n // 100_000, p=16 / (10**5 - 1), q=2 / (n - 10**5), seed=5)
    s = sample_sbm_device(params)
    g = s.graph
    rp, col = g.row_offsets, g.col_indices.astype(np.int64)
    row = np.repeat(np.arange(g.n), np.diff(rp))
    assert np.all(col != row)
    inrow = np.diff(col) > 0
    assert np.all(inrow | (np.diff(row) != 0))  # strictly increasing inside every row
    assert abs(g.nnz / g.n - 18.0) < 0.05
    same = s.planted[row] == s.planted[col]
    assert abs(same.mean() - 16 / 18) < 0.002
    # symmetry: the multiset of (row, col) equals that of (col, row)
    key = row * g.n + col
    tkey = col * g.n + row
    assert np.array_equal(np.sort(key), np.sort(tkey))


# ---- weighted device generators (sc_generate_wt.cu): configs 3 and 4


@pytest.mark.parametrize("n,k,sigma,seed", [(3000, 7, 0.05, 3),   # clustered
                                             (1500, 1, 0.3, 4),    # one diffuse cluster
                                             (600, 5, 0.0, 5)])    # exact duplicates: d2 ties
def test_device_knn3d_matches_restated_law(n, k, sigma, seed):
    with DeviceCSR.knn3d(n, k, seed, sigma=sigma) as d:
        s = d.download()
    rp, col, val, deg, orig, _, _ = O.device_knn3d(n, k, sigma, 16, 0.01, seed)
    g = s.graph
    assert np.array_equal(g.row_offsets, rp)
    assert np.array_equal(g.col_indices, col)
    assert np.array_equal(g.weights, val)
    assert np.array_equal(g.degrees, deg)


@pytest.mark.parametrize("n,k,seed", [(3000, 6, 2), (2500, 1, 7), (4000, 40, 9)])
def test_device_dcsbm_matches_restated_law(n, k, seed):
    from paper_2310_10939_b200.generate import dcsbm_block_offsets, dcsbm_power_law

    with DeviceCSR.dcsbm(n, k, seed) as d:
        s = d.download()
    offs = dcsbm_block_offsets(n, k, seed)
    A, B, inv_a = dcsbm_power_law()
    rp, col, val, deg, orig = O.device_dcsbm(n, offs, A, B, inv_a, 5, 5000, 0.1, 0.5, 1.5, seed)
    g = s.graph
    assert np.array_equal(g.row_offsets, rp)
    assert np.array_equal(g.col_indices, col)
    assert np.array_equal(g.weights, val)
    assert np.array_equal(g.degrees, deg)
    assert np.array_equal(s.planted, np.searchsorted(offs, orig, side="right") - 1)
    assert len(s.dropped) == n - orig.size


def test_weighted_device_csr_graph_equals_host_upload():
    """sc_graph_create_from_csr with device weights == the same graph uploaded from the host."""
    with DeviceCSR.dcsbm(300_000, 12, 1) as d:
        host = d.download()
        with DeviceGraph.from_device_csr(d) as dg1, DeviceGraph(host.graph) as dg2:
            dg1.sample_irwin_hall(2)
            dg2.sample_irwin_hall(2)
            a, fa = dg1.power_iterate(30)
            b, fb = dg2.power_iterate(30)
    assert np.array_equal(a, b) and np.array_equal(fa, fb)
