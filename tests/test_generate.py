"""Input generators restated from the reference reproduce its graphs bit for bit."""

import hashlib
import json
import os

import numpy as np

from paper_2310_10939_b200 import from_edges
from paper_2310_10939_b200.generate import (config_sbm, sample_dcsbm, sample_sbm,
                                            sample_weighted_rgg)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def graph_hash(g, weighted=False):
    h = hashlib.sha256()
    h.update(np.asarray(g.row_offsets, dtype=np.int64).tobytes())
    h.update(np.asarray(g.col_indices, dtype=np.int32).tobytes())
    h.update(np.asarray(g.degrees, dtype=np.float64).tobytes())
    if weighted:
        h.update(np.asarray(g.weights, dtype=np.float64).tobytes())
    return h.hexdigest()


def meta():
    with open(os.path.join(GOLD, "golden.json")) as fh:
        return json.load(fh)


def test_sbm_config1_matches_reference():
    s = sample_sbm(config_sbm(1))
    assert graph_hash(s.graph) == meta()["configs"]["c1"]["graph_sha"]
    c1 = np.load(os.path.join(GOLD, "c1.npz"))
    assert np.array_equal(s.planted, c1["planted"])


def test_weighted_from_edges_matches_reference():
    # same construction as make_golden.py, built with this package's from_edges
    rng = np.random.default_rng(20231019)
    n, m = 2000, 24000
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    blk = u // (n // 4)
    inside = rng.random(m) < 0.8
    v = np.where(inside, blk * (n // 4) + (v % (n // 4)), v)
    keep = u != v
    w = 0.5 + rng.random(m)
    g, dropped = from_edges(n, u[keep], v[keep], w[keep], drop_isolated=True)
    ref = meta()["configs"]["weighted"]
    assert len(dropped) == ref["dropped"]
    gold = np.load(os.path.join(GOLD, "weighted.npz"))
    assert np.array_equal(g.row_offsets, gold["rp"]) and np.array_equal(g.col_indices, gold["col"])
    assert np.array_equal(g.degrees, gold["deg"])
    # Duplicate edges are summed; scipy sums a run of >= 3 duplicates in the order its
    # unstable std::sort leaves them (csr_sort_indices), we in input order: such sums may
    # differ in the last bit.  Every other stored weight is identical.
    diff = np.flatnonzero(g.weights != gold["w"])
    assert diff.size <= 4
    assert np.allclose(g.weights[diff], gold["w"][diff], rtol=4e-16, atol=0)


def test_dcsbm_shape():
    s = sample_dcsbm(20000, 8, seed=1)
    g = s.graph
    g.validate()
    assert g.weights is not None and g.weights.min() >= 0.5  # multi-edges are summed
    assert np.any(g.degrees != np.floor(g.degrees))
    assert s.planted.size == g.n


def test_rgg_shape():
    s = sample_weighted_rgg(5000, 10, seed=2)
    g = s.graph
    g.validate()
    assert g.nnz >= 16 * g.n  # union of 16-NN lists, symmetrised
    assert np.all(g.weights > 0) and np.all(g.weights <= 1.0)


def test_device_sbm_law_restatement_statistics():
    """The numpy restatement of the device generator's law (oracle.device_sbm): edge
    densities inside / across blocks match p / q within 5 sigma; symmetric CSR."""
    from oracle import oracle as O

    n, k, p, q = 3000, 3, 0.01, 0.001
    rp, col, deg, orig = O.device_sbm(n, k, p, q, 11)
    row = np.repeat(np.arange(orig.size), np.diff(rp))
    blk_r, blk_c = orig[row] // (n // k), orig[col] // (n // k)
    s = n // k
    e_in = np.sum(blk_r == blk_c) / 2
    e_out = np.sum(blk_r != blk_c) / 2
    t_in, t_out = k * s * (s - 1) / 2, s * s * k * (k - 1) / 2
    assert abs(e_in - p * t_in) < 5 * np.sqrt(p * t_in)
    assert abs(e_out - q * t_out) < 5 * np.sqrt(q * t_out)
    assert np.array_equal(np.sort(row * n + col), np.sort(col.astype(np.int64) * n + row))
    assert np.array_equal(deg, np.diff(rp))


def test_restated_weighted_generator_laws_are_symmetric_graphs():
    """oracle.device_knn3d / device_dcsbm (the laws of sc_generate_wt.cu): symmetric, sorted
    rows without self loops, every kNN row holds at least 16 neighbours, degrees are the
    rows' left-to-right weight sums, and sc_exp tracks exp to a few ulps."""
    import functools
    import operator

    from oracle import oracle as O
    from paper_2310_10939_b200.generate import dcsbm_block_offsets, dcsbm_power_law

    y = np.linspace(-50.0, 8.0, 2001)
    assert np.max(np.abs(O.np_sc_exp(y) / np.exp(y) - 1.0)) < 4e-16
    rp, col, val, deg, orig, pts, lab = O.device_knn3d(400, 4, 0.05, 16, 0.01, 1)
    offs = dcsbm_block_offsets(500, 5, 3)
    A, B, inv_a = dcsbm_power_law()
    graphs = [(rp, col, val, deg), O.device_dcsbm(500, offs, A, B, inv_a, 5, 5000, 0.1, 0.5, 1.5, 3)[:4]]
    assert np.all(np.diff(rp) >= 16)
    for rp_, col_, val_, deg_ in graphs:
        n = rp_.size - 1
        row = np.repeat(np.arange(n), np.diff(rp_))
        assert np.all(col_ != row)
        assert np.all((np.diff(col_) > 0) | (np.diff(row) != 0))
        key, tkey = row * n + col_, col_.astype(np.int64) * n + row
        o1, o2 = np.argsort(key), np.argsort(tkey)
        assert np.array_equal(key[o1], tkey[o2]) and np.array_equal(val_[o1], val_[o2])
        # (functools.reduce: Python's sum() compensates float rounding since 3.12)
        ref = np.array([functools.reduce(operator.add, val_[rp_[i]:rp_[i + 1]].tolist(), 0.0)
                        for i in range(n)])
        assert np.array_equal(deg_, ref)
