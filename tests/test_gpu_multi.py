"""Multi-GPU handle in one process (sc_graph_create_multi; SURVEY.md §8(b)'s n_gpus and §8(e)):
row blocks balanced by entries, per-shard SELL / column-panel layouts, z mirrored into every
peer's copy by the SpMV epilogue, shards ordered by stream events.  gpurun gives one GPU, so
the shards share it (``devices=[0, 0, ...]``: the same code path, peer pointers on one device;
no shard ever spins on another, so this is a valid stand-in).  Bar: x0, x_T, f and labels
bit-identical to the single-GPU handle and the oracle (rows are never split and keep their
stored order).  Reference entry point: pipeline.py:127 (one call, unchanged signature)."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_10939_b200 import (DeviceGraph, KMeans1D, SpectralParams, fast_spectral_cluster,
                                   from_csr)
from paper_2310_10939_b200.errors import InputError, SpeclusterError
from paper_2310_10939_b200.generate import config_sbm, sample_dcsbm, sample_sbm

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1():
    return sample_sbm(config_sbm(1)).graph


@pytest.fixture(scope="module")
def c2():
    return sample_sbm(config_sbm(2)).graph


@pytest.fixture(scope="module")
def heavy():
    # DC-SBM shape: weighted, heavy-tailed degrees (rows > 256 entries take the wide kernel)
    return sample_dcsbm(200_000, 8, 5).graph


def _run(g, T, seed=0, sign=1.0, sym=False, **kw):
    with DeviceGraph(g, **kw) as dg:
        x0 = dg.sample_irwin_hall(seed, return_host=True)
        xT, f = dg.power_iterate(T, sign=sign, sym=sym)
        info = dg.info()
        lay = dg.shard_layout()
    return x0, xT, f, info, lay


@pytest.mark.parametrize("shards", [2, 3, 5])
def test_c1_shards_bit_exact(c1, shards):
    x0, xT, f, info, lay = _run(c1, 50, devices=[0] * shards)
    assert info["n_gpus"] == shards and len(lay) == shards
    xo0 = O.irwin_hall(c1.degrees, 0)
    xo, fo = O.power_iterate(c1.row_offsets, c1.col_indices, None, c1.degrees, xo0, 50)
    assert np.array_equal(x0, xo0)
    assert np.array_equal(xT, xo) and np.array_equal(f, fo)
    # contiguous row blocks covering [0, n), z blocks 8192-aligned
    assert lay[0][0] == 0 and sum(r for _, r, _, _ in lay) == c1.n
    for (r0, nr, zo, _), (r1, _, z1, _) in zip(lay, lay[1:]):
        assert r1 == r0 + nr and z1 % 8192 == 0 and z1 >= zo + nr


@pytest.mark.parametrize("variant", [dict(sign=-1.0), dict(sym=True), dict(T=0), dict(T=1)])
def test_c1_variants(c1, variant):
    T = variant.pop("T", 17)
    _, xs, fs, _, _ = _run(c1, T, **variant)
    _, xm, fm, _, _ = _run(c1, T, devices=[0, 0, 0], **variant)
    assert np.array_equal(xs, xm) and np.array_equal(fs, fm)


def test_c2_four_shards_with_panels(c2):
    _, xs, fs, si, _ = _run(c2, 100, panels=True)
    _, xm, fm, mi, lay = _run(c2, 100, panels=True, devices=[0, 0, 0, 0])
    assert si["panel_groups"] > 0 and mi["panel_groups"] > 0, "panel layout expected on shards"
    assert np.array_equal(xs, xm) and np.array_equal(fs, fm)
    # nnz balance of the row blocks
    rp = c2.row_offsets
    loads = [rp[r0 + nr] - rp[r0] for r0, nr, _, _ in lay]
    assert max(loads) - min(loads) <= 2 * int(np.diff(rp).max())


def test_weighted_wide_rows_shards(heavy):
    _, xs, fs, si, _ = _run(heavy, 40)
    _, xm, fm, mi, _ = _run(heavy, 40, devices=[0, 0, 0])
    assert si["long_rows"] > 0 and mi["long_rows"] > 0
    assert np.array_equal(xs, xm) and np.array_equal(fs, fm)


def test_caller_x0_and_rerun(c1):
    x0 = np.random.default_rng(4).random(c1.n)
    with DeviceGraph(c1, devices=[0, 0]) as dg:
        dg.set_x0(x0)
        a, fa = dg.power_iterate(9)
        b, fb = dg.power_iterate(9)  # reruns start again from x0
    xo, fo = O.power_iterate(c1.row_offsets, c1.col_indices, None, c1.degrees, x0, 9)
    assert np.array_equal(a, xo) and np.array_equal(b, xo) and np.array_equal(fb, fo)


def test_pipeline_multi_equals_single(c2):
    p1 = SpectralParams(k=10, t=100, mode="one_vector", seed=0)
    pm = SpectralParams(k=10, t=100, mode="one_vector", seed=0, devices=(0, 0, 0))
    r1 = fast_spectral_cluster(c2, p1)
    rm = fast_spectral_cluster(c2, pm)
    assert np.array_equal(r1.embedding.data, rm.embedding.data)
    assert np.array_equal(r1.partition.labels, rm.partition.labels)
    assert set(rm.timings) == {"embed", "scale", "kmeans", "total"}


def test_kmeans_from_multi_handle(c1):
    with DeviceGraph(c1, devices=[0, 0]) as dg:
        dg.sample_irwin_hall(0)
        _, f = dg.power_iterate(50)
        with KMeans1D(graph=dg) as km:
            part = km.lloyd(5, O.kmeans_seed(0))
    lab, _ = O.lloyd(f, 5, O.kmeans_seed(0))
    assert np.array_equal(part.labels, lab)


def test_multi_refusals(c1):
    with pytest.raises(InputError):
        DeviceGraph(c1, devices=[0, 0], reorder="bfs")
    with pytest.raises(InputError):
        DeviceGraph(c1, devices=[0, 99])
    with DeviceGraph(c1, devices=[0, 0]) as dg:
        with pytest.raises(SpeclusterError):
            dg.power_iterate(3)  # no start vector yet
        dg.sample_irwin_hall(0)
        with pytest.raises(SpeclusterError):
            dg.power_iterate_block(np.ones((c1.n, 2)), 2)  # single-GPU only


def test_bad_column_rejected_before_upload():
    rp = np.array([0, 1, 2], dtype=np.int64)
    col = np.array([1, 7], dtype=np.int32)
    g = from_csr(2, rp, col, None, np.array([1.0, 1.0]))
    with pytest.raises(InputError):
        DeviceGraph(g, devices=[0, 0])


def test_fp32_values_shards_equal_single(heavy):
    """the optional fp32-value variant on shards: the same fp32 weights and fp64 sums as the
    single handle, so the results are identical to it (and within 1e-5 of the fp64 oracle)"""
    _, xs, fs, _, _ = _run(heavy, 25, fp32_values=True)
    _, xm, fm, _, _ = _run(heavy, 25, fp32_values=True, devices=[0, 0, 0])
    assert np.array_equal(xs, xm) and np.array_equal(fs, fm)
    _, x64, _, _, _ = _run(heavy, 25)
    assert np.max(np.abs(xm - x64) / np.abs(x64)) < 1e-5
