"""Configs 3-5 of BASELINE.json (shapes the reference cannot generate): bit-exact against
the C oracle at reduced sizes, size-independent properties at full size (config 3)."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_10939_b200 import DeviceGraph, KMeans1D, SpectralParams, fast_spectral_cluster
from paper_2310_10939_b200.generate import (SbmParams, sample_dcsbm, sample_sbm,
                                            sample_weighted_rgg)

pytestmark = pytest.mark.gpu


def _exact_power(g, T, seed=0, threads=8):
    x0 = O.irwin_hall(g.degrees, seed, threads=threads)
    with DeviceGraph(g) as dg:
        x0d = dg.sample_irwin_hall(seed, return_host=True)
        xT, f = dg.power_iterate(T)
        info = dg.info()
    assert np.array_equal(x0d, x0)
    xo, fo = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0, T,
                             threads=threads)
    assert np.array_equal(xT, xo)
    assert np.array_equal(f, fo)
    return f, info


def test_config3_shape_dcsbm_bit_exact():
    """Degree-corrected SBM (power-law degrees up to ~5000, weights U(0.5,1.5), Dirichlet
    blocks) at n = 300k: wide rows, non-integer degrees, T = 200 as in config 3."""
    g = sample_dcsbm(300_000, 50, seed=1).graph
    f, info = _exact_power(g, 200, seed=1)
    assert info["long_rows"] > 0 and not info["unit_weights"]
    part = fast_spectral_cluster(g, SpectralParams(k=50, t=200, mode="one_vector", seed=1,
                                                   restarts=2)).partition
    lab, _ = O.lloyd(f, 50, O.kmeans_seed(1), restarts=2)
    assert np.array_equal(part.labels, lab)


def test_config4_shape_rgg_bit_exact():
    """Weighted random geometric cluster graph (16-NN union, exp(-d^2/0.01) weights) at
    n = 200k, T = 300 as in config 4."""
    g = sample_weighted_rgg(200_000, 100, seed=2).graph
    f, _ = _exact_power(g, 300)
    with KMeans1D(f) as km:
        part = km.lloyd(100, O.kmeans_seed(2), restarts=2)
    lab, _ = O.lloyd(f, 100, O.kmeans_seed(2), restarts=2)
    assert np.array_equal(part.labels, lab)


def test_config5_shape_sbm_bit_exact():
    """Config 5's SBM law (blocks of 1e5, expected degree 16 in / 2 out), 5 blocks."""
    n = 500_000
    p = SbmParams(n=n, k=5, p=16 / (10**5 - 1), q=2 / (n - 10**5), seed=5)
    g = sample_sbm(p).graph
    _exact_power(g, 100)


def test_config3_full_size_properties():
    """Config 3 at full size (n = 4e6): the lazy walk conserves mass (1^T M = 1^T), keeps
    x nonnegative, f = x_T / d exactly, and two runs are bitwise identical."""
    g = sample_dcsbm(4_000_000, 50, seed=0).graph
    with DeviceGraph(g) as dg:
        x0 = dg.sample_irwin_hall(0, return_host=True)
        a, fa = dg.power_iterate(200)
        b, fb = dg.power_iterate(200)
    assert np.array_equal(a, b) and np.array_equal(fa, fb)
    assert np.all(a >= 0)
    assert abs(a.sum() - x0.sum()) <= 1e-9 * x0.sum()
    assert np.array_equal(fa, a / g.degrees)
    # Irwin-Hall moments: E x0 = deg/2, Var = (floor(deg) + frac(deg)^2) / 12
    fl = np.floor(g.degrees)
    z = (x0 - g.degrees / 2) / np.sqrt((fl + (g.degrees - fl) ** 2) / 12)
    assert abs(z.mean()) < 0.01 and abs(z.var() - 1) < 0.02


def test_config5_full_size_properties():
    """Maximum size: config 5 (n = 1e8, ~1.8e9 stored entries) generated on
    the device and iterated T = 100 times; size-independent checks on the whole vectors:
    mass conservation, non-negativity, f = x_T / d exactly, bitwise-identical reruns."""
    from paper_2310_10939_b200.generate import DeviceCSR, config_sbm

    with DeviceCSR(config_sbm(5)) as d:
        assert d.nnz > 1_700_000_000 and d.n == 10**8
        deg = np.empty(d.n)
        from paper_2310_10939_b200 import _lib
        _lib.check(_lib.load().sc_csr_download(d.handle, None, None, _lib.ptr(deg), None))
        dg = DeviceGraph.from_device_csr(d)
    with dg:
        x0 = dg.sample_irwin_hall(0, return_host=True)
        a, fa = dg.power_iterate(100)
        b, fb = dg.power_iterate(100)
    assert np.array_equal(a, b) and np.array_equal(fa, fb)
    assert np.all(a >= 0)
    assert abs(a.sum() - x0.sum()) <= 1e-9 * x0.sum()
    assert np.array_equal(fa, a / deg)
