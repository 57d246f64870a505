"""Block power method (pm_log_k's embedding) against the reference's power_method on the
SignlessLaplacianOp with its own Gaussian start block (tests/golden/block.npz): every column
bit for bit, unit weights (config 1) and weighted with hub rows (wide-row kernel)."""

import os

import numpy as np
import pytest

from paper_2310_10939_b200 import DeviceGraph, SignlessLaplacianOp, from_csr
from paper_2310_10939_b200.spectral import sample_gaussian_vectors

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "block.npz"))


@pytest.mark.parametrize("name", ["c1", "wide"])
def test_block_power_method_bit_exact(name):
    G = {k[len(name) + 1:]: GOLD[k] for k in GOLD.files if k.startswith(name + "_")}
    g = from_csr(len(G["deg"]), G["rp"], G["col"], G["w"], G["deg"])
    x0 = sample_gaussian_vectors(g.n, G["x0"].shape[1], int(G["seed"])).data
    assert np.array_equal(x0, G["x0"])
    with DeviceGraph(g) as dg:
        raw, scaled = dg.power_iterate_block(x0, int(G["t"]))
        assert np.array_equal(raw, G["raw"])
        assert np.array_equal(scaled, G["scaled"])
        # the operator protocol routes blocks through the same kernel
        assert np.array_equal(SignlessLaplacianOp(dg).power(x0, int(G["t"])), G["raw"])
        raw0, _ = dg.power_iterate_block(x0, 0)
        assert np.array_equal(raw0, x0)


@pytest.mark.parametrize("case", ["c1", "sbm8"])
def test_pm_log_k_pipeline_against_reference(case):
    """The whole pm_log_k pipeline: the embedding handed to k-means is bit-identical to the
    reference's; the labels come from the d-dimensional device k-means (same seeding draws,
    same np.add.at means and einsum cost; distances in our order instead of BLAS's), which
    must reproduce the reference's partition on these instances."""
    from oracle import oracle as O
    from paper_2310_10939_b200 import SpectralParams, fast_spectral_cluster

    if case == "c1":
        g = from_csr(len(GOLD["c1_deg"]), GOLD["c1_rp"], GOLD["c1_col"], None, GOLD["c1_deg"])
        k, seed = 5, 0
    else:
        g = from_csr(len(GOLD["sbm8_deg"]), GOLD["sbm8_rp"], GOLD["sbm8_col"], None,
                     GOLD["sbm8_deg"])
        k, seed = 8, 2
    res = fast_spectral_cluster(g, SpectralParams(k=k, seed=seed, mode="pm_log_k"))
    assert np.array_equal(res.embedding.data, GOLD[f"{case}_pipeline_embedding"
                                                   if case == "c1" else "sbm8_embedding"])
    ref = GOLD["c1_pipeline_labels" if case == "c1" else "sbm8_labels"]
    assert np.array_equal(O.canonical_labels(res.partition.labels), O.canonical_labels(ref))
