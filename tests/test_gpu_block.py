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
