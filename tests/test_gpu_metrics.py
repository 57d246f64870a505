"""GPU evaluation metrics vs the reference's own values (tests/golden/metrics.npz, made by
tests/golden/make_metrics_golden.py from specluster.metrics): ARI, NMI, conductances and the
matched symmetric-difference volume, all bit for bit; np.add.at semantics of the device
keyed sums on adversarial values."""

import os

import numpy as np
import pytest

from paper_2310_10939_b200 import from_csr
from paper_2310_10939_b200 import metrics as M
from paper_2310_10939_b200.errors import InputError

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "metrics.npz"))


@pytest.mark.parametrize("name", ["sbm", "weighted", "ring"])
def test_metrics_match_reference_bit_for_bit(name):
    G = {k[len(name) + 1:]: GOLD[k] for k in GOLD.files if k.startswith(name + "_")}
    g = from_csr(len(G["deg"]), G["rp"], G["col"], G["w"], G["deg"])
    pred, truth = G["pred"], G["truth"]
    assert M.ari(pred, truth) == float(G["ari"])
    assert M.nmi(pred, truth) == float(G["nmi"])
    assert np.array_equal(M.partition_conductances(g, pred), G["cond"])
    v, perm = M.matched_sym_diff_volume(g, pred, truth)
    assert v == float(G["msdv"])
    assert np.array_equal(perm, G["perm"])
    rep = M.evaluate_partition(g, pred, truth)
    assert rep.max_conductance == float(G["cond"].max())


def test_keyed_sums_are_np_add_at():
    rng = np.random.default_rng(5)
    m, k = 200_000, 37
    keys = rng.integers(0, k, m)
    vals = np.exp(rng.uniform(-30, 30, m))  # 26 decades: every rounding matters
    vals[::17] = 1e-310                      # subnormals
    ref = np.zeros(k)
    np.add.at(ref, keys, vals)
    assert np.array_equal(M.keyed_sums(keys, vals, k), ref)
    with pytest.raises(InputError):
        M.keyed_sums(np.array([0, 5]), np.ones(2), 3)


def test_contingency_and_labels_validation():
    a = np.array([0, 1, 1, 2, 2, 2])
    b = np.array([1, 1, 0, 0, 0, 1])
    ct = M.ContingencyTable.from_labels(a, b)
    ref = np.zeros((3, 2), dtype=np.int64)
    np.add.at(ref, (a, b), 1)
    assert np.array_equal(ct.counts, ref)
    with pytest.raises(InputError):
        M.ContingencyTable.from_labels(a, np.array([0, 1, 2, 3, -1, 0]))
