"""CLI end to end on the GPU: `cluster` on config 1 written as a reference edge list gives
the reference's labels (golden c1.npz), and repeated runs are byte-identical (labels,
embedding, report -- test_acceptance.py:317-340 of the reference); `evaluate` matches the
metrics module; the device generator writes a loadable binary CSR."""

import os

import numpy as np
import pytest

from paper_2310_10939_b200 import cli, from_csr
from paper_2310_10939_b200 import metrics as M
from paper_2310_10939_b200.csrio import load_csr
from paper_2310_10939_b200.textio import load_embedding, load_labels, save_edge_list, save_labels

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_cluster_config1_matches_reference_and_is_byte_deterministic(tmp_path):
    d = dict(np.load(os.path.join(GOLD, "c1.npz")))
    g = from_csr(len(d["deg"]), d["rp"], d["col"], None, d["deg"])
    save_edge_list(g, tmp_path / "g.tsv")
    outs = []
    for run in range(2):
        o = tmp_path / f"run{run}"
        assert cli.main(["cluster", "--graph", str(tmp_path / "g.tsv"), "--k", "5", "--t", "50",
                         "--mode", "one_vector",
                         "--seed", "0", "--out", str(o)]) == 0
        outs.append(o)
    lab = load_labels(outs[0] / "labels.txt", expected_n=g.n)
    assert np.array_equal(lab, d["labels"])
    emb, scaled, seed = load_embedding(outs[0] / "embedding.csv")
    assert scaled and seed == 0 and np.array_equal(emb[:, 0], d["f"])
    for name in ("labels.txt", "embedding.csv", "report.json"):
        assert (outs[0] / name).read_bytes() == (outs[1] / name).read_bytes()
    # evaluate against the planted partition (blocks of 200)
    save_labels(np.arange(g.n) // 200, tmp_path / "truth.txt")
    assert cli.main(["evaluate", "--graph", str(tmp_path / "g.tsv"), "--labels",
                     str(outs[0] / "labels.txt"), "--truth", str(tmp_path / "truth.txt"),
                     "--out", str(tmp_path / "ev")]) == 0
    import json
    rep = json.loads((tmp_path / "ev" / "report.json").read_text())
    assert rep["ari"] == M.ari(lab, np.arange(g.n) // 200)


def test_device_generator_cli_writes_binary_csr(tmp_path):
    assert cli.main(["generate-sbm", "--n", "20000", "--k", "4", "--p", "0.002", "--q", "0.0002",
                     "--device-generator", "--format", "sccsr", "--out", str(tmp_path)]) == 0
    g = load_csr(tmp_path / "graph.sccsr")
    assert g.n <= 20000 and g.nnz > 0 and np.all(g.degrees > 0)
    assert load_labels(tmp_path / "labels.txt", expected_n=g.n).max() == 3
