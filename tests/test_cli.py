"""CLI (host side, no GPU): generator outputs round-trip through the reference text formats,
input errors exit with code 2 as in the reference (cli.py:411-427)."""

import numpy as np
import pytest

from paper_2310_10939_b200 import cli
from paper_2310_10939_b200.csrio import load_csr
from paper_2310_10939_b200.generate import SbmParams, sample_sbm
from paper_2310_10939_b200.textio import load_edge_list, load_labels, save_embedding, load_embedding


@pytest.mark.parametrize("fmt", ["tsv", "sccsr"])
def test_generate_sbm_outputs_round_trip(tmp_path, fmt):
    rc = cli.main(["generate-sbm", "--n", "600", "--k", "3", "--p", "0.05", "--q", "0.005",
                   "--seed", "4", "--format", fmt, "--out", str(tmp_path)])
    assert rc == 0
    ref = sample_sbm(SbmParams(n=600, k=3, p=0.05, q=0.005, seed=4))
    g = (load_edge_list(tmp_path / "graph.tsv").graph if fmt == "tsv"
         else load_csr(tmp_path / "graph.sccsr"))
    assert np.array_equal(g.row_offsets, ref.graph.row_offsets)
    assert np.array_equal(g.col_indices, ref.graph.col_indices)
    assert np.array_equal(g.degrees, ref.graph.degrees)
    assert np.array_equal(load_labels(tmp_path / "labels.txt", expected_n=g.n), ref.planted)
    assert (tmp_path / "meta.json").exists() and (tmp_path / "meta.jsonl").exists()


def test_edge_list_tokens_weights_and_errors(tmp_path):
    p = tmp_path / "g.tsv"
    p.write_text("# comment\na\tb\t2.5\nb\tc\nc\ta\t0.5\n", encoding="utf-8")
    r = load_edge_list(p)
    assert r.id_map == ["a", "b", "c"] and r.graph.n == 3
    assert np.allclose(r.graph.degrees, [3.0, 3.5, 1.5])
    bad = tmp_path / "bad.tsv"
    bad.write_text("0\t1\t-1\n", encoding="utf-8")
    assert cli.main(["cluster", "--graph", str(bad), "--k", "2", "--out", str(tmp_path / "o")]) == 2
    assert cli.main(["cluster", "--graph", str(tmp_path / "missing.tsv"), "--k", "2",
                     "--out", str(tmp_path / "o")]) == 2
    assert cli.main(["bench-growk", "--kmax", "3", "--out", str(tmp_path / "b")]) == 2


def test_embedding_file_round_trip(tmp_path):
    x = np.random.default_rng(0).standard_normal(50) * 1e-7
    save_embedding(x, tmp_path / "e.csv", scaled=True, seed=3)
    d, scaled, seed = load_embedding(tmp_path / "e.csv")
    assert scaled and seed == 3 and np.array_equal(d[:, 0], x)
    assert cli.bench_grid("growk", 40) == [5, 10, 20, 40]
    assert cli.bench_grid("grown", 100_000) == [20_000, 40_000, 80_000]
