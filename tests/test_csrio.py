"""Binary CSR files: round trips (unit / weighted, mmap / read), corruption is rejected."""

import numpy as np
import pytest

from paper_2310_10939_b200 import from_edges
from paper_2310_10939_b200.csrio import load_csr, save_csr
from paper_2310_10939_b200.errors import GraphFormatError
from paper_2310_10939_b200.generate import SbmParams, sample_sbm


def _same(a, b):
    assert a.n == b.n
    assert np.array_equal(a.row_offsets, b.row_offsets)
    assert np.array_equal(a.col_indices, b.col_indices)
    assert (a.weights is None) == (b.weights is None)
    if a.weights is not None:
        assert np.array_equal(a.weights, b.weights)
    assert np.array_equal(a.degrees, b.degrees)  # verbatim, bit for bit


@pytest.mark.parametrize("mmap", [True, False])
def test_roundtrip_unit_and_weighted(tmp_path, mmap):
    g = sample_sbm(SbmParams(n=2000, k=4, p=0.05, q=0.005, seed=3)).graph
    save_csr(g, tmp_path / "u.sccsr")
    _same(g, load_csr(tmp_path / "u.sccsr", mmap=mmap))
    rng = np.random.default_rng(0)
    u, v = rng.integers(0, 500, 4000), rng.integers(0, 500, 4000)
    keep = u != v
    gw, _ = from_edges(500, u[keep], v[keep], rng.random(keep.sum()) + 0.25, drop_isolated=True)
    save_csr(gw, tmp_path / "w.sccsr")
    _same(gw, load_csr(tmp_path / "w.sccsr", mmap=mmap))


def test_corrupt_files_rejected(tmp_path):
    g = sample_sbm(SbmParams(n=400, k=2, p=0.1, q=0.01, seed=1)).graph
    p = tmp_path / "g.sccsr"
    save_csr(g, p)
    raw = p.read_bytes()
    (tmp_path / "short").write_bytes(raw[:100])
    with pytest.raises(GraphFormatError, match="truncated"):
        load_csr(tmp_path / "short")
    (tmp_path / "magic").write_bytes(b"NOTCSR!!" + raw[8:])
    with pytest.raises(GraphFormatError, match="magic"):
        load_csr(tmp_path / "magic")
    (tmp_path / "tiny").write_bytes(raw[:10])
    with pytest.raises(GraphFormatError):
        load_csr(tmp_path / "tiny")
