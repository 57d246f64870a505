"""Freeze the reference's Algorithm-2 embedding (pm_log_k, pipeline.py:144-147) for the
block power method: run in the build container (reads /root/reference), writes
tests/golden/block.npz.

Cases: config 1 (sample_sbm) with l = ceil(log2 5) = 3 Gaussian columns and the default
t; a weighted graph from the reference's from_edges with two hub rows longer than the
device's 256-entry slice limit (wide-row kernel) and l = 7."""

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from specluster.generate import SbmParams, sample_sbm  # noqa: E402
from specluster.graph import from_edges  # noqa: E402
from specluster.pipeline import SpectralParams  # noqa: E402
from specluster.spectral import (SignlessLaplacianOp, power_method,  # noqa: E402
                                 sample_gaussian_vectors)


def run(g, k, seed, out, name, l=None):
    params = SpectralParams(k=k, seed=seed, l=l)
    cols, t = params.num_columns(g.n), params.num_steps(g.n)
    x0 = sample_gaussian_vectors(g.n, cols, seed).data
    op = SignlessLaplacianOp(g)
    raw = power_method(op, x0, t)
    out.update({f"{name}_rp": g.row_offsets, f"{name}_col": g.col_indices,
                f"{name}_w": g.weights, f"{name}_deg": g.degrees, f"{name}_x0": x0,
                f"{name}_raw": raw, f"{name}_scaled": raw * op.inv_sqrt_degrees[:, None],
                f"{name}_t": np.int64(t), f"{name}_k": np.int64(k), f"{name}_seed": np.int64(seed)})


def main():
    out = {}
    s = sample_sbm(SbmParams(n=1000, k=5, p=0.3, q=0.01, seed=0))
    run(s.graph, 5, 0, out, "c1")
    rng = np.random.default_rng(9)
    n, m = 4000, 30000
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    u = np.concatenate([u, np.zeros(900, int), np.full(700, 17)])
    v = np.concatenate([v, rng.integers(1, n, 900), rng.integers(18, n, 700)])
    keep = u != v
    g, _ = from_edges(n, u[keep], v[keep], 0.25 + rng.random(keep.sum()), drop_isolated=True)
    assert np.diff(g.row_offsets).max() > 256
    run(g, 100, 3, out, "wide", l=7)
    # the reference's whole pm_log_k pipeline (labels through its BLAS-based k-means)
    from specluster.pipeline import fast_spectral_cluster
    r = fast_spectral_cluster(s.graph, SpectralParams(k=5, seed=0))
    out["c1_pipeline_labels"] = r.partition.labels
    out["c1_pipeline_embedding"] = r.embedding.data
    s2 = sample_sbm(SbmParams(n=20000, k=8, p=0.01, q=0.0005, seed=2))
    r2 = fast_spectral_cluster(s2.graph, SpectralParams(k=8, seed=2))
    out.update({"sbm8_rp": s2.graph.row_offsets, "sbm8_col": s2.graph.col_indices,
                "sbm8_deg": s2.graph.degrees, "sbm8_labels": r2.partition.labels,
                "sbm8_embedding": r2.embedding.data})
    np.savez_compressed(os.path.join(HERE, "block.npz"), **out)
    print({k: out[k].shape for k in out if k.endswith("_raw")}, int(out["c1_t"]))


if __name__ == "__main__":
    main()
