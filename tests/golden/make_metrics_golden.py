"""Freeze golden values of the reference's evaluation metrics (run in the build container,
where /root/reference exists; tests read only the committed output):

    python tests/golden/make_metrics_golden.py   # writes tests/golden/metrics.npz

Cases: (1) config 1 (reference sample_sbm) with its planted labels vs a perturbed labelling
(unit weights); (2) a weighted graph from the reference's from_edges with non-integer
weights and random labels, predicted k != truth k (padded matching); (3) 2-part
partitions of a weighted ring (near-equal volumes).  For each: ari, nmi, per-part
conductances, matched symmetric-difference volume and permutation, bit for bit."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from specluster.generate import SbmParams, sample_sbm  # noqa: E402
from specluster.graph import from_edges  # noqa: E402
from specluster.metrics import (ari, matched_sym_diff_volume, nmi,  # noqa: E402
                                partition_conductances)


def case(name, g, pred, truth, out):
    out[f"{name}_rp"] = g.row_offsets
    out[f"{name}_col"] = g.col_indices
    out[f"{name}_w"] = g.weights
    out[f"{name}_deg"] = g.degrees
    out[f"{name}_pred"] = pred
    out[f"{name}_truth"] = truth
    out[f"{name}_ari"] = np.float64(ari(pred, truth))
    out[f"{name}_nmi"] = np.float64(nmi(pred, truth))
    out[f"{name}_cond"] = partition_conductances(g, pred)
    v, perm = matched_sym_diff_volume(g, pred, truth)
    out[f"{name}_msdv"] = np.float64(v)
    out[f"{name}_perm"] = perm


def main():
    out = {}
    s = sample_sbm(SbmParams(n=1000, k=5, p=0.3, q=0.01, seed=0))
    truth = s.planted.labels.astype(np.int64)
    rng = np.random.default_rng(1)
    pred = truth.copy()
    flip = rng.random(pred.size) < 0.1
    pred[flip] = rng.integers(0, 5, flip.sum())
    case("sbm", s.graph, pred, truth, out)

    rng = np.random.default_rng(2)
    n, m = 3000, 40000
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    keep = u != v
    g, _ = from_edges(n, u[keep], v[keep], 0.1 + rng.random(keep.sum()) * 3.7,
                      drop_isolated=True)
    pred = rng.integers(0, 7, g.n)
    truth = rng.integers(0, 5, g.n)
    case("weighted", g, pred, truth, out)

    n = 2000
    u = np.arange(n)
    g, _ = from_edges(n, u, (u + 1) % n, 1.0 / (1.0 + (u % 13)))
    truth = (u >= n // 2).astype(np.int64)
    pred = ((u + 37) % n >= n // 2).astype(np.int64)
    case("ring", g, pred, truth, out)
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **out)
    print({k: out[k] for k in out if k.endswith(("_ari", "_nmi", "_msdv"))})


if __name__ == "__main__":
    main()
