"""Freeze golden vectors by running the REFERENCE package itself (run in the build
container, where /root/reference exists; the outputs are committed and are what the
tests read -- nothing at test time reads /root/reference).

    python tests/golden/make_golden.py            # writes tests/golden/*.npz + golden.json

What is frozen (SURVEY.md CS2 composed from reference functions only):
  * graphs: specluster.generate.sample_sbm (configs 1, 2) and specluster.graph.from_edges
    (a weighted graph with non-integer degrees);
  * x_T: specluster.spectral.power_method with the rw callable
    ``lambda x: 0.5*x + 0.5*(A @ (x/d))`` (and the '-' sign, and the reference's own
    SignlessLaplacianOp);
  * labels: specluster.kmeans.lloyd(PointSet(f[:, None]), k, seed=_kmeans_seed(seed));
  * k-means edge cases (duplicates -> degenerate k-means++ rounds, empty-cluster repair);
  * numpy Philox / einsum / cumsum known answers the restatements rely on.
The start vector x0 is the one-vector Irwin-Hall draw (no reference implementation
exists); it is produced by numpy's own Philox (oracle.np_irwin_hall) and cross-checked
against the C restatement before anything is frozen.
"""

from __future__ import annotations

import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import scipy  # noqa: E402
from specluster.generate import SbmParams, sample_sbm  # noqa: E402
from specluster.graph import from_edges  # noqa: E402
from specluster.kmeans import PointSet, lloyd  # noqa: E402
from specluster.pipeline import _kmeans_seed  # noqa: E402
from specluster.spectral import SignlessLaplacianOp, power_method  # noqa: E402

from oracle import oracle as O  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def graph_hash(rp, col, deg, w=None) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(rp, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(col, dtype=np.int32).tobytes())
    h.update(np.ascontiguousarray(deg, dtype=np.float64).tobytes())
    if w is not None:
        h.update(np.ascontiguousarray(w, dtype=np.float64).tobytes())
    return h.hexdigest()


def rw(A, d, sign=1.0):
    if sign > 0:
        return lambda x: 0.5 * x + 0.5 * (A @ (x / d))
    return lambda x: 0.5 * x - 0.5 * (A @ (x / d))


def run_path(g, T, k, seed, *, x0=None, sign=1.0, with_sym=False):
    d = g.degrees
    A = g.adjacency_csr()
    if x0 is None:
        x0 = O.np_irwin_hall(d, seed) if g.n <= 20000 else None
        x0c = O.irwin_hall(d, seed, threads=8)
        if x0 is not None:
            assert np.array_equal(x0, x0c), "numpy-Philox and C Irwin-Hall disagree"
        x0 = x0c
    t = time.perf_counter()
    xT = power_method(rw(A, d, sign), x0, T)
    t_pm = time.perf_counter() - t
    f = xT / d
    out = {"x0": x0, "xT": xT, "f": f}
    if k:
        t = time.perf_counter()
        out["labels"] = lloyd(PointSet(f[:, None]), k, seed=_kmeans_seed(seed)).labels
        out["t_lloyd"] = time.perf_counter() - t
    out["t_pm"] = t_pm
    if with_sym:
        out["xT_sym"] = power_method(SignlessLaplacianOp(g), x0, T)
    return out


def main():
    meta = {
        "generated_by": "tests/golden/make_golden.py",
        "reference": "/root/reference/pkg (specluster 0.1.0)",
        "python": platform.python_version(),
        "numpy": np.__version__,
        "scipy": scipy.__version__,
        "machine": platform.machine(),
        "configs": {},
    }

    # ---- config 1 (full arrays) ------------------------------------------------
    s1 = sample_sbm(SbmParams(n=1000, k=5, p=0.3, q=0.01, seed=0))
    g1 = s1.graph
    r1 = run_path(g1, 50, 5, 0, with_sym=True)
    r1m = run_path(g1, 10, 0, 0, x0=r1["x0"], sign=-1.0)
    np.savez_compressed(
        os.path.join(HERE, "c1.npz"), rp=g1.row_offsets, col=g1.col_indices.astype(np.int32),
        deg=g1.degrees, planted=s1.planted.labels, x0=r1["x0"], xT=r1["xT"], f=r1["f"],
        labels=r1["labels"], xT_sym=r1["xT_sym"], xT_minus10=r1m["xT"])
    meta["configs"]["c1"] = {
        "n": g1.n, "nnz": int(g1.col_indices.size), "T": 50, "k": 5, "seed": 0,
        "graph_sha": graph_hash(g1.row_offsets, g1.col_indices, g1.degrees),
        "sizes": np.bincount(r1["labels"], minlength=5).tolist(),
    }

    # ---- weighted graph, non-integer degrees ---------------------------------
    rng = np.random.default_rng(20231019)
    n = 2000
    m = 24000
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    keep = u != v
    # plant 4 communities: bias 80% of the edges to stay inside u's block
    blk = u // (n // 4)
    inside = rng.random(m) < 0.8
    v = np.where(inside, blk * (n // 4) + (v % (n // 4)), v)
    keep = u != v
    w = 0.5 + rng.random(m)
    gw, dropped = from_edges(n, u[keep], v[keep], w[keep], drop_isolated=True)
    rw_ = run_path(gw, 40, 4, 3)
    rwm = run_path(gw, 12, 0, 3, x0=rw_["x0"], sign=-1.0)
    np.savez_compressed(
        os.path.join(HERE, "weighted.npz"), rp=gw.row_offsets, col=gw.col_indices.astype(np.int32),
        w=gw.weights, deg=gw.degrees, x0=rw_["x0"], xT=rw_["xT"], f=rw_["f"],
        labels=rw_["labels"], xT_minus12=rwm["xT"])
    meta["configs"]["weighted"] = {
        "n": gw.n, "nnz": int(gw.col_indices.size), "T": 40, "k": 4, "seed": 3,
        "dropped": len(dropped),
        "graph_sha": graph_hash(gw.row_offsets, gw.col_indices, gw.degrees, gw.weights),
    }

    # ---- k-means edge cases (reference lloyd on 1-D point sets) ---------------
    cases = {}
    rng = np.random.default_rng(7)
    pts = {
        "dup3_k5": np.repeat([0.25, 0.5, 0.75], [40, 30, 30]).astype(np.float64),
        "dup2_k4": np.array([1.0] * 7 + [2.0] * 5),
        "tiny_k2": np.array([0.0, 1.0, 1.0, 3.0]),
        "equal_k3": np.full(9, 0.3),
        "blobs_k3": np.concatenate([rng.normal(0, 0.1, 60), rng.normal(5, 0.1, 50),
                                    rng.normal(10, 0.1, 40)]),
        "far_outlier_k6": np.concatenate([rng.random(200) * 1e-3, [1e3], rng.random(50) + 7.0]),
        "uniform_k10": rng.random(5000),
        "spread_k50": np.sort(rng.random(3000)) ** 3,
        "neg_k4": rng.normal(-2.0, 1.0, 800),
    }
    ks = {"dup3_k5": 5, "dup2_k4": 4, "tiny_k2": 2, "equal_k3": 3, "blobs_k3": 3,
          "far_outlier_k6": 6, "uniform_k10": 10, "spread_k50": 50, "neg_k4": 4}
    arrays = {}
    for name, x in pts.items():
        k = ks[name]
        for seed in (0, 11):
            lab = lloyd(PointSet(x[:, None]), k, seed=seed).labels
            arrays[f"{name}__x"] = x
            arrays[f"{name}__s{seed}"] = lab
            cases[f"{name}__s{seed}"] = {"k": k, "seed": seed}
    np.savez_compressed(os.path.join(HERE, "kmeans_cases.npz"), **arrays)
    meta["kmeans_cases"] = cases

    # ---- numpy known answers ------------------------------------------------
    ka = {}
    for key, ctr in [([7, 0], [0, 0, 0, 0]), ([123456789, 987654321], [5, 77, 0, 0]),
                     ([2**64 - 1, 3], [2**64 - 1, 41, 0, 0])]:
        bg = np.random.Philox(key=np.array(key, dtype=np.uint64),
                              counter=np.array(ctr, dtype=np.uint64))
        ka[f"philox_{key}_{ctr}"] = {
            "key": [str(v) for v in key], "counter": [str(v) for v in ctr],
            "raw8": [str(int(v)) for v in bg.random_raw(8)],
        }
    meta["philox_known_answers"] = ka
    rng = np.random.default_rng(99)
    es = {}
    for nn in (1, 7, 8, 9, 17, 8191, 8192, 8193, 20000, 100003):
        dd = (rng.random((nn, 1)) - 0.5) * 1e-4
        es[str(nn)] = {"seed": 99, "value": float(np.einsum("ij,ij->", dd, dd))}
    meta["einsum_known_answers_note"] = "default_rng(99), sizes drawn in this order, (rand-0.5)*1e-4"
    meta["einsum_known_answers"] = es
    meta["kmeans_seed_0"] = _kmeans_seed(0)

    # ---- config 2 (hashes only: the arrays are 0.5 GB) -----------------------
    if "--skip-c2" not in sys.argv:
        t = time.perf_counter()
        s2 = sample_sbm(SbmParams(n=10**6, k=10, p=40 / (10**5 - 1), q=4 / (9 * 10**5), seed=0))
        t_gen = time.perf_counter() - t
        g2 = s2.graph
        r2 = run_path(g2, 100, 10, 0)
        meta["configs"]["c2"] = {
            "n": g2.n, "nnz": int(g2.col_indices.size), "T": 100, "k": 10, "seed": 0,
            "graph_sha": graph_hash(g2.row_offsets, g2.col_indices, g2.degrees),
            "x0_sha": sha(r2["x0"]), "xT_sha": sha(r2["xT"]), "f_sha": sha(r2["f"]),
            "labels_canon_sha": sha(O.canonical_labels(r2["labels"])),
            "labels_sha": sha(r2["labels"].astype(np.int64)),
            "sizes": np.bincount(r2["labels"], minlength=10).tolist(),
            "xT_head": r2["xT"][:4].tolist(), "f_head": r2["f"][:4].tolist(),
            "xT_sum": float(r2["xT"].sum()), "x0_sum": float(r2["x0"].sum()),
            "ref_seconds": {"sample_sbm": t_gen, "power_method": r2["t_pm"],
                            "lloyd": r2["t_lloyd"]},
        }

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(json.dumps({k: v for k, v in meta["configs"].items()}, indent=1)[:2000])


if __name__ == "__main__":
    main()
