"""Randomised soak of the certified fast k-means++ draw: seeds with the fast path (default and
with its margin widened) against the exact pipeline (SC_KPP_NOFAST) on random inputs.
Usage: kpp_fast_soak.py [trials] [n_lo] [n_hi]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2310_10939_b200 import KMeans1D  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 24
n_lo = int(float(sys.argv[2])) if len(sys.argv) > 2 else 5_000
n_hi = int(float(sys.argv[3])) if len(sys.argv) > 3 else 3_000_000
rng = np.random.default_rng(2024)
bad = 0
for t in range(trials):
    n = int(rng.integers(n_lo, n_hi))
    kind = t % 6
    if kind == 0:
        x = 0.5 + 10.0 ** rng.integers(-12, -3) * rng.standard_normal(n)
    elif kind == 1:
        x = rng.random(n)
    elif kind == 2:
        x = np.repeat(rng.random(max(2, n // 1000)), 1000)[:n]
    elif kind == 3:
        x = -rng.random(n) ** 4 - 1e-3
    elif kind == 4:
        x = np.round(rng.random(n), 3)  # many exact duplicates -> zero weights, degenerate rounds
    else:
        x = np.concatenate([rng.normal(c, 1e-4, n // 8 + 1) for c in rng.random(8)])[:n]
    n = x.size
    k = int(rng.integers(2, 65))
    R = int(rng.integers(1, 17))
    seed = int(rng.integers(0, 2**31))
    out = {}
    for mode, env in (("exact", {"SC_KPP_NOFAST": "1"}), ("fast", {}), ("mixed", {"SC_KPP_EPS_SCALE": "3e4"})):
        for kk in ("SC_KPP_NOFAST", "SC_KPP_EPS_SCALE"):
            os.environ.pop(kk, None)
        os.environ.update(env)
        with KMeans1D(x) as km:
            out[mode] = km.seed_centers(k, seed, R)
    ok = np.array_equal(out["exact"], out["fast"]) and np.array_equal(out["exact"], out["mixed"])
    bad += not ok
    print(f"trial {t}: n={n} k={k} R={R} kind={kind} {'ok' if ok else 'MISMATCH'}", flush=True)
print("mismatches:", bad)
sys.exit(1 if bad else 0)
