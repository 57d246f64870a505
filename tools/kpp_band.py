"""k-means++ on a narrow band of 1-D points (the shape of the embeddings: x = 0.5 + 1e-9 N(0,1))
-- for launch lists / phase profiles of the seeding.  Usage: kpp_band.py [n] [k] [scale]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2310_10939_b200 import KMeans1D  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**6
k = int(sys.argv[2]) if len(sys.argv) > 2 else 100
sc = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-9
x = 0.5 + sc * np.random.default_rng(0).standard_normal(n)
with KMeans1D(x) as km:
    t = time.perf_counter()
    km.seed_centers(k, 3, 10)
    print(f"n={n} k={k} scale={sc}: {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)

if len(sys.argv) > 4 and sys.argv[4] == "check":
    # the oracle's own k-means++ (oracle/sc_oracle.c orc_kmeanspp + host draws) per restart
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_2310_10939_b200.generate import rng_for

    with KMeans1D(x) as km:
        ch = km.seed_centers(k, 3, 10)
    ok = all(np.array_equal(ch[r], O.kmeanspp_indices(x, k, rng_for(3, r))) for r in range(10))
    print(f"oracle check n={n} k={k} scale={sc}: identical={ok}", flush=True)
