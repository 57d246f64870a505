"""Compare GPU k-means++ picks / per-restart Lloyd costs with the oracle on one input."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2310_10939_b200 import KMeans1D  # noqa: E402

rng = np.random.default_rng(5)
case = sys.argv[1] if len(sys.argv) > 1 else "wide_range"
if case == "wide_range":
    x, k = np.exp(rng.normal(0, 12, 20000)), 9
elif case == "tiny_subnormal":
    x, k = rng.random(5000) * 1e-300, 4
else:
    x, k = rng.random(300000) * 1e-3 + 0.5, 20
seed, R = 77, 10
with KMeans1D(x) as km:
    ch = km.seed_centers(k, seed, R)
    part = km.lloyd(k, seed, restarts=R)
    costs = km.last["costs"]
for r in range(R):
    co = O.kmeanspp_indices(x, k, O.rng_for(seed, r))
    lab = np.empty(x.size, dtype=np.int64)
    c = ctypes.c_double()
    it = O.lib().orc_lloyd_restart(x.size, O._p(x), k, O._p(x[co].copy()), 100, 1e-6, O._p(lab),
                                   ctypes.byref(c))
    same = np.array_equal(co, ch[r])
    print(r, "kpp_same", same, "" if same else (co.tolist(), ch[r].tolist()),
          "cost", costs[r], c.value, costs[r] == c.value, "iters_o", it)
