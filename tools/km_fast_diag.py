"""Exact replica vs sorted (fast) Lloyd on config 2: per-restart costs / iterations and
label differences."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2310_10939_b200 import DeviceGraph, KMeans1D  # noqa: E402
from paper_2310_10939_b200.generate import config_sbm, sample_sbm  # noqa: E402
from paper_2310_10939_b200.pipeline import _kmeans_seed  # noqa: E402

g = sample_sbm(config_sbm(2)).graph
with DeviceGraph(g) as dg:
    dg.sample_irwin_hall(0)
    _, f = dg.power_iterate(100, want_x=False)
with KMeans1D(f) as km:
    a = km.lloyd(10, _kmeans_seed(0))
    la = dict(km.last)
    b = km.lloyd(10, _kmeans_seed(0), method="sorted")
    lb = dict(km.last)
np.set_printoptions(precision=17)
print("exact  costs", la["costs"], "iters", la["iters"], "best", la["best_restart"])
print("sorted costs", lb["costs"], "iters", lb["iters"], "best", lb["best_restart"])
print("rel cost diff", (lb["costs"] - la["costs"]) / la["costs"])
print("labels differ:", int(np.sum(a.labels != b.labels)))
