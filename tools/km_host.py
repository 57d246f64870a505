"""Host-side breakdown of KMeans1D.lloyd on the config-2 embedding (seeding vs the fused kernel)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2310_10939_b200 import DeviceGraph, KMeans1D  # noqa: E402
from paper_2310_10939_b200.generate import config_sbm, sample_sbm  # noqa: E402
from paper_2310_10939_b200.pipeline import _kmeans_seed  # noqa: E402

g = sample_sbm(config_sbm(2)).graph
dg = DeviceGraph(g)
dg.sample_irwin_hall(0)
dg.power_iterate(100, want_x=False)
for rep in range(4):
    t0 = time.perf_counter()
    km = KMeans1D(graph=dg)
    t1 = time.perf_counter()
    ch = km.seed_centers(10, _kmeans_seed(0), 10)
    t2 = time.perf_counter()
    part = km.lloyd(10, _kmeans_seed(0))
    t3 = time.perf_counter()
    km.close()
    t4 = time.perf_counter()
    print(f"ctx {1e3*(t1-t0):.2f}  seed {1e3*(t2-t1):.2f}  lloyd(incl seed) {1e3*(t3-t2):.2f} "
          f"(lib {km.last['lloyd_ms']:.2f})  close {1e3*(t4-t3):.2f} ms", flush=True)
