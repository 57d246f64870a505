"""Where the end-to-end cluster time goes at config 2 (upload, x0, power, f, k-means)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2310_10939_b200 import DeviceGraph, KMeans1D  # noqa: E402
from paper_2310_10939_b200.generate import config_sbm, sample_sbm  # noqa: E402
from paper_2310_10939_b200.pipeline import _kmeans_seed  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g = sample_sbm(config_sbm(cfg)).graph
T, k = (100, 10) if cfg == 2 else (50, 5)
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    t0 = time.perf_counter()
    dg = DeviceGraph(g)
    t1 = time.perf_counter()
    dg.sample_irwin_hall(0)
    t2 = time.perf_counter()
    _, f = dg.power_iterate(T, want_x=False)
    t3 = time.perf_counter()
    km = KMeans1D(graph=dg)
    t4 = time.perf_counter()
    ch = km.seed_centers(k, _kmeans_seed(0), 10)
    t5 = time.perf_counter()
    part = km.lloyd(k, _kmeans_seed(0))
    t6 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f}  x0 {1e3*(t2-t1):.1f}  power {1e3*(t3-t2):.1f} (dev {dg.last_timing['power_ms']:.2f}) "
          f"km_ctx {1e3*(t4-t3):.1f}  kpp {1e3*(t5-t4):.1f}  lloyd(total incl kpp) {1e3*(t6-t5):.1f} "
          f"lloyd_dev {km.last['lloyd_ms']:.1f} iters {km.last['iters'].tolist()}", flush=True)
    km.close()
    dg.close()
