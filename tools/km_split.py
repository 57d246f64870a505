"""Exact k-means phase split at a config: k-means++ seeding (sc_kmeans_pp rounds, host PCG64
replay included) vs Lloyd (sc_kmeans_lloyd), warm, on the device-resident embedding of the
config's graph.  Usage: python tools/km_split.py CFG [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_10939_b200 import DeviceGraph, KMeans1D  # noqa: E402
from paper_2310_10939_b200.generate import (CONFIG_K, CONFIG_T, config_device_csr,  # noqa: E402
                                            config_sbm, sample_sbm)
from paper_2310_10939_b200.pipeline import _kmeans_seed  # noqa: E402

cfg = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
T, k = CONFIG_T[cfg], CONFIG_K[cfg]
if cfg in (1, 2):
    dg = DeviceGraph(sample_sbm(config_sbm(cfg)).graph)
else:
    with config_device_csr(cfg) as d:
        dg = DeviceGraph.from_device_csr(d)
dg.sample_irwin_hall(0)
dg.power_iterate(T, want_x=False, want_f=False)
seed = _kmeans_seed(0)
for rep in range(reps):
    t0 = time.perf_counter()
    km = KMeans1D(graph=dg)
    t1 = time.perf_counter()
    km.seed_centers(k, seed, 10)
    t2 = time.perf_counter()
    km.lloyd(k, seed, assert_cost=False)
    t3 = time.perf_counter()
    print(f"cfg {cfg} n={dg.n} k={k} rep {rep}: ctx {1e3 * (t1 - t0):.1f} ms, k-means++ "
          f"{1e3 * (t2 - t1):.1f} ms, lloyd() total {1e3 * (t3 - t2):.1f} ms (device Lloyd "
          f"{km.last['lloyd_ms']:.1f} ms), iters {km.last['iters'].tolist()}", flush=True)
    km.close()
