import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2310_10939_b200 import DeviceGraph, KMeans1D
from paper_2310_10939_b200.generate import config_sbm, sample_sbm
from paper_2310_10939_b200.pipeline import _kmeans_seed
g = sample_sbm(config_sbm(2)).graph
dg = DeviceGraph(g); dg.sample_irwin_hall(0); dg.power_iterate(100, want_x=False)
for rep in range(4):
    km = KMeans1D(graph=dg)
    t0 = time.perf_counter(); ch = km.seed_centers(10, _kmeans_seed(0), 10); t1 = time.perf_counter()
    part = km.lloyd(10, _kmeans_seed(0)); t2 = time.perf_counter()
    km.close()
    print(f"seed {1e3*(t1-t0):.2f} ms, lloyd(incl seed) {1e3*(t2-t1):.2f} ms, iters {km.last['iters'].tolist()}", flush=True)
