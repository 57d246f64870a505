"""k-means replica at scale: SBM of the config-5 law with n vertices (default 1e7), T power
steps, then restarted Lloyd with k clusters on the device-resident f; prints phase times
(SC_KMEANS_PROFILE=1 adds the per-phase split).  Usage: big_kmeans.py [n] [k] [restarts]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_10939_b200 import DeviceGraph, KMeans1D  # noqa: E402
from paper_2310_10939_b200.generate import DeviceCSR, SbmParams  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**7
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
R = int(sys.argv[3]) if len(sys.argv) > 3 else 10
params = SbmParams(n=n, k=n // 100_000, p=16 / (10**5 - 1), q=2 / (n - 10**5), seed=0)
with DeviceCSR(params) as d:
    dg = DeviceGraph.from_device_csr(d)
dg.sample_irwin_hall(0)
dg.power_iterate(100, want_x=False)
t0 = time.perf_counter()
km = KMeans1D(graph=dg)
t1 = time.perf_counter()
ch = km.seed_centers(k, 7, R)
t2 = time.perf_counter()
part = km.lloyd(k, 7, restarts=R)
t3 = time.perf_counter()
print(f"n={n} k={k} R={R}: ctx {t1 - t0:.3f} s, k-means++ {t2 - t1:.3f} s, "
      f"lloyd (incl. seeding) {t3 - t2:.3f} s, iters {getattr(part, 'iters', None)}", flush=True)
