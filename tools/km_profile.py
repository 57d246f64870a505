"""One exact k-means (C2 embedding, k=10, 10 restarts) inside a cudaProfilerStart/Stop range,
for `ncu --profile-from-start off --metrics gpu__time_duration.sum` launch lists."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2310_10939_b200 import DeviceGraph, KMeans1D  # noqa: E402
from paper_2310_10939_b200.generate import config_sbm, sample_sbm  # noqa: E402
from paper_2310_10939_b200.pipeline import _kmeans_seed  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g = sample_sbm(config_sbm(cfg)).graph
T, k = (100, 10) if cfg == 2 else (50, 5)
dg = DeviceGraph(g)
dg.sample_irwin_hall(0)
dg.power_iterate(T, want_x=False)
for rep in range(3):
    km = KMeans1D(graph=dg)
    if rep == 2:
        torch.cuda.profiler.start()
    t0 = time.perf_counter()
    part = km.lloyd(k, _kmeans_seed(0))
    t1 = time.perf_counter()
    if rep == 2:
        torch.cuda.profiler.stop()
    print(f"rep {rep}: lloyd incl. seeding {1e3 * (t1 - t0):.2f} ms, iters {km.last['iters'].tolist()}",
          flush=True)
    km.close()
