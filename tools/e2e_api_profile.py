"""Time each piece of one fast_spectral_cluster call at config 2 (pinned host graph)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2310_10939_b200 import DeviceGraph, KMeans1D  # noqa: E402
from paper_2310_10939_b200.graph import Graph  # noqa: E402
from paper_2310_10939_b200.pipeline import _kmeans_seed  # noqa: E402

g, T, k = bench.build_config(2)
gp = Graph(n=g.n, row_offsets=bench.pinned_copy(g.row_offsets),
           col_indices=bench.pinned_copy(g.col_indices), weights=None,
           degrees=bench.pinned_copy(g.degrees))
for rep in range(5):
    t = [time.perf_counter()]
    dg = DeviceGraph(gp, panels=True); t.append(time.perf_counter())
    dg.sample_irwin_hall(0); t.append(time.perf_counter())
    _, f = dg.power_iterate(T, want_x=False); t.append(time.perf_counter())
    km = KMeans1D(graph=dg); t.append(time.perf_counter())
    part = km.lloyd(k, _kmeans_seed(0)); t.append(time.perf_counter())
    km.close(); t.append(time.perf_counter())
    dg.close(); t.append(time.perf_counter())
    names = ["upload", "x0", "power+f", "km_ctx", "kmeans", "km_close", "g_close"]
    print(" ".join(f"{n} {1e3*(b-a):.1f}" for n, a, b in zip(names, t, t[1:])),
          f"total {1e3*(t[-1]-t[0]):.1f}", flush=True)
