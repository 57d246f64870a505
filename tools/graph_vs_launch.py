"""Fresh handle per call (the drop-in's case): wall time of the T-step power iteration with the
captured CUDA graph (capture + instantiate + launch) vs plain stream launches, config 2."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2310_10939_b200 import DeviceGraph  # noqa: E402
from paper_2310_10939_b200.graph import Graph  # noqa: E402

g, T, k = bench.build_config(2)
gp = Graph(n=g.n, row_offsets=bench.pinned_copy(g.row_offsets), col_indices=bench.pinned_copy(g.col_indices),
           weights=None, degrees=bench.pinned_copy(g.degrees))
for mode in (True, False, True, False):
    ts = []
    for rep in range(6):
        with DeviceGraph(gp, panels=True) as dg:
            dg.sample_irwin_hall(0)
            t0 = time.perf_counter()
            dg.power_iterate(T, want_x=False, want_f=False, cuda_graph=mode)
            ts.append(1e3 * (time.perf_counter() - t0))
    print(f"cuda_graph={mode}: power_iterate wall ms {[round(t, 2) for t in ts]}", flush=True)
