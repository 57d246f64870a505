"""Graph-handle creation time at config 2 from PAGEABLE numpy arrays (the reference caller's
case) and from pinned copies, steady state."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2310_10939_b200 import DeviceGraph  # noqa: E402
from paper_2310_10939_b200.generate import config_sbm, sample_sbm  # noqa: E402
from paper_2310_10939_b200.graph import Graph  # noqa: E402

g = sample_sbm(config_sbm(2)).graph
gp = Graph(n=g.n, row_offsets=np.array(g.row_offsets), col_indices=np.array(g.col_indices, dtype=np.int32),
           weights=None, degrees=np.array(g.degrees))
ts = []
for i in range(6):
    t = time.perf_counter()
    dg = DeviceGraph(gp, panels=True)
    ts.append(1e3 * (time.perf_counter() - t))
    dg.close()
print(f"pageable DeviceGraph(panels) ms: {[round(t, 2) for t in ts]}", flush=True)
