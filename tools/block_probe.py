"""Block power method (pm_log_k embedding) throughput at config 2: us per step and
GNNZ*cols/s for L = 1..16 columns (unit weights)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2310_10939_b200 import DeviceGraph  # noqa: E402

g, _, _ = bench.build_config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
T = 50
with DeviceGraph(g) as dg:
    for L in (1, 2, 3, 4, 6, 8, 10, 12, 16):
        x0 = np.random.default_rng(0).standard_normal((g.n, L))
        dg.power_iterate_block(x0, T, want_raw=False)
        dg.power_iterate_block(x0, T, want_raw=False)
        ms = dg.last_timing["kernel_ms"]
        print(f"L={L:2d}: {ms * 1e3:7.1f} us/step  {g.nnz * L / (ms * 1e-3) / 1e9:7.1f} "
              f"GNNZ*col/s", flush=True)
