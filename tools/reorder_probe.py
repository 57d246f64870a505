"""SpMV step time with and without the BFS locality pre-order (configs 2 and 4)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2310_10939_b200 import DeviceGraph  # noqa: E402

for cfg in [int(c) for c in (sys.argv[1:] or ["2", "4"])]:
    g, T, _ = bench.build_config(cfg)
    for reorder in (None, "bfs"):
        with DeviceGraph(g, reorder=reorder) as dg:
            dg.sample_irwin_hall(0)
            for _ in range(2):
                dg.power_iterate(T, want_x=False, want_f=False)
            ms = dg.last_timing["kernel_ms"]
        print(f"config {cfg} reorder={reorder}: {ms * 1e3:.1f} us/step, "
              f"{g.nnz / (ms * 1e-3) / 1e9:.1f} GNNZ/s", flush=True)
