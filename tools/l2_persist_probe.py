"""Effect of the L2 persisting access-policy window on the gathered vector z for the larger
configs (z = 8n bytes: 32 MB at config 3, 80 MB at config 4, 800 MB at config 5)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2310_10939_b200 import DeviceGraph  # noqa: E402

for cfg in [int(c) for c in (sys.argv[1:] or ["3", "4"])]:
    g, T, _ = bench.build_config(cfg)
    with DeviceGraph(g) as dg:
        dg.sample_irwin_hall(0)
        for l2 in (False, True, False, True):
            dg.power_iterate(T, want_x=False, want_f=False, l2_persist=l2)
            tm = dg.last_timing
            print(f"config {cfg} l2_persist={l2}: {tm['kernel_ms'] * 1e3:.1f} us/step, "
                  f"{g.nnz / (tm['kernel_ms'] * 1e-3) / 1e9:.1f} GNNZ/s", flush=True)
