"""Column-panel layout vs SELL on one handle (bench configs): build time, per-step kernel time
from the T-step CUDA graph, bit-identity.  Usage: python tools/panel_probe.py [cfg ...] [--weighted]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2310_10939_b200 import DeviceGraph  # noqa: E402

weighted = "--weighted" in sys.argv
cfgs = [int(a) for a in sys.argv[1:] if a.isdigit()] or [2]
for cfg in cfgs:
    t = time.time()
    g, T, k = bench.build_config(cfg)
    print(f"cfg {cfg}: n={g.n} nnz={g.nnz} built in {time.time() - t:.1f}s", flush=True)
    t = time.time()
    dg = DeviceGraph(g, panels=True, keep_weights=weighted)
    t_create = time.time() - t
    info = dg.info()
    print(f"  handle {t_create * 1e3:.0f} ms; panel groups {info['panel_groups']} "
          f"bytes {info['panel_bytes'] / 1e6:.1f} MB", flush=True)
    dg.sample_irwin_hall(0)
    res = {}
    for name, fs in (("panel", False), ("sell", True)):
        best = 1e9
        for rep in range(4):
            xT, f = dg.power_iterate(T, force_sell=fs)
            best = min(best, dg.last_timing["kernel_ms"])
        res[name] = (xT, f)
        print(f"  {name:5s}: {best * 1e3:8.1f} us/step  {g.nnz / best / 1e6:7.1f} GNNZ/s", flush=True)
    same = all(np.array_equal(a, b) for a, b in zip(res["panel"], res["sell"]))
    print(f"  bit-identical: {same}", flush=True)
    dg.close()
