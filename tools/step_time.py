"""Per-step SpMV time of a config's layout as the bench builds it (reorder auto, panels when
T >= 64, row windows unless --no-windows), CUDA-event timed over 3 T-step passes.
Usage: step_time.py CFG [--no-windows] [--fp32]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_10939_b200 import DeviceGraph  # noqa: E402
from paper_2310_10939_b200.generate import CONFIG_T, config_device_csr, config_sbm, sample_sbm  # noqa: E402

cfg = int(sys.argv[1])
T = CONFIG_T[cfg]
win = "--no-windows" not in sys.argv
f32 = "--fp32" in sys.argv
if cfg in (1, 2):
    dg = DeviceGraph(sample_sbm(config_sbm(cfg)).graph, reorder="auto", panels=T >= 64)
elif cfg == 4:  # the BFS pre-order needs the host graph path (as the bench)
    with config_device_csr(cfg) as d:
        g = d.download().graph
    dg = DeviceGraph(g, reorder="auto", panels=T >= 64, windows=win, fp32_values=f32)
else:
    with config_device_csr(cfg) as d:
        dg = DeviceGraph.from_device_csr(d, panels=T >= 64, windows=win, fp32_values=f32)
dg.sample_irwin_hall(0)
ts = []
for rep in range(4):
    dg.power_iterate(T, want_x=False, want_f=False)
    ts.append(dg.last_timing["kernel_ms"] * 1e3)
info = dg.info()
print(f"cfg {cfg} windows={info['window_items']} panels={info['panel_groups']} fp32={f32}: "
      f"per-step us {[round(t, 1) for t in ts[1:]]}", flush=True)
