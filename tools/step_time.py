"""Per-step SpMV time of a config's layout as the bench builds it (reorder auto, panels when
T >= 64), CUDA-event timed over 3 T-step passes.  Usage: step_time.py CFG"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_10939_b200 import DeviceGraph  # noqa: E402
from paper_2310_10939_b200.generate import CONFIG_T, config_device_csr, config_sbm, sample_sbm  # noqa: E402

cfg = int(sys.argv[1])
T = CONFIG_T[cfg]
if cfg in (1, 2):
    dg = DeviceGraph(sample_sbm(config_sbm(cfg)).graph, reorder="auto", panels=T >= 64)
elif cfg == 4:  # the BFS pre-order needs the host graph path (as the bench)
    with config_device_csr(cfg) as d:
        g = d.download().graph
    dg = DeviceGraph(g, reorder="auto", panels=T >= 64)
else:
    with config_device_csr(cfg) as d:
        dg = DeviceGraph.from_device_csr(d, panels=T >= 64)
dg.sample_irwin_hall(0)
ts = []
for rep in range(4):
    dg.power_iterate(T, want_x=False, want_f=False)
    ts.append(dg.last_timing["kernel_ms"] * 1e3)
print(f"cfg {cfg} SC_FAR_HINT={os.environ.get('SC_FAR_HINT', '-')}: per-step us {[round(t, 1) for t in ts[1:]]}",
      flush=True)
