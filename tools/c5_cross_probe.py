"""Config-5 law with and without its cross-block edges: how much of the step time and of the
DRAM traffic belongs to the random cross-block gathers?  Usage: c5_cross_probe.py [q_scale ...]
(q = q_scale * config-5 q; default 1 and 1e-6).  One T-step pass per graph without a CUDA graph
when --ncu is given (so ncu sees the launches)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_10939_b200 import DeviceGraph  # noqa: E402
from paper_2310_10939_b200.generate import DeviceCSR, SbmParams, config_sbm  # noqa: E402

ncu = "--ncu" in sys.argv
scales = [float(a) for a in sys.argv[1:] if not a.startswith("--")] or [1.0, 1e-6]
base = config_sbm(5)
for sc in scales:
    p = SbmParams(n=base.n, k=base.k, p=base.p, q=base.q * sc, seed=0)
    with DeviceCSR(p) as d:
        dg = DeviceGraph.from_device_csr(d)
    dg.sample_irwin_hall(0)
    ts = []
    for rep in range(1 if ncu else 3):
        dg.power_iterate(3 if ncu else 20, want_x=False, want_f=False, cuda_graph=not ncu)
        ts.append(dg.last_timing["kernel_ms"])
    print(f"q_scale {sc:g}: n={dg.n} nnz={dg.nnz} per-step ms {[round(t, 3) for t in ts]} "
          f"-> {dg.nnz / (min(ts) * 1e-3) / 1e9:.1f} GNNZ/s", flush=True)
    dg.close()
