"""Profiling driver: config-2 power iteration without CUDA graphs (so ncu sees each
kernel launch), a few iterations.  Usage: python tools/prof_spmv.py [T] [--weighted] [--panels] [--windows] [--cfg N] [--no-reorder]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_10939_b200 import DeviceGraph  # noqa: E402
from paper_2310_10939_b200.generate import config_sbm, sample_sbm  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 4
weighted = "--weighted" in sys.argv
panels = "--panels" in sys.argv
cfg = 2
if "--cfg" in sys.argv:
    cfg = int(sys.argv[sys.argv.index("--cfg") + 1])
t = time.time()
import bench  # noqa: E402

g, _, _ = bench.build_config(cfg)
print(f"graph n={g.n} nnz={g.nnz} in {time.time()-t:.1f}s", flush=True)
# same pre-order choice as the bench and fast_spectral_cluster ("auto": BFS for scattered ids)
dg = DeviceGraph(g, keep_weights=weighted, panels=panels, windows="--windows" in sys.argv,
                 reorder=None if "--no-reorder" in sys.argv else "auto")
print("layout", {k: v for k, v in dg.info().items()}, "reorder", dg.reorder, flush=True)
dg.sample_irwin_hall(0)
for rep in range(2):
    dg.power_iterate(T, cuda_graph=False, want_x=False, want_f=False, force_weighted=weighted)
    print("rep", rep, dg.last_timing, flush=True)
