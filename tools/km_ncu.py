"""One exact k-means on the config-2 embedding, for `ncu -k regex:k_fused_lloyd` captures."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2310_10939_b200 import DeviceGraph, KMeans1D  # noqa: E402
from paper_2310_10939_b200.generate import config_sbm, sample_sbm  # noqa: E402
from paper_2310_10939_b200.pipeline import _kmeans_seed  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g = sample_sbm(config_sbm(cfg)).graph
T, k = (100, 10) if cfg == 2 else (50, 5)
dg = DeviceGraph(g)
dg.sample_irwin_hall(0)
dg.power_iterate(T, want_x=False)
with KMeans1D(graph=dg) as km:
    part = km.lloyd(k, _kmeans_seed(0))
print("iters", km.last["iters"].tolist())
