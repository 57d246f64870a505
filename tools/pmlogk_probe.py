"""pm_log_k at config 2 through fast_spectral_cluster: stage timings."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2310_10939_b200 import SpectralParams, fast_spectral_cluster  # noqa: E402
from paper_2310_10939_b200.generate import config_sbm, sample_sbm  # noqa: E402

g = sample_sbm(config_sbm(2)).graph
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    t = time.perf_counter()
    r = fast_spectral_cluster(g, SpectralParams(k=10, mode="pm_log_k", seed=0))
    print("pm_log_k", r.l, r.t, round((time.perf_counter() - t) * 1e3, 1), "ms",
          {k_: round(v, 1) for k_, v in r.timings.items()}, flush=True)
