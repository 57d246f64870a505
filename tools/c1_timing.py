"""Config 1 through fast_spectral_cluster, cold then warm: stage timings (ms)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2310_10939_b200 import SpectralParams, fast_spectral_cluster  # noqa: E402
from paper_2310_10939_b200.generate import config_sbm, sample_sbm  # noqa: E402

g = sample_sbm(config_sbm(1)).graph
for rep in range(6):
    t0 = time.perf_counter()
    res = fast_spectral_cluster(g, SpectralParams(k=5, t=50, mode="one_vector", seed=0))
    t1 = time.perf_counter()
    print(f"rep {rep}: wall {1e3 * (t1 - t0):.2f} ms, stages { {k: round(v, 3) for k, v in res.timings.items()} }",
          flush=True)
