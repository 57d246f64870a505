"""Device generation of configs 3, 4 (and 5): sizes, generation and download times."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2310_10939_b200.generate import config_device_csr  # noqa: E402

for cfg in [int(a) for a in sys.argv[1:]] or [3, 4]:
    for rep in range(2):
        t0 = time.perf_counter()
        d = config_device_csr(cfg)
        t1 = time.perf_counter()
        s = d.download(pinned=True)
        t2 = time.perf_counter()
        g = s.graph
        deg = np.diff(g.row_offsets)
        print(f"config {cfg}: n={g.n} (generated {d.n_generated}) nnz={g.nnz} mean row {g.nnz / g.n:.2f} "
              f"max row {deg.max()} gen {1e3 * (t1 - t0):.0f} ms download {1e3 * (t2 - t1):.0f} ms "
              f"weights [{g.weights.min():.4g}, {g.weights.max():.4g}]" if g.weights is not None else "",
              flush=True)
        d.close()
