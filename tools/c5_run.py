"""Config 5 at full size on one GPU: device SBM generation (n = 1e8, blocks of 1e5, expected
degree 16 in / 2 out), graph build straight from the device CSR, Irwin-Hall x0 and T = 100
power steps; prints timings and the size-independent checks."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2310_10939_b200 import DeviceGraph  # noqa: E402
from paper_2310_10939_b200.generate import DeviceCSR, config_sbm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10**8
T = 100
params = config_sbm(5) if n == 10**8 else None
if params is None:
    from paper_2310_10939_b200.generate import SbmParams
    params = SbmParams(n=n, k=n // 100_000, p=16 / (10**5 - 1), q=2 / (n - 10**5), seed=0)
t0 = time.perf_counter()
d = DeviceCSR(params)
t1 = time.perf_counter()
print(f"generate: n={d.n} (of {d.n_generated}) nnz={d.nnz} in {t1 - t0:.2f} s", flush=True)
dg = DeviceGraph.from_device_csr(d)
t2 = time.perf_counter()
info = dg.info()
print(f"graph: {t2 - t1:.2f} s, device bytes {info['device_bytes'] / 1e9:.1f} GB, "
      f"slices {info['ntiles']}, wide {info['long_rows']}", flush=True)
d.close()
x0 = dg.sample_irwin_hall(0, return_host=True)
for rep in range(2):
    xT, f = dg.power_iterate(T)
    tm = dg.last_timing
    print(f"power T={T}: {tm['power_ms']:.1f} ms, {tm['kernel_ms'] * 1e3:.1f} us/step, "
          f"{info['nnz'] * T / (tm['power_ms'] / 1e3) / 1e9:.1f} GNNZ/s", flush=True)
print("mass rel err", abs(xT.sum() - x0.sum()) / x0.sum(), "min x", xT.min(), flush=True)
