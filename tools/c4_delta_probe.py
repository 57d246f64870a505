"""How far apart are a row and its columns after the device renumbering (BFS pre-order +
SELL)?  For the C4 graph: the fraction of stored entries whose renumbered column lies within
+-2^15 / +-2^16 of the row, and within the slice's [min, min + 2^16) window -- what a 16-bit
column encoding could cover."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2310_10939_b200 import DeviceGraph  # noqa: E402
from paper_2310_10939_b200.generate import config_device_csr  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
with config_device_csr(cfg) as d:
    g = d.download().graph
with DeviceGraph(g, reorder="auto") as dg:
    import ctypes
    from paper_2310_10939_b200 import _lib
    perm = np.empty(g.n, dtype=np.int32)
    _lib.check(_lib.load().sc_graph_order(dg.handle, _lib.ptr(perm)))
    print("reorder", dg.reorder, dg.info()["long_rows"], flush=True)
iperm = np.empty_like(perm)
iperm[perm] = np.arange(g.n, dtype=np.int32)
rows = np.repeat(np.arange(g.n, dtype=np.int32), np.diff(g.row_offsets))
rr = iperm[rows].astype(np.int64)
cc = iperm[g.col_indices].astype(np.int64)
dlt = np.abs(cc - rr)
for b in (12, 15, 16, 18, 20):
    print(f"|c - r| < 2^{b}: {np.mean(dlt < (1 << b)):.4f}", flush=True)
# per 32-row slice window [min, min + 2^16)
sl = rr // 32
order = np.argsort(sl, kind="stable")
s_sorted = sl[order]
c_sorted = cc[order]
starts = np.flatnonzero(np.r_[True, s_sorted[1:] != s_sorted[:-1]])
mins = np.minimum.reduceat(c_sorted, starts)
maxs = np.maximum.reduceat(c_sorted, starts)
span = maxs - mins
cnt = np.diff(np.r_[starts, len(s_sorted)])
print(f"slices with column span < 2^16: {np.mean(span < 65535):.4f} (entries {np.sum(cnt[span < 65535]) / len(cc):.4f})")
