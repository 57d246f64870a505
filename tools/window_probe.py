"""How much of a row region's gathers would a few z panels staged in shared memory serve?

For config N (default 4) with the BFS pre-order: rows are cut into regions of P renumbered rows
(one CTA each), columns into panels of P renumbered ids; per region the panels are ranked by the
number of the region's entries they hold, and the coverage of the top-m panels is printed.
Runs on the GPU box (torch on cuda:0 for the 181M-entry histograms)."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2310_10939_b200 import DeviceGraph, _lib  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reorder = sys.argv[2] if len(sys.argv) > 2 else "bfs"
g, T, _ = bench.build_config(cfg)
n = g.n
with DeviceGraph(g, reorder=None if reorder == "none" else reorder) as dg:
    perm = np.empty(n, dtype=np.int32)
    st = _lib.load().sc_graph_order(dg.handle, perm.ctypes.data_as(ctypes.c_void_p))
    assert st == 0
dev = torch.device("cuda:0")
perm_t = torch.from_numpy(perm.astype(np.int64)).to(dev)
iperm = torch.empty(n, dtype=torch.int64, device=dev)
iperm[perm_t] = torch.arange(n, device=dev)
rp = torch.from_numpy(np.asarray(g.row_offsets)).to(dev)
col = torch.from_numpy(np.asarray(g.col_indices)).to(dev).long()
rows_old = torch.repeat_interleave(torch.arange(n, device=dev), rp[1:] - rp[:-1])
r_new = iperm[rows_old]
c_new = iperm[col]
del rows_old, col
nnz = r_new.numel()
print(f"config {cfg} reorder={reorder}: n={n} nnz={nnz}", flush=True)
for P in (2048, 4096, 8192):
    nreg = (n + P - 1) // P
    key = (r_new // P) * nreg + (c_new // P)
    uk, cnt = torch.unique(key, return_counts=True)
    reg = uk // nreg
    same = cnt[(uk % nreg) == reg].sum().item() / nnz
    # rank panels inside each region by count (descending)
    order = torch.argsort(reg * (1 << 32) + ((1 << 31) - cnt), stable=True)
    reg_s, cnt_s = reg[order], cnt[order]
    first = torch.ones_like(reg_s, dtype=torch.bool)
    first[1:] = reg_s[1:] != reg_s[:-1]
    idx = torch.arange(reg_s.numel(), device=dev)
    start = torch.cummax(torch.where(first, idx, torch.zeros_like(idx)), 0).values
    rank = idx - start
    line = [f"P={P}: own panel {same:.3f}; panels/region {uk.numel() / nreg:.1f}; top-m coverage"]
    for m in (1, 2, 3, 4, 5, 6, 8, 12):
        line.append(f"m={m}:{cnt_s[rank < m].sum().item() / nnz:.3f}")
    print(" ".join(line), flush=True)
    del key, uk, cnt, reg, order, reg_s, cnt_s, first, idx, start, rank
