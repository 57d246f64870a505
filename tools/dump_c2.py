"""Writes the config-2 CSR (original ids) to /tmp/c2.rp / /tmp/c2.col for panel_jds_bench."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
g, _, _ = bench.build_config(2)
np.asarray(g.row_offsets, np.int64).tofile("/tmp/c2.rp")
np.asarray(g.col_indices, np.int32).tofile("/tmp/c2.col")
if len(sys.argv) > 1:  # also the SELL-renumbered graph (rows and columns renamed)
    from paper_2310_10939_b200 import _lib
    import ctypes
    rp = np.asarray(g.row_offsets, np.int64)
    perm = np.empty(g.n, np.int32)
    _lib.check(_lib.load().sc_sell_order(_lib.ptr(rp), g.n, _lib.ptr(perm)))
    iperm = np.empty(g.n, np.int64)
    iperm[perm] = np.arange(g.n)
    lens = np.diff(rp)[perm]
    nrp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = np.repeat(rp[:-1][perm] - nrp[:-1], lens) + np.arange(nrp[-1])
    ncol = iperm[np.asarray(g.col_indices)[idx]].astype(np.int32)
    nrp.tofile("/tmp/c2s.rp")
    ncol.tofile("/tmp/c2s.col")
