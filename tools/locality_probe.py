"""How much would a locality-preserving vertex numbering buy on config 4 (random ids w.r.t.
the geometry)?  Time the SpMV step with the generator's ids and with ids sorted by planted
cluster (an oracle ordering a graph-only BFS/RCM ordering would approximate)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402

from paper_2310_10939_b200 import DeviceGraph, from_csr  # noqa: E402
from paper_2310_10939_b200.generate import sample_weighted_rgg  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**7
s = sample_weighted_rgg(n, 100, seed=0)
g = s.graph


def timed(gg, name):
    with DeviceGraph(gg) as dg:
        dg.sample_irwin_hall(0)
        for _ in range(2):
            dg.power_iterate(50, want_x=False, want_f=False)
        ms = dg.last_timing["kernel_ms"]
    print(f"{name}: {ms * 1e3:.1f} us/step, {gg.nnz / (ms * 1e-3) / 1e9:.1f} GNNZ/s", flush=True)


timed(g, "generator ids")
t = time.time()
order = np.argsort(s.planted, kind="stable")  # new id -> old id
A = sp.csr_matrix((g.weights, g.col_indices, g.row_offsets), shape=(g.n, g.n))
B = A[order][:, order].tocsr()
B.sort_indices()
gb = from_csr(g.n, B.indptr.astype(np.int64), B.indices.astype(np.int32), B.data, g.degrees[order])
print(f"relabel on host: {time.time() - t:.1f} s", flush=True)
timed(gb, "cluster-sorted ids")
