"""Check sc_seqsum (exact sequential sums on the GPU) against a scalar loop."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2310_10939_b200 import _lib  # noqa: E402


def run(vals, offs):
    tot = np.empty(len(offs) - 1)
    nch = sum((offs[i + 1] - offs[i] + 255) // 256 for i in range(len(offs) - 1))
    cs = np.empty(max(nch, 1))
    _lib.check(_lib.load().sc_seqsum(_lib.ptr(vals), len(offs) - 1,
                                     _lib.ptr(np.asarray(offs, dtype=np.int64)), 0, _lib.ptr(tot),
                                     _lib.ptr(cs)))
    return tot, cs


rng = np.random.default_rng(0)
cases = {
    "uniform": rng.random(100000),
    "wide": np.exp(rng.normal(0, 12, 20000)),
    "wide2": np.exp(rng.normal(0, 40, 20000)),
    "dyadic": rng.integers(0, 4096, 50000) * 0.125,
    "ints": rng.integers(0, 3, 70000).astype(float),
    "zeros_then": np.concatenate([np.zeros(1000), rng.random(5000)]),
    "sub": rng.random(3000) * 1e-310,
    "spiky": np.where(rng.random(50000) < 0.001, 1e30, rng.random(50000)),
    "d2like": (rng.random(20000) - 0.5) ** 2 * np.exp(rng.normal(0, 10, 20000)),
}
for name, a in cases.items():
    a = np.ascontiguousarray(a)
    tot, cs = run(a, [0, a.size])
    cum = np.concatenate([[0.0], np.cumsum(a)])
    starts = cum[np.arange(0, a.size, 256)]
    ok = tot[0] == cum[-1] and np.array_equal(cs[: starts.size], starts)
    if not ok:
        fb = np.flatnonzero(cs[: starts.size] != starts)
        print("FAIL", name, tot[0], cum[-1], "first bad chunks", fb[:5].tolist(),
              cs[fb[:2]].tolist() if fb.size else None, starts[fb[:2]].tolist() if fb.size else None)
    else:
        print("ok", name)
a = np.exp(rng.normal(0, 8, 200000))
offs = [0] + np.sort(rng.choice(np.arange(1, a.size), 99, replace=False)).tolist() + [a.size]
tot, _ = run(a, offs)
ref = np.array([np.cumsum(a[offs[i]:offs[i + 1]])[-1] for i in range(len(offs) - 1)])
print("segments", np.array_equal(tot, ref), np.flatnonzero(tot != ref)[:5])
