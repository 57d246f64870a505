"""The 64-byte L2 fetch hint variants of the SELL kernels (BIGZ slice kernel, hinted wide-row
gathers; chosen at launch when the z space is larger than the L2, i.e. only at config-5 scale)
forced on small graphs in a subprocess (SC_ZHINT=1 is read once per process): weighted, unit,
fp32-value, sym / sign variants and wide rows, bit-identical to the unhinted kernels and to the
oracle."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import sys
import numpy as np
sys.path.insert(0, %r)
from oracle import oracle as O
from paper_2310_10939_b200 import DeviceGraph, from_edges

rng = np.random.default_rng(21)
n = 40_000
u, v = rng.integers(0, n, 260_000), rng.integers(0, n, 260_000)
hub_u = np.concatenate([np.full(700, 5), np.full(300, 31_000)])
hub_v = rng.integers(0, n, hub_u.size)
u, v = np.concatenate([u, hub_u]), np.concatenate([v, hub_v])
keep = u != v
a, b = np.minimum(u[keep], v[keep]), np.maximum(u[keep], v[keep])
key, first = np.unique(a * n + b, return_index=True)
w = (0.5 + rng.random(keep.sum()))[first]
out = {}
for name, ww, f32 in (("weighted", w, False), ("unit", None, False), ("fp32", w, True)):
    g, _ = from_edges(n, key // n, key %% n, ww, drop_isolated=True)
    with DeviceGraph(g, fp32_values=f32) as dg:
        assert dg.info()["long_rows"] >= 2
        x0 = dg.sample_irwin_hall(3, return_host=True)
        res = {}
        for sym in (False, True):
            for sign in (1.0, -1.0):
                res[(sym, sign)] = dg.power_iterate(9, sym=sym, sign=sign)
    if not f32:
        xo, fo = O.power_iterate(g.row_offsets, g.col_indices, g.weights, g.degrees, x0, 9)
        assert np.array_equal(res[(False, 1.0)][0], xo) and np.array_equal(res[(False, 1.0)][1], fo)
    out[name] = res
np.savez(sys.argv[1], **{f"{k}_{int(s)}_{int(sg)}_{i}": r[(s, sg)][i]
                         for k, r in out.items() for (s, sg) in r for i in (0, 1)})
print("ok")
""" % ROOT


def _run(tmp_path, hint):
    out = tmp_path / f"zhint{hint}.npz"
    env = dict(os.environ, SC_ZHINT=str(hint))
    r = subprocess.run([sys.executable, "-c", CODE, str(out)], capture_output=True, text=True,
                       env=env, cwd=ROOT, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
    return out


def test_hinted_kernels_bit_identical(tmp_path):
    import numpy as np

    a = np.load(_run(tmp_path, 1))
    b = np.load(_run(tmp_path, 0))
    assert sorted(a.files) == sorted(b.files) and len(a.files) == 24
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
