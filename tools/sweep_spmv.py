"""Time the SpMV tile variants (SC_SPMV_VARIANT) on a config graph and check they agree.
Usage: python tools/sweep_spmv.py [--cfg 2] [--weighted] [--variants 0,1,2,3]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys, time, hashlib, json
sys.path.insert(0, ROOT)
import numpy as np
from paper_2310_10939_b200 import DeviceGraph
from paper_2310_10939_b200.generate import config_sbm, sample_sbm, sample_dcsbm
cfg = int(os.environ["CFG"]); weighted = os.environ.get("W") == "1"
if cfg == 3:
    g = sample_dcsbm(4_000_000, 50, seed=0).graph
else:
    g = sample_sbm(config_sbm(cfg)).graph
dg = DeviceGraph(g)
dg.sample_irwin_hall(0)
T = 20
for _ in range(3):
    dg.power_iterate(T, want_x=False, want_f=False, force_weighted=weighted)
ts = []
for _ in range(5):
    dg.power_iterate(T, want_x=False, want_f=False, force_weighted=weighted)
    ts.append(dg.last_timing["kernel_ms"])
x, _ = dg.power_iterate(T, force_weighted=weighted, want_f=False)
print(json.dumps({"variant": os.environ.get("SC_SPMV_VARIANT", "0"), "kernel_us": 1e3 * min(ts),
                  "median_us": 1e3 * sorted(ts)[2], "nnz": g.nnz, "n": g.n,
                  "sha": hashlib.sha256(x.tobytes()).hexdigest()[:16], "info": dg.info()["ntiles"]}))
'''.replace("ROOT", repr(ROOT))

args = sys.argv[1:]
cfg = args[args.index("--cfg") + 1] if "--cfg" in args else "2"
variants = args[args.index("--variants") + 1].split(",") if "--variants" in args else ["0", "1", "2", "3"]
carveouts = args[args.index("--carveouts") + 1].split(",") if "--carveouts" in args else ["-1"]
for v in variants:
    for cv in carveouts:
        env = dict(os.environ, SC_SPMV_VARIANT=v, CFG=cfg, SC_SPMV_CARVEOUT=cv,
                   W="1" if "--weighted" in args else "0")
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        print("carveout", cv, out.stdout.strip()[:110] or out.stderr[-2000:], flush=True)
