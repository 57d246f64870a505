import sys, time; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2310_10939_b200 import DeviceGraph
from paper_2310_10939_b200.generate import config_sbm, sample_sbm
from paper_2310_10939_b200.graph import as_graph
g = sample_sbm(config_sbm(2)).graph
for i in range(3):
    t = time.perf_counter(); g2 = as_graph(g); g2.validate(); t1 = time.perf_counter()
    dg = DeviceGraph(g); t2 = time.perf_counter()
    print(f"py validate {1e3*(t1-t):.1f} ms, DeviceGraph total {1e3*(t2-t1):.1f} ms", flush=True)
    dg.close()
