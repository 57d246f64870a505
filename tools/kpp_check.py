"""k-means++ seeding: the fused 1-D pipeline (k_kpp_update_map / chunk-map fix / compose mode 2
/ k_kpp_search2) against the classic per-round pipeline (SC_KPP_CLASSIC=1, run in a child
process) and the oracle, on random and clustered 1-D points.  Prints timings."""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2310_10939_b200 import KMeans1D  # noqa: E402


def seeds(x, k, R=10, seed=3):
    with KMeans1D(x) as km:
        km.seed_centers(k, seed, R)  # warm
        t = time.perf_counter()
        ch = km.seed_centers(k, seed, R)
        return ch, time.perf_counter() - t


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        n, k, kind = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
        x = np.load(f"/tmp/kpp_x_{kind}_{n}.npy")
        ch, t = seeds(x, k)
        np.save(f"/tmp/kpp_ch_{kind}_{n}_{k}.npy", ch)
        print(f"classic {t * 1e3:.1f} ms", flush=True)
        sys.exit(0)
    rng = np.random.default_rng(0)
    for n, k in [(50_000, 10), (1_000_000, 10), (1_000_000, 100), (3_000_000, 300)]:
        for kind in ("uniform", "band"):
            x = rng.random(n) if kind == "uniform" else 0.5 + 1e-9 * rng.standard_normal(n)
            np.save(f"/tmp/kpp_x_{kind}_{n}.npy", x)
            ch, t = seeds(x, k)
            env = dict(os.environ, SC_KPP_CLASSIC="1")
            out = subprocess.run([sys.executable, __file__, "child", str(n), str(k), kind], env=env,
                                 capture_output=True, text=True, timeout=600)
            ref = np.load(f"/tmp/kpp_ch_{kind}_{n}_{k}.npy")
            print(f"n={n} k={k} {kind}: fused {t * 1e3:.1f} ms, {out.stdout.strip()}, "
                  f"identical={np.array_equal(ch, ref)}", flush=True)
