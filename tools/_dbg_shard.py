import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
from test_gpu_panels import _blocked
from oracle import oracle as O
from paper_2310_10939_b200 import distributed as D
g = _blocked(150_000, 50_000, 20, 2, seed=11)
rp, col, deg = g.row_offsets, g.col_indices.astype(np.int32), g.degrees
for world in (1, 2):
    for panels in (False, True):
        starts = D.partition_rows(rp, world)
        lrps = [rp[starts[r]:starts[r + 1] + 1] - rp[starts[r]] for r in range(world)]
        plan = D.ShardPlan(starts, [D.sell_order(x) for x in lrps], [D.n_sell_rows(x) for x in lrps], 1)
        r = 0
        lo, hi = int(starts[r]), int(starts[r + 1])
        s = D.CudaShard(lrps[r], plan.rename(col[rp[lo]:rp[hi]]), None, deg[lo:hi], plan, r, 0)
        if panels: print("built", s.build_panels())
        # z = x0/d for the whole graph in plan z space
        x0 = O.irwin_hall(deg, 2)
        zfull = s.zspace(plan.ncols)
        # place every rank's z into z space: perms
        for q in range(world):
            ql, qh = int(starts[q]), int(starts[q+1])
            perm = plan.perms[q]
            zq = (x0[ql:qh] / deg[ql:qh])[perm]
            own = plan.own(0, q)
            zfull[own[0]:own[0] + (qh - ql)] = torch.from_numpy(zq).cuda()
        xin = torch.from_numpy(x0[lo:hi][plan.perms[r]]).cuda()
        xout = s.zeros(s.n); zout = s.zspace(plan.ncols)
        s.step_piece(0, zfull, xin, xout, zout)
        torch.cuda.synchronize()
        got = s.to_original(xout)
        xT, f = O.power_iterate(rp, col, None, deg, x0, 1)
        ref = xT[lo:hi]
        bad = np.flatnonzero(got != ref)
        print(world, panels, "bad", bad.size, bad[:10], got[bad[:3]], ref[bad[:3]])
        s.close()
# diagnose world 2 panels: which neighbour is missing
world = 2
starts = D.partition_rows(rp, world)
lrps = [rp[starts[r]:starts[r + 1] + 1] - rp[starts[r]] for r in range(world)]
plan = D.ShardPlan(starts, [D.sell_order(x) for x in lrps], [D.n_sell_rows(x) for x in lrps], 1)
lo, hi = int(starts[0]), int(starts[1])
rc = plan.rename(col[rp[lo]:rp[hi]])
s = D.CudaShard(lrps[0], rc, None, deg[lo:hi], plan, 0, 0)
s.build_panels()
x0 = O.irwin_hall(deg, 2)
zfull = s.zspace(plan.ncols)
zhost = np.zeros(plan.ncols)
for q in range(world):
    ql, qh = int(starts[q]), int(starts[q+1])
    zq = (x0[ql:qh] / deg[ql:qh])[plan.perms[q]]
    own = plan.own(0, q)
    zhost[own[0]:own[0] + (qh - ql)] = zq
zfull.copy_(torch.from_numpy(zhost).cuda())
xin = torch.from_numpy(x0[lo:hi][plan.perms[0]]).cuda()
xout = s.zeros(s.n); zout = s.zspace(plan.ncols)
s.step_piece(0, zfull, xin, xout, zout)
torch.cuda.synchronize()
got = s.to_original(xout)
xT, f = O.power_iterate(rp, col, None, deg, x0, 1)
ref = xT[lo:hi]
bad = np.flatnonzero(got != ref)
from collections import Counter
cnt = Counter(); pos = Counter()
for i in bad[:400]:
    miss = 2 * (ref[i] - got[i])
    cs = rc[rp[lo + i] - rp[lo]: rp[lo + i + 1] - rp[lo]]
    j = np.argmin(np.abs(zhost[cs] - miss))
    cnt[int(cs[j]) // 8192] += 1
    pos[(int(j), len(cs))] += 1
print("missing column panels", sorted(cnt.items()))
print("position in row (j, len)", pos.most_common(8))
print("ncols", plan.ncols, "own0", plan.own(0, 0), "own1", plan.own(0, 1))
iperm = np.empty(len(plan.perms[0]), np.int64); iperm[plan.perms[0]] = np.arange(len(plan.perms[0]))
rows_by_cta = Counter()
for i in bad[:2000]:
    rows_by_cta[int(iperm[i]) // 1696] += 1
print("bad per CTA", sorted(rows_by_cta.items())[:60])
for i in bad[:6]:
    miss = 2 * (ref[i] - got[i])
    cs = rc[rp[lo + i] - rp[lo]: rp[lo + i + 1] - rp[lo]]
    j = np.argmin(np.abs(zhost[cs] - miss))
    print("row", i, "renum", iperm[i], "cta", iperm[i] // 1696, "missing col", cs[j], "panel", cs[j] // 8192, "pos", j, len(cs), "cols", cs.tolist())
