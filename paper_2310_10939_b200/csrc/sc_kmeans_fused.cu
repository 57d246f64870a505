// sc_kmeans_fused.cu -- the exact restarted Lloyd (specluster/kmeans.py:167-215) for 1-D
// points of one sign and k <= 32, every iteration of every restart inside ONE persistent
// cooperative kernel: no host round trip, no sort, no per-phase launches.
//
// The arithmetic contract is the one of sc_kmeans.cu, element by element:
//   distances   _sq_dists_to (kmeans.py:106-113) = d2ref, argmin lowest index (:199)
//   repair      _repair_empty (kmeans.py:151-164): empties listed once, in order, each takes
//               the first point of maximal own distance, whose own distance is then zeroed
//   means       np.add.at (kmeans.py:89): per cluster, a SEQUENTIAL sum in point-index order,
//               then / count (empty -> 0)
//   cost        kmeans_cost (kmeans.py:96-103): numpy einsum order (sc_oracle.c
//               orc_einsum_sumsq) -- see "stop decisions" below
//   stop rules  kmeans.py:202-210, the cost assertion of :206, best = first strictly smallest
//
// How the means stay exact without sorting.  Points are cut into chunks of 1024 consecutive
// indices (32 per lane, lane-contiguous).  Per (restart r, cluster j):
//   P1  one warp per (r, chunk): assignment, changed count, and per cluster present in the
//       chunk its count and an approximate sum (any order);
//   P2  one warp per (r, j): approximate prefix over the chunks -> the binade the exact
//       running sum is expected to sit in across each chunk (sc_seqsum.cuh "ulp grid");
//   P3  one warp per (r, chunk): for each cluster whose chunk has a predicted binade, the
//       parity map of its elements (sc_seqsum.cuh PMap) on that grid, composed in index order;
//   P4  one warp per (r, j): walks the chunks in order with the EXACT running sum: 32 chunk
//       maps are composed and applied at once when they share the running sum's grid and the
//       result stays inside the binade, otherwise chunk by chunk, and a chunk whose prediction
//       fails (a binade crossing) is added element by element.  Every shortcut is verified
//       against the exact value, so predictions only decide speed, never bits.  The points
//       are of one sign (x < 0 inputs run on -x: d2ref, the means and the cost are odd/even
//       functions under exact negation), so running sums are monotone and "start and end in
//       one binade" proves that no intermediate sum left it.
//
// Stop decisions without the einsum chain.  The reference's cost is a sum of the terms
// t_i = fl(fl(x_i - mu)^2) in numpy's einsum order: chains of <= 4096 dependent adds per
// 8192-element buffer, then one add per buffer.  Each iteration computes instead C~, the same
// terms summed in a fixed tree order, and the proven bound |C - C~| <= delta * C~ with
// delta = 2 * (4097 + nbuf + depth(tree)) * 2^-53 (both are sums of the same nonnegative
// terms; each term passes through at most that many roundings).  The stop rule
// (fl(P - C) <= fl(tol * max(P, 1e-300))) and the assertion are evaluated on intervals; only
// if an interval straddles the threshold are the exact einsum-order costs of that iteration
// and of the previous one computed (same kernel, all warps).  Unchanged labels stop without a
// cost (kmeans.py:201,208), and then C == P exactly.  The costs that pick the best restart are
// always the exact einsum-order values.
//
// Speculation.  P1 of iteration it+1 also accumulates the cost terms of iteration it (the
// same pass reads x, the labels of it and the means of it), so the stop decision for it is
// taken in P2 of it+1; a restart that stops ignores the work it did for it+1.  Labels and
// centres are triple-buffered so the previous iteration's labels/means survive for an exact
// cost recomputation.
#include <cuda_runtime.h>

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "sc_common.cuh"
#include "sc_seqsum.cuh"

namespace cg = cooperative_groups;

namespace sc {

constexpr int kFlChunk = 1024;  // points per chunk
constexpr int kFlLane = 32;     // points per lane (lane-contiguous)
constexpr int kFlMaxK = 32;
constexpr int kFlMaxR = 64;
constexpr int kFlMaxRK = 1024;
constexpr int kFlThreads = 256;
constexpr int kFlWarps = kFlThreads / 32;
constexpr int kFlEinsumBuf = 8192;
constexpr int kSkip = kNoGrid + 1;  // chunk holds no element of the cluster
constexpr int kCrossTag = 1 << 20;   // pred = kCrossTag + grid: one binade crossing predicted
__device__ __forceinline__ bool is_cross(int p) { return p >= kCrossTag / 2; }
__device__ __forceinline__ bool is_grid(int p) { return p > kSkip && p < kCrossTag / 2; }
constexpr int kFlStage = 256;       // exact-cost staging window per warp
constexpr int kXsPitch = 33;        // doubles per lane row of a warp's chunk tile (2-way banks)
constexpr int kXsWarp = 32 * kXsPitch;
constexpr int kFlDynSmem = kFlWarps * kXsWarp * 8;

// control block (int32 slots)
enum : int {
    kCtlAmb = 0,      // some restart needs the exact costs of its last two iterations
    kCtlRepair = 1,   // some restart has an empty cluster after assignment
    kCtlErr = 2,      // cost assertion failed (kmeans.py:206): restart + 1
    kCtlErrIt = 3,
    kCtlIters = 4,    // iterations executed by the kernel
    kCtlBest = 5,
    kCtlSlots = 8
};

struct FlArgs {
    const double *x;  // [n] points, all >= 0
    int64_t n;
    int64_t ln;        // label row stride (n rounded up to a chunk: aligned vector access)
    int k, R, nch, max_iters;
    int64_t nbuf;
    double tol, delta;
    double xmax;       // max point value (rounding bands of the sorted-centre assignment)
    uint8_t *lab;      // [3][R][n]
    double *cen;       // [3][R][k]
    double *A;         // [R][k][nch] approximate chunk sums
    int32_t *cnt;      // [R][k][nch]
    int32_t *pred;     // [R][k][nch] grid scale of the chunk, kNoGrid, kSkip
    int64_t *M;        // [R][k][nch][2] parity maps (before the crossing, if any)
    int64_t *MC;       // [R][k][nch][4] crossing chunks: map after, crossing value, grid after
    double *AS;        // [R][k][nch] approximate running sum at each chunk start
    double *cpart;     // [R][nch] approximate cost partials
    int32_t *tot;      // [R][k] cluster sizes
    int32_t *changed;  // [2][R]
    int32_t *ctl;      // kCtlSlots
    int32_t *stop;     // [R] sticky: restart finished
    int32_t *amb;      // [R]
    int32_t *rep;      // [R]
    int32_t *final_it; // [R]
    double *capprox;   // [R] cost of the previous decided iteration (C~ or exact)
    double *cfresh;    // [R] C~ of the iteration being decided
    double *bpart;     // [2][R][nbuf] exact cost buffer partials
    double *cexact;    // [R] exact final costs
    double *own;       // [n] repair scratch
    double *gval;      // [grid] argmax partials
    int64_t *gidx;
    unsigned long long *tprof;  // optional phase timestamps [256][8] (SC_KMEANS_PROFILE)
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ uint8_t *lab_buf(const FlArgs &a, int it, int r) {
    return a.lab + ((size_t)(it % 3) * a.R + r) * a.ln;
}
__device__ __forceinline__ double *cen_buf(const FlArgs &a, int it, int r) {
    return a.cen + ((size_t)(it % 3) * a.R + r) * a.k;
}

// ordered (index-order) composition of the 32 lanes' maps; result valid in lane 0
__device__ __forceinline__ PMap warp_reduce_pmap(PMap m) {
    const int lane = lane_id();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        PMap o;
        o.i0 = __shfl_down_sync(0xffffffffu, m.i0, d);
        o.i1 = __shfl_down_sync(0xffffffffu, m.i1, d);
        if ((lane & (2 * d - 1)) == 0) m = pmap_then(m, o);
    }
    return m;
}

// fixed-order warp sum (deterministic); result in every lane
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int warp_isum(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// the labels of a lane's 32 points, packed 4 per word
struct Lab32 {
    uint32_t w[8];
    __device__ __forceinline__ int get(int t) const { return (w[t >> 2] >> (8 * (t & 3))) & 0xff; }
    __device__ __forceinline__ void set(int t, int v) {
        w[t >> 2] = (w[t >> 2] & ~(0xffu << (8 * (t & 3)))) | ((uint32_t)v << (8 * (t & 3)));
    }
};

__device__ __forceinline__ void load_lab32(const uint8_t *p, int m, Lab32 &L) {
    if (m == kFlLane) {
        const uint4 a = __ldcg(reinterpret_cast<const uint4 *>(p));
        const uint4 b = __ldcg(reinterpret_cast<const uint4 *>(p) + 1);
        L.w[0] = a.x; L.w[1] = a.y; L.w[2] = a.z; L.w[3] = a.w;
        L.w[4] = b.x; L.w[5] = b.y; L.w[6] = b.z; L.w[7] = b.w;
    } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) L.w[q] = 0;
#pragma unroll
        for (int t = 0; t < kFlLane; ++t)
            if (t < m) L.set(t, __ldcg(p + t));
    }
}

__device__ __forceinline__ void store_lab32(uint8_t *p, int m, const Lab32 &L) {
    if (m == kFlLane) {
        __stcg(reinterpret_cast<uint4 *>(p), make_uint4(L.w[0], L.w[1], L.w[2], L.w[3]));
        __stcg(reinterpret_cast<uint4 *>(p) + 1, make_uint4(L.w[4], L.w[5], L.w[6], L.w[7]));
    } else {
#pragma unroll
        for (int t = 0; t < kFlLane; ++t)
            if (t < m) p[t] = (uint8_t)L.get(t);
    }
}

// chunk c's points into the warp's tile: lane t's run of 32 at xs[t * kXsPitch + q]; zeros
// past n.  Coalesced global loads (256 contiguous bytes per warp instruction), 8 in flight.
__device__ __forceinline__ void stage_chunk(const FlArgs &a, int c, double *xs) {
    const int lane = lane_id();
    const int64_t base = (int64_t)c * kFlChunk;
    __syncwarp();
    if (base + kFlChunk <= a.n) {
#pragma unroll
        for (int g = 0; g < 32; g += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(a.x + base + 32 * (g + u) + lane);
#pragma unroll
            for (int u = 0; u < 8; ++u) xs[(g + u) * kXsPitch + lane] = v[u];
        }
    } else {
        for (int u = 0; u < 32; ++u) {
            const int64_t i = base + 32 * u + lane;
            xs[u * kXsPitch + lane] = i < a.n ? __ldg(a.x + i) : 0.0;
        }
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------------------
// P1 for one (r, chunk).  assign: new labels from the centres in shared memory.
// resum: the labels of iteration it are read back (after a repair).  cost: C~ terms of
// iteration it-1 (neither assign nor resum: the cost terms only, for the last iteration).
// Per-restart centre tables built by every block at the top of an iteration: the distinct
// centre values sorted ascending (each with its lowest centre id: equal values have equal
// distances, and argmin keeps the lowest id), and around each midpoint m_i a band
// [m_i - eps_i, m_i + eps_i] with eps_i = 8 u M^2 / gap_i (M = max point / centre value).
// For x >= 0 and c in [0, M], |d2ref(x, c) - (x - c)^2| <= 6 u M^2, and the exact distances of
// the two neighbours differ by 2 gap_i |x - m_i|; so outside every band the centre of x's
// interval beats every other centre under d2ref strictly, and inside band i only the two
// neighbours can win (bands are disjoint, else the restart takes the brute-force argmin).
// Non-negative doubles order like their bit patterns: the band search is integer compares.
struct CenTab {
    double *cen;               // [R*k] by id
    double *sv;                // [R*k] sorted distinct values (restart r at r*k)
    uint8_t *sid;              // their ids
    unsigned long long *bl, *bh;  // band bounds (bits), kd-1 per restart
    int *kd;                   // distinct count, or -1: brute force
};

__device__ __forceinline__ int assign_one(const CenTab &T, int r, int k, double xv) {
    const int kd = T.kd[r];
    const double *cr = T.cen + r * k;
    if (kd < 0) {
        const double xx = __dmul_rn(xv, xv), tx = __dmul_rn(2.0, xv);
        double bv = INFINITY;
        int lb = 0;
        for (int j = 0; j < k; ++j) {
            const double c = cr[j];
            double v = __dadd_rn(__dsub_rn(xx, __dmul_rn(tx, c)), __dmul_rn(c, c));
            v = v < 0.0 ? 0.0 : v;
            if (v < bv) {
                bv = v;
                lb = j;
            }
        }
        return lb;
    }
    const unsigned long long xb = (unsigned long long)__double_as_longlong(xv);
    const unsigned long long *bl = T.bl + r * k, *bh = T.bh + r * k;
    const int nb = kd - 1;
    int pos = 0;
#pragma unroll
    for (int step = 16; step; step >>= 1)
        if (pos + step <= nb && bl[pos + step - 1] <= xb) pos += step;
    if (pos > 0 && bh[pos - 1] >= xb) {
        const double c1 = T.sv[r * k + pos - 1], c2 = T.sv[r * k + pos];
        const int i1 = T.sid[r * k + pos - 1], i2 = T.sid[r * k + pos];
        const double d1 = d2ref(xv, c1), d2 = d2ref(xv, c2);
        return (d2 < d1 || (d2 == d1 && i2 < i1)) ? i2 : i1;
    }
    return T.sid[r * k + pos];
}

// block-wide: tables of every restart from T.cen (the centres of this iteration)
__device__ void build_tables(const CenTab &T, int R, int k, double xmax) {
    const int rk = R * k;
    __syncthreads();
    for (int t = threadIdx.x; t < R; t += blockDim.x) T.kd[t] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < rk; t += blockDim.x) {
        const int r = t / k, j = t % k;
        const double c = T.cen[t];
        bool first = true;
        for (int q = 0; q < j; ++q) first &= T.cen[r * k + q] != c;
        if (!first) continue;
        int rank = 0;  // distinct values below c (each counted at its first id)
        for (int q = 0; q < k; ++q) {
            const double o = T.cen[r * k + q];
            if (o < c) {
                bool f2 = true;
                for (int q2 = 0; q2 < q; ++q2) f2 &= T.cen[r * k + q2] != o;
                rank += f2;
            }
        }
        T.sv[r * k + rank] = c;
        T.sid[r * k + rank] = (uint8_t)j;
        atomicAdd(T.kd + r, 1);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < rk; t += blockDim.x) {
        const int r = t / k, i = t % k;
        const int kd = T.kd[r];
        if (i + 1 >= kd) continue;
        const double lo = T.sv[r * k + i], hi = T.sv[r * k + i + 1];
        const double M = fmax(xmax, T.sv[r * k + kd - 1]);
        const double gap = hi - lo;
        const double eps = (M * M) * (8.0 * 1.1102230246251565e-16) / gap * (1.0 + 1.0 / 65536.0);
        const double mid = 0.5 * (lo + hi);
        double b0 = mid - eps, b1 = mid + eps;
        if (!(b0 > 0.0)) b0 = 0.0;
        if (!(b1 <= 1.7976931348623157e308)) b1 = INFINITY;
        T.bl[r * k + i] = (unsigned long long)__double_as_longlong(b0);
        T.bh[r * k + i] = (unsigned long long)__double_as_longlong(b1);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < rk; t += blockDim.x) {
        const int r = t / k, i = t % k;
        const int kd = T.kd[r];
        if (kd < 0 || i + 2 >= kd) continue;
        if (T.bh[r * k + i] >= T.bl[r * k + i + 1]) T.kd[r] = -1;  // bands overlap
    }
    __syncthreads();
    for (int t = threadIdx.x; t < R; t += blockDim.x)  // M^2 would overflow, or underflow so
        if (!(xmax <= 1e150 && xmax >= 1e-140)) T.kd[t] = -1;  // far that subnormal rounding counts
    __syncthreads();
}

__device__ void p1_chunk(const FlArgs &a, int it, int r, int c, bool assign, bool resum, bool cost,
                         const CenTab &T, double *swarp, double *xs) {
    const double *scen = T.cen;
    const bool summ = assign || resum;
    const int lane = lane_id();
    const int k = a.k;
    const int64_t i0 = (int64_t)c * kFlChunk + (int64_t)lane * kFlLane;
    const int m = (int)max((int64_t)0, min((int64_t)kFlLane, a.n - i0));
    const double *cr = scen + r * k;
    stage_chunk(a, c, xs);
    const double *xr = xs + lane * kXsPitch;
    Lab32 prev, cur;
#pragma unroll
    for (int q = 0; q < 8; ++q) prev.w[q] = cur.w[q] = 0;
    if (m > 0) load_lab32(lab_buf(a, it + 2, r) + i0, m, prev);
    if (resum && m > 0) load_lab32(lab_buf(a, it, r) + i0, m, cur);
    double csum = 0.0;
    int nchg = 0;
    uint32_t mask = 0;
#pragma unroll
    for (int t = 0; t < kFlLane; ++t) {
        if (t < m) {
            const double xv = xr[t];
            const int pl = prev.get(t);
            if (cost) {
                const double d = __dsub_rn(xv, cr[pl]);
                csum = __dadd_rn(csum, __dmul_rn(d, d));
            }
            if (summ) {
                int lb;
                if (assign) {
                    lb = assign_one(T, r, k, xv);
                    cur.set(t, lb);
                } else {
                    lb = cur.get(t);
                }
                nchg += lb != pl;
                mask |= 1u << lb;
            }
        }
    }
    if (assign && m > 0) store_lab32(lab_buf(a, it, r) + i0, m, cur);
    if (cost) {
        csum = warp_sum(csum);
        if (lane == 0) __stcg(a.cpart + (size_t)r * a.nch + c, csum);
    }
    if (!summ) return;
    // per-cluster counts and approximate sums, clusters present in the chunk only
    double *sA = swarp;                                    // [k]
    int *sC = reinterpret_cast<int *>(swarp + kFlMaxK);    // [k]
    if (lane < k) {
        sA[lane] = 0.0;
        sC[lane] = 0;
    }
    __syncwarp();
    uint32_t wm = mask;
#pragma unroll
    for (int o = 16; o; o >>= 1) wm |= __shfl_xor_sync(0xffffffffu, wm, o);
    while (wm) {
        const int j = __ffs(wm) - 1;
        wm &= wm - 1;
        double sj = 0.0;
        int q = 0;
        if (mask & (1u << j)) {
            uint32_t bits = 0;
#pragma unroll
            for (int t = 0; t < kFlLane; ++t)
                if (t < m && cur.get(t) == j) bits |= 1u << t;
            q = __popc(bits);
            for (; bits; bits &= bits - 1) sj += xr[__ffs(bits) - 1];
        }
        sj = warp_sum(sj);
        q = warp_isum(q);
        if (lane == 0) {
            sA[j] = sj;
            sC[j] = q;
        }
    }
    __syncwarp();
    if (lane < k) {
        const size_t o = ((size_t)r * k + lane) * a.nch + c;
        __stcg(a.A + o, sA[lane]);
        __stcg(a.cnt + o, sC[lane]);
    }
    nchg = warp_isum(nchg);
    if (lane == 0 && nchg) atomicAdd(a.changed + (it & 1) * a.R + r, nchg);
    __syncwarp();
}

// ---------------------------------------------------------------------------------------
// P2 for one (r, j): approximate prefix -> per chunk the binade the exact running sum is
// expected in (or one predicted crossing into the next binade); cluster size.
__device__ void p2_scan(const FlArgs &a, int r, int j) {
    const int lane = lane_id();
    const size_t base = ((size_t)r * a.k + j) * a.nch;
    const double lo_f = 1.0 - 1.0 / 1048576.0, hi_f = 1.0 + 1.0 / 1048576.0;
    double carry = 0.0;
    int total = 0;
    constexpr int kU = 4;  // batches in flight
    for (int c00 = 0; c00 < a.nch; c00 += 32 * kU) {
        double av[kU];
        int cn[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int c = c00 + 32 * u + lane;
            av[u] = c < a.nch ? __ldcg(a.A + base + c) : 0.0;
            cn[u] = c < a.nch ? __ldcg(a.cnt + base + c) : 0;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int c = c00 + 32 * u + lane;
            double incl = av[u];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double o = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += o;
            }
            if (c < a.nch) {
                const double st = carry + (incl - av[u]);
                int kp = kSkip;
                if (cn[u]) {
                    kp = kNoGrid;
                    const double plo = st * lo_f, phi = (carry + incl) * hi_f;
                    if (plo >= 2.2250738585072014e-308) {
                        const Grid ga = grid_of(plo), gb = grid_of(phi);
                        if (ga.k == gb.k) kp = ga.k;
                        else if (gb.k == ga.k - 1 && gb.top == ga.top) kp = kCrossTag + ga.k;
                    } else if (phi == 0.0) {
                        kp = grid_of(0.0).k;  // zeros only: identity maps on the subnormal grid
                    }
                }
                __stcg(a.pred + base + c, kp);
                __stcg(a.AS + base + c, st);
            }
            carry += __shfl_sync(0xffffffffu, incl, 31);
            total += warp_isum(cn[u]);
        }
    }
    if (lane == 0) {
        __stcg(a.tot + (size_t)r * a.k + j, total);
        if (total == 0) {
            a.rep[r] = 1;
            atomicExch(a.ctl + kCtlRepair, 1);
        }
    }
}

// ---------------------------------------------------------------------------------------
// P3 for one (r, chunk): per cluster with a prediction, the parity map of its points on the
// predicted grid; for a predicted crossing, the point whose add crosses into the next binade
// (found on an approximate running sum with a relative margin of 2^-24, else the chunk is
// left to the walk), the map of the points before it and the map of the points after it.
__device__ void p3_chunk(const FlArgs &a, int it, int r, int c, int *spred, double *sas, double *xs) {
    const int lane = lane_id();
    const int k = a.k;
    const int64_t i0 = (int64_t)c * kFlChunk + (int64_t)lane * kFlLane;
    const int m = (int)max((int64_t)0, min((int64_t)kFlLane, a.n - i0));
    if (lane < k) {
        const size_t o = ((size_t)r * k + lane) * a.nch + c;
        const int p = __ldcg(a.pred + o);
        spred[lane] = p;
        sas[lane] = is_cross(p) ? __ldcg(a.AS + o) : 0.0;
    }
    __syncwarp();
    uint32_t want = 0;
    for (int j = 0; j < k; ++j) {
        const int p = spred[j];
        if (is_grid(p) || is_cross(p)) want |= 1u << j;
    }
    if (!want) return;
    stage_chunk(a, c, xs);
    const double *xr = xs + lane * kXsPitch;
    Lab32 cur;
#pragma unroll
    for (int q = 0; q < 8; ++q) cur.w[q] = 0;
    if (m > 0) load_lab32(lab_buf(a, it, r) + i0, m, cur);
    const double mlo = 1.0 - 1.0 / 16777216.0, mhi = 1.0 + 1.0 / 16777216.0;
    while (want) {
        const int j = __ffs(want) - 1;
        want &= want - 1;
        const int p = spred[j];
        uint32_t bits = 0;
#pragma unroll
        for (int t = 0; t < kFlLane; ++t)
            if (t < m && cur.get(t) == j) bits |= 1u << t;
        const size_t o = ((size_t)r * k + j) * a.nch + c;
        if (is_grid(p)) {
            PMap lm = pmap_id();
            for (uint32_t b = bits; b; b &= b - 1) lm = pmap_then(lm, pmap_elem(to_units(xr[__ffs(b) - 1], p)));
            lm = warp_reduce_pmap(lm);
            if (lane == 0) {
                __stcg(a.M + 2 * o, lm.i0);
                __stcg(a.M + 2 * o + 1, lm.i1);
            }
            continue;
        }
        const int g1 = p - kCrossTag, g2 = g1 - 1;
        const double B = scalbn(1.0, 53 - g1);  // bottom of the next binade
        double as = 0.0;
        for (uint32_t b = bits; b; b &= b - 1) as += xr[__ffs(b) - 1];
        double incl = as;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const double ov = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += ov;
        }
        const double st = sas[j] + (incl - as), en = sas[j] + incl;
        PMap m1 = pmap_id(), m2 = pmap_id();
        double ac = 0.0;
        int role;  // 0 before, 2 after, 1 holds the crossing, 3 undecidable
        if (!bits || en < B * mlo) role = 0;
        else if (st >= B * mhi) role = 2;
        else if (st < B * mlo) role = 1;
        else role = 3;
        if (role == 0) {
            for (uint32_t b = bits; b; b &= b - 1) m1 = pmap_then(m1, pmap_elem(to_units(xr[__ffs(b) - 1], g1)));
        } else if (role == 2) {
            for (uint32_t b = bits; b; b &= b - 1) m2 = pmap_then(m2, pmap_elem(to_units(xr[__ffs(b) - 1], g2)));
        } else if (role == 1) {
            double rr = st;
            int phase = 0;
            for (uint32_t b = bits; b; b &= b - 1) {
                const double xv = xr[__ffs(b) - 1];
                const double nr = rr + xv;
                if (phase == 0 && nr >= B * mlo) {
                    if (nr < B * mhi) role = 3;
                    ac = xv;
                    phase = 1;
                } else if (phase == 0) {
                    m1 = pmap_then(m1, pmap_elem(to_units(xv, g1)));
                } else {
                    m2 = pmap_then(m2, pmap_elem(to_units(xv, g2)));
                }
                rr = nr;
            }
            if (!phase) role = 3;
        }
        const unsigned holders = __ballot_sync(0xffffffffu, role == 1);
        const bool ok = !__any_sync(0xffffffffu, role == 3) && __popc(holders) == 1;
        m1 = warp_reduce_pmap(m1);
        m2 = warp_reduce_pmap(m2);
        const double acv = __shfl_sync(0xffffffffu, ac, holders ? __ffs(holders) - 1 : 0);
        if (lane == 0) {
            if (ok) {
                __stcg(a.M + 2 * o, m1.i0);
                __stcg(a.M + 2 * o + 1, m1.i1);
                __stcg(a.MC + 4 * o, m2.i0);
                __stcg(a.MC + 4 * o + 1, m2.i1);
                __stcg(reinterpret_cast<double *>(a.MC) + 4 * o + 2, acv);
                __stcg(a.MC + 4 * o + 3, (int64_t)g2);
            } else {
                __stcg(a.pred + o, kNoGrid);  // the walk adds this chunk element by element
            }
        }
    }
    __syncwarp();
}

// Exact addition of cluster j's points of chunk c to the running sum s where the chunk-level
// prediction failed (binade crossings).  Each lane predicts the binade of its own run of 32
// from s plus an approximate prefix and builds its run's parity map; the warp then advances
// over maximal runs of lanes that share the running sum's binade with one composed map, and
// adds a lane's run element by element only where a crossing falls inside it.
__device__ double cross_chunk(const FlArgs &a, int it, int r, int j, int c, double s, double *xs) {
    const int lane = lane_id();
    const int64_t i0 = (int64_t)c * kFlChunk + (int64_t)lane * kFlLane;
    const int m = (int)max((int64_t)0, min((int64_t)kFlLane, a.n - i0));
    stage_chunk(a, c, xs);
    const double *xr = xs + lane * kXsPitch;
    Lab32 cur;
#pragma unroll
    for (int q = 0; q < 8; ++q) cur.w[q] = 0;
    if (m > 0) load_lab32(lab_buf(a, it, r) + i0, m, cur);
    uint32_t bits = 0;
    double as = 0.0;
#pragma unroll
    for (int t = 0; t < kFlLane; ++t)
        if (t < m && cur.get(t) == j) {
            bits |= 1u << t;
            as += xr[t];
        }
    double incl = as;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += o;
    }
    const double lo_f = 1.0 - 1.0 / 1048576.0, hi_f = 1.0 + 1.0 / 1048576.0;
    int g = kSkip;
    PMap lm = pmap_id();
    if (bits) {
        g = kNoGrid;
        const double plo = (s + (incl - as)) * lo_f, phi = (s + incl) * hi_f;
        if (plo >= 2.2250738585072014e-308) {
            const Grid ga = grid_of(plo), gb = grid_of(phi);
            if (ga.k == gb.k) g = ga.k;
        }
        if (g != kNoGrid) {
#pragma unroll
            for (int t = 0; t < kFlLane; ++t)
                if ((bits >> t) & 1u) lm = pmap_then(lm, pmap_elem(to_units(xr[t], g)));
        }
    }
    int L = 0;
    while (L < 32) {
        const Grid gs = grid_of(s);
        const bool ok = g == kSkip || g == gs.k;
        const unsigned badm = __ballot_sync(0xffffffffu, !ok && lane >= L);
        const int L2 = badm ? __ffs(badm) - 1 : 32;
        if (L2 > L) {
            PMap pm = (lane >= L && lane < L2 && g != kSkip) ? lm : pmap_id();
            pm = warp_reduce_pmap(pm);
            const PMap bm{__shfl_sync(0xffffffffu, pm.i0, 0), __shfl_sync(0xffffffffu, pm.i1, 0)};
            const int64_t S1 = pmap_apply(bm, (int64_t)to_units(s, gs.k));
            if (S1 < gs.top) {
                s = from_units(S1, gs.k);
                L = L2;
                continue;
            }
        }
        double v = s;  // lane L element by element
        if (lane == L) {
#pragma unroll
            for (int t = 0; t < kFlLane; ++t)
                if ((bits >> t) & 1u) v = __dadd_rn(v, xr[t]);
        }
        s = __shfl_sync(0xffffffffu, v, L);
        L += 1;
    }
    return s;
}

// P4 for one (r, j): the exact walk over the chunks, 32 at a time: maximal runs of chunks on
// the running sum's grid advance with one composed map, a predicted crossing with its two
// maps and one real add of the crossing point, anything else element by element.  Every
// step is verified against the exact running value.  Writes the mean for iteration it+1.
__device__ void p4_walk(const FlArgs &a, int it, int r, int j, double *xs) {
    const int lane = lane_id();
    const size_t base = ((size_t)r * a.k + j) * a.nch;
    double s = 0.0;
    int pn = kSkip;
    PMap mn = pmap_id(), m2n = pmap_id();
    double acn = 0.0;
    int g2n = 0;
    auto fetch = [&](int c) {
        pn = kSkip;
        if (c < a.nch) {
            pn = __ldcg(a.pred + base + c);
            if (is_grid(pn) || is_cross(pn)) {
                mn.i0 = __ldcg(a.M + 2 * (base + c));
                mn.i1 = __ldcg(a.M + 2 * (base + c) + 1);
            }
            if (is_cross(pn)) {
                m2n.i0 = __ldcg(a.MC + 4 * (base + c));
                m2n.i1 = __ldcg(a.MC + 4 * (base + c) + 1);
                acn = __ldcg(reinterpret_cast<const double *>(a.MC) + 4 * (base + c) + 2);
                g2n = (int)__ldcg(a.MC + 4 * (base + c) + 3);
            }
        }
    };
    fetch(lane);
    for (int c0 = 0; c0 < a.nch; c0 += 32) {
        const int p = pn, g2 = g2n;
        const PMap mm = mn, m2 = m2n;
        const double ac = acn;
        fetch(c0 + 32 + lane);  // independent of the running value
        const int lim = min(32, a.nch - c0);
        if (__all_sync(0xffffffffu, p == kSkip)) continue;
        int L = 0;
        while (L < lim) {
            const Grid gs = grid_of(s);
            const bool ok = p == kSkip || p == gs.k;
            const unsigned badm = __ballot_sync(0xffffffffu, !ok && lane >= L && lane < lim);
            const int L2 = badm ? __ffs(badm) - 1 : lim;
            if (L2 > L) {
                const bool any = __any_sync(0xffffffffu, lane >= L && lane < L2 && p != kSkip);
                if (any) {
                    PMap pm = (lane >= L && lane < L2 && p != kSkip) ? mm : pmap_id();
                    pm = warp_reduce_pmap(pm);
                    const PMap bm{__shfl_sync(0xffffffffu, pm.i0, 0), __shfl_sync(0xffffffffu, pm.i1, 0)};
                    const int64_t S1 = pmap_apply(bm, (int64_t)to_units(s, gs.k));
                    if (S1 >= gs.top) {  // left the binade inside the run: first chunk by hand
                        s = cross_chunk(a, it, r, j, c0 + L, s, xs);
                        L += 1;
                        continue;
                    }
                    s = from_units(S1, gs.k);
                }
                L = L2;
                continue;
            }
            // chunk L is off the running grid
            const int pL = __shfl_sync(0xffffffffu, p, L);
            bool done = false;
            if (is_cross(pL) && pL - kCrossTag == gs.k) {
                const PMap a1{__shfl_sync(0xffffffffu, mm.i0, L), __shfl_sync(0xffffffffu, mm.i1, L)};
                const PMap a2{__shfl_sync(0xffffffffu, m2.i0, L), __shfl_sync(0xffffffffu, m2.i1, L)};
                const double acl = __shfl_sync(0xffffffffu, ac, L);
                const int g2l = __shfl_sync(0xffffffffu, g2, L);
                const int64_t S1 = pmap_apply(a1, (int64_t)to_units(s, gs.k));
                if (S1 < gs.top) {
                    const double s2 = __dadd_rn(from_units(S1, gs.k), acl);
                    const Grid g2s = grid_of(s2);
                    if (g2s.k == g2l) {
                        const int64_t S2 = pmap_apply(a2, (int64_t)to_units(s2, g2l));
                        if (S2 < g2s.top) {
                            s = from_units(S2, g2l);
                            done = true;
                        }
                    }
                }
            }
            if (!done) s = cross_chunk(a, it, r, j, c0 + L, s, xs);
            L += 1;
        }
    }
    if (lane == 0) {
        const int t = __ldcg(a.tot + (size_t)r * a.k + j);
        __stcg(cen_buf(a, it + 1, r) + j, t > 0 ? __ddiv_rn(s, (double)t) : 0.0);
    }
}

// ---------------------------------------------------------------------------------------
// Exact einsum-order cost partial of one 8192-point buffer (sc_oracle.c orc_einsum_sumsq):
// lanes stage fl(fl(x - mu)^2) 256 at a time, lanes 0/1 run the two SSE lane chains.
__device__ double exact_buf(const FlArgs &a, const uint8_t *lab, const double *cen, int64_t b,
                            double *stage) {
    const int lane = lane_id();
    const int64_t c0 = b * kFlEinsumBuf;
    const int64_t mtot = min((int64_t)kFlEinsumBuf, a.n - c0);
    const int64_t full_end = (mtot / 8) * 8;  // buffer-relative end of the 8-element steps
    double acc = 0.0;  // lane 0: a0, lane 1: a1
    double xv[8];
    int lv[8];
    auto fetch = [&](int64_t w0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int64_t t = w0 + 32 * q + lane;
            xv[q] = t < mtot ? __ldg(a.x + c0 + t) : 0.0;
            lv[q] = t < mtot ? (int)__ldcg(lab + c0 + t) : -1;
        }
    };
    fetch(0);
    for (int64_t w0 = 0; w0 < mtot; w0 += kFlStage) {
        const int wm = (int)min((int64_t)kFlStage, mtot - w0);
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            double v = 0.0;
            if (lv[q] >= 0) {
                const double d = __dsub_rn(xv[q], cen[lv[q]]);
                v = __dmul_rn(d, d);
            }
            stage[32 * q + lane] = v;
        }
        __syncwarp();
        if (w0 + kFlStage < mtot) fetch(w0 + kFlStage);
        if (lane < 2) {
            const int nfull = (int)min((int64_t)wm, full_end - w0);
            int t = 0;
#pragma unroll 4
            for (; t < nfull; t += 8) {
                acc = __dadd_rn(stage[t + 6 + lane], acc);
                acc = __dadd_rn(stage[t + 4 + lane], acc);
                acc = __dadd_rn(stage[t + 2 + lane], acc);
                acc = __dadd_rn(stage[t + lane], acc);
            }
            for (; t < wm; t += 2) {  // buffer tail: pairs, zero fill
                const double v = (t + lane < wm) ? stage[t + lane] : 0.0;
                acc = __dadd_rn(v, acc);
            }
        }
    }
    const double a1 = __shfl_sync(0xffffffffu, acc, 1);
    return __dadd_rn(acc, a1);  // lane 0: a0 + a1
}

// exact costs of restarts with flag[r] (labels/means of iterations it_of(r)), partials into
// bpart slot `slot`; all warps of the grid
__device__ void exact_partials(const FlArgs &a, const int32_t *flag, int it_lab, int slot,
                               double *stage, int gw, int nw) {
    const int64_t tasks = (int64_t)a.R * a.nbuf;
    for (int64_t t = gw; t < tasks; t += nw) {
        const int r = (int)(t / a.nbuf);
        const int64_t b = t - (int64_t)r * a.nbuf;
        if (!flag[r]) continue;
        const int f = it_lab >= 0 ? it_lab : a.final_it[r];
        const double v = exact_buf(a, lab_buf(a, f, r), cen_buf(a, f + 1, r), b, stage);
        if (lane_id() == 0) __stcg(a.bpart + ((size_t)slot * a.R + r) * a.nbuf + b, v);
    }
}

__device__ double exact_combine(const FlArgs &a, int slot, int r) {
    double out = 0.0;
    const double *p = a.bpart + ((size_t)slot * a.R + r) * a.nbuf;
    for (int64_t b = 0; b < a.nbuf; ++b) out = __dadd_rn(__ldcg(p + b), out);
    return out;
}

// interval evaluation of kmeans.py:206-207 with |P - P~| <= d P~, |C - C~| <= d C~.
// returns 1 small gain, 0 no small gain, -1 undecidable; *bad = 1 if the assertion fails
// for sure, -1 if undecidable
__device__ int certify(double P, double C, double tol, double d, int *bad) {
    const double u2 = 2.3e-16;  // 2 * 2^-53 (+ slack)
    *bad = 0;
    if (!(tol >= 0.0) || !(P >= 1e-280) || !(C >= 0.0)) {
        *bad = -1;
        return -1;
    }
    const double Plo = P * (1.0 - d), Phi = P * (1.0 + d), Clo = C * (1.0 - d), Chi = C * (1.0 + d);
    const double lim_lo = (Plo * (1.0 + 1e-12) + 1e-12) * (1.0 - 2 * u2);
    const double lim_hi = (Phi * (1.0 + 1e-12) + 1e-12) * (1.0 + 2 * u2);
    if (Clo > lim_hi) *bad = 1;
    else if (!(Chi <= lim_lo)) *bad = -1;
    const double L_lo = Plo - Chi, L_hi = Phi - Clo;
    const double f_lo = L_lo - fabs(L_lo) * u2 - 1e-300, f_hi = L_hi + fabs(L_hi) * u2 + 1e-300;
    const double r_lo = tol * Plo * (1.0 - u2), r_hi = tol * Phi * (1.0 + u2);
    if (f_hi <= r_lo) return 1;
    if (f_lo > r_hi) return 0;
    return -1;
}

// the reference's decision on exact costs; returns stop (1/0), error via *bad
__device__ int decide_exact(double P, double C, double tol, int *bad) {
    *bad = !(C <= P * (1.0 + 1e-12) + 1e-12);
    return (P - C <= tol * fmax(P, 1e-300)) ? 1 : 0;
}

// ---------------------------------------------------------------------------------------
// Repair of one restart's empty clusters after the assignment of iteration it
// (kmeans.py:151-164), then its chunk summaries and scans are redone.  Grid-uniform.
__device__ void repair_restart(const FlArgs &a, cg::grid_group &grid, int it, int r,
                               const CenTab &T, double *swarp, double *xs, int gw, int nw) {
    const double *scen = T.cen;
    const int k = a.k;
    uint8_t *lab = lab_buf(a, it, r);
    const double *cr = scen + r * k;
    // the empties, listed once (np.flatnonzero(counts == 0) before the loop)
    uint32_t empties = 0;
    for (int j = 0; j < k; ++j)
        if (__ldcg(a.tot + (size_t)r * k + j) == 0) empties |= 1u << j;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < a.n; i += nth) {
        const double xv = __ldg(a.x + i);
        const int l = __ldcg(lab + i);
        const double xx = __dmul_rn(xv, xv), tx = __dmul_rn(2.0, xv);
        double v = __dadd_rn(__dsub_rn(xx, __dmul_rn(tx, cr[l])), __dmul_rn(cr[l], cr[l]));
        a.own[i] = v < 0.0 ? 0.0 : v;
    }
    grid.sync();
    __shared__ double bv_s[kFlWarps];
    __shared__ int64_t bi_s[kFlWarps];
    while (empties) {
        const int j = __ffs(empties) - 1;
        empties &= empties - 1;
        double bv = -1.0;
        int64_t bi = a.n;
        for (int64_t i = tid; i < a.n; i += nth) {
            const double v = __ldcg(a.own + i);
            if (v > bv) {
                bv = v;
                bi = i;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane_id() == 0) {
            bv_s[threadIdx.x >> 5] = bv;
            bi_s[threadIdx.x >> 5] = bi;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < kFlWarps; ++w)
                if (bv_s[w] > bv_s[0] || (bv_s[w] == bv_s[0] && bi_s[w] < bi_s[0])) {
                    bv_s[0] = bv_s[w];
                    bi_s[0] = bi_s[w];
                }
            a.gval[blockIdx.x] = bv_s[0];
            a.gidx[blockIdx.x] = bi_s[0];
        }
        __syncthreads();
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            double v = -1.0;
            int64_t far = a.n;
            for (int b = 0; b < (int)gridDim.x; ++b) {
                const double ov = __ldcg(a.gval + b);
                const int64_t oi = __ldcg(a.gidx + b);
                if (ov > v || (ov == v && oi < far)) {
                    v = ov;
                    far = oi;
                }
            }
            lab[far] = (uint8_t)j;
            a.own[far] = 0.0;
        }
        grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.changed[(it & 1) * a.R + r] = 0;
    grid.sync();
    for (int c = gw; c < a.nch; c += nw) p1_chunk(a, it, r, c, false, true, false, T, swarp + (threadIdx.x >> 5) * 2 * kFlMaxK, xs);
    grid.sync();
    for (int j = gw; j < k; j += nw) p2_scan(a, r, j);
    grid.sync();
}

__device__ __forceinline__ void tmark(const FlArgs &a, int it, int ph) {
    if (a.tprof && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.tprof[(size_t)min(it, 255) * 8 + ph] = t;
    }
}

__global__ void __launch_bounds__(kFlThreads, 2) k_fused_lloyd(FlArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double scen[kFlMaxRK], ssv[kFlMaxRK];
    __shared__ unsigned long long sbl[kFlMaxRK], sbh[kFlMaxRK];
    __shared__ uint8_t ssid[kFlMaxRK];
    __shared__ int skd[kFlMaxR];
    __shared__ double sas_all[kFlWarps][kFlMaxK];
    CenTab T{scen, ssv, ssid, sbl, sbh, skd};
    __shared__ double swarp[kFlWarps * 2 * kFlMaxK];
    extern __shared__ double fl_dyn[];  // kFlWarps chunk tiles (also the exact-cost stage)
    __shared__ int act[kFlMaxR];
    __shared__ int nact_s;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int gw = blockIdx.x * kFlWarps + warp, nw = gridDim.x * kFlWarps;
    double *sw = swarp + warp * 2 * kFlMaxK;
    double *xs = fl_dyn + warp * kXsWarp;
    double *stage = xs;
    const int R = a.R, k = a.k, rk = R * k;
    auto load_active = [&]() {
        if (threadIdx.x == 0) {
            int q = 0;
            for (int r = 0; r < R; ++r)
                if (!__ldcg(a.stop + r)) act[q++] = r;
            nact_s = q;
        }
        __syncthreads();
    };
    load_active();
    int it = 0;
    for (;; ++it) {
        tmark(a, it, 0);
        const bool assign = it < a.max_iters, cost = it > 0;
        // centres of iteration it (= means of it-1) and their squares
        for (int t = threadIdx.x; t < rk; t += blockDim.x) {
            const double c = __ldcg(a.cen + (size_t)(it % 3) * rk + t);
            scen[t] = c;
        }
        if (assign) build_tables(T, R, k, a.xmax);
        __syncthreads();
        const int nact = nact_s;
        // ---- P1: assignment of it, C~ terms of it-1
        for (int t = gw; t < nact * a.nch; t += nw)
            p1_chunk(a, it, act[t / a.nch], t % a.nch, assign, false, cost, T, sw, xs);
        grid.sync();
        tmark(a, it, 1);
        // ---- P2: grid predictions of it; decision for it-1 (task index j == k)
        for (int t = gw; t < nact * (k + 1); t += nw) {
            const int r = act[t / (k + 1)], j = t % (k + 1);
            if (j < k) {
                if (assign) p2_scan(a, r, j);
                continue;
            }
            if (!cost) continue;
            double cs = 0.0;
            for (int c = lane; c < a.nch; c += 32) cs = __dadd_rn(cs, __ldcg(a.cpart + (size_t)r * a.nch + c));
            cs = warp_sum(cs);
            if (lane) continue;
            const int d_it = it - 1;  // iteration being decided
            const double P = a.capprox[r];
            const bool fin = d_it > 0;
            const bool unchanged = fin && __ldcg(a.changed + (d_it & 1) * R + r) == 0;
            int stop = 0, amb = 0;
            if (unchanged) {
                stop = 1;
            } else if (fin) {
                int bad = 0;
                const int sg = certify(P, cs, a.tol, a.delta, &bad);
                if (sg < 0 || bad < 0) amb = 1;
                else if (bad > 0) {
                    amb = 1;  // confirm with exact costs before raising
                } else {
                    stop = sg;
                }
            }
            a.cfresh[r] = cs;
            if (amb) {
                a.amb[r] = 1;
                atomicExch(a.ctl + kCtlAmb, 1);
                continue;
            }
            a.capprox[r] = cs;
            if (stop || d_it + 1 >= a.max_iters) {
                a.final_it[r] = d_it;
                a.stop[r] = 1;
            }
        }
        grid.sync();
        tmark(a, it, 2);
        if (__ldcg(a.ctl + kCtlAmb)) {
            // exact costs of it-1 (slot 0) and it-2 (slot 1) for the undecided restarts
            exact_partials(a, a.amb, it - 1, 0, stage, gw, nw);
            exact_partials(a, a.amb, it - 2, 1, stage, gw, nw);
            grid.sync();
            if (blockIdx.x == 0 && threadIdx.x < R) {
                const int r = threadIdx.x;
                if (a.amb[r]) {
                    const double C = exact_combine(a, 0, r), P = exact_combine(a, 1, r);
                    int bad = 0;
                    const int stop = decide_exact(P, C, a.tol, &bad);
                    if (bad) {
                        atomicCAS(a.ctl + kCtlErr, 0, r + 1);
                        a.ctl[kCtlErrIt] = it - 1;
                    }
                    a.capprox[r] = C;
                    if (stop || it >= a.max_iters) {
                        a.final_it[r] = it - 1;
                        a.stop[r] = 1;
                    }
                    a.amb[r] = 0;
                }
            }
            grid.sync();
            if (blockIdx.x == 0 && threadIdx.x == 0) a.ctl[kCtlAmb] = 0;
            if (__ldcg(a.ctl + kCtlErr)) break;  // uniform: read after the sync
        }
        __syncthreads();
        load_active();
        if (!assign || nact_s == 0) break;
        // ---- repair of empty clusters (rare)
        if (__ldcg(a.ctl + kCtlRepair)) {
            for (int q = 0; q < nact_s; ++q) {
                const int r = act[q];
                if (__ldcg(a.rep + r)) repair_restart(a, grid, it, r, T, swarp, xs, gw, nw);
            }
            if (blockIdx.x == 0 && threadIdx.x < R) a.rep[threadIdx.x] = 0;
            if (blockIdx.x == 0 && threadIdx.x == 0) a.ctl[kCtlRepair] = 0;
            // (the flags are next read after two more grid syncs)
        }
        // ---- P3: parity maps
        tmark(a, it, 3);
        const int na = nact_s;
        for (int t = gw; t < na * a.nch; t += nw)
            p3_chunk(a, it, act[t / a.nch], t % a.nch, reinterpret_cast<int *>(sw), sas_all[warp], xs);
        grid.sync();
        tmark(a, it, 4);
        // ---- P4: exact walks -> means of it
        for (int t = gw; t < na * k; t += nw) p4_walk(a, it, act[t / k], t % k, xs);
        if (blockIdx.x == 0 && threadIdx.x < R) a.changed[((it + 1) & 1) * R + threadIdx.x] = 0;
        grid.sync();
        tmark(a, it, 5);
    }
    tmark(a, 255, 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) a.ctl[kCtlIters] = it;
    if (__ldcg(a.ctl + kCtlErr)) return;
    // ---- exact final costs of every restart, best = first strictly smallest
    {
        int32_t *all = a.amb;  // reuse as "all restarts" flags
        if (blockIdx.x == 0 && threadIdx.x < R) all[threadIdx.x] = 1;
        grid.sync();
        exact_partials(a, all, -1, 0, stage, gw, nw);
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x < R) a.cexact[threadIdx.x] = exact_combine(a, 0, threadIdx.x);
        __syncthreads();
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            int best = -1;
            double bc = INFINITY;
            for (int r = 0; r < R; ++r) {
                a.amb[r] = 0;
                if (a.cexact[r] < bc) {
                    bc = a.cexact[r];
                    best = r;
                }
            }
            a.ctl[kCtlBest] = best;
        }
        tmark(a, 255, 1);
    }
}

__global__ void k_fl_init(FlArgs a, const double *xsrc, double sign, const int64_t *chosen) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int rk = a.R * a.k;
    for (int64_t t = tid; t < rk; t += nth) a.cen[t] = sign * xsrc[chosen[t]];  // cen[0]
    for (int64_t t = tid; t < (int64_t)a.R * a.ln; t += nth) a.lab[(size_t)2 * a.R * a.ln + t] = 0;
    for (int64_t t = tid; t < a.R; t += nth) {
        a.stop[t] = 0;
        a.amb[t] = 0;
        a.rep[t] = 0;
        a.final_it[t] = -1;
        a.capprox[t] = INFINITY;
        a.changed[t] = 0;
        a.changed[a.R + t] = 0;
    }
    for (int64_t t = tid; t < kCtlSlots; t += nth) a.ctl[t] = 0;
}

__global__ void k_fl_sign(const double *x, int64_t n, int32_t *flags, unsigned long long *amax) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    int neg = 0, pos = 0, bad = 0;
    unsigned long long mx = 0;  // max |x| as bits (nonnegative doubles order like their bits)
    for (int64_t i = tid; i < n; i += nth) {
        const double v = x[i];
        neg |= v < 0.0 || (v == 0.0 && signbit(v));
        pos |= v > 0.0;
        bad |= !isfinite(v);
        const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(v));
        mx = b > mx ? b : mx;
    }
    neg = __any_sync(0xffffffffu, neg);
    pos = __any_sync(0xffffffffu, pos);
    bad = __any_sync(0xffffffffu, bad);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long ob = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = ob > mx ? ob : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        if (neg) atomicOr(flags, 1);
        if (pos) atomicOr(flags, 2);
        if (bad) atomicOr(flags, 4);
        atomicMax(amax, mx);
    }
}

__global__ void k_fl_negate(const double *x, int64_t n, double *out) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t i = tid; i < n; i += (int64_t)gridDim.x * blockDim.x) out[i] = -x[i];
}

// ---------------------------------------------------------------------------------------
// host side

struct FusedLloyd {
    int device = -1;
    int64_t n = 0;
    int sign = 0;  // +1 all >= 0 (no -0.0), -1 all <= 0, 0 mixed / unusable
    double xmax = 0.0;
    double *xneg = nullptr;
    int grid = 0;
    void *buf = nullptr;
    size_t buf_bytes = 0;
    int32_t *h_ctl = nullptr;  // pinned
};

static size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

void fused_lloyd_free(FusedLloyd *f) {
    if (!f) return;
    if (f->xneg) cudaFree(f->xneg);
    if (f->buf) cudaFree(f->buf);
    if (f->h_ctl) cudaFreeHost(f->h_ctl);
    delete f;
}

bool fused_lloyd_eligible(int l, int k, int R, int64_t n) {
    return l == 1 && k >= 1 && k <= kFlMaxK && R >= 1 && R <= kFlMaxR && R * k <= kFlMaxRK &&
           n >= 1 && n < (int64_t(1) << 31) && getenv("SC_KMEANS_NO_FUSED") == nullptr;
}

// returns SC_OK, an error, or 1 = "not applicable" (mixed signs): the caller runs the
// general path
int32_t fused_lloyd(FusedLloyd **pctx, int device, int sm_count, cudaStream_t s, const double *d_x,
                    int64_t n, int k, int R, const int64_t *d_chosen, int max_iters, double tol,
                    int64_t *labels_out, double *costs_out, int32_t *iters_out, int32_t *best_out) {
    if (!*pctx) {
        FusedLloyd *f = new FusedLloyd();
        f->device = device;
        f->n = n;
        SC_CUDA(cudaMallocHost((void **)&f->h_ctl, 64));
        int32_t *d_flags = nullptr;
        SC_CUDA(cudaMallocAsync((void **)&d_flags, 16, s));
        SC_CUDA(cudaMemsetAsync(d_flags, 0, 16, s));
        k_fl_sign<<<sm_count * 4, 256, 0, s>>>(d_x, n, d_flags,
                                               reinterpret_cast<unsigned long long *>(d_flags + 2));
        SC_CUDA(cudaMemcpyAsync(f->h_ctl, d_flags, 16, cudaMemcpyDeviceToHost, s));
        SC_CUDA(cudaFreeAsync(d_flags, s));
        SC_CUDA(cudaStreamSynchronize(s));
        const int fl = f->h_ctl[0];
        f->sign = (fl & 4) ? 0 : (fl & 1) && (fl & 2) ? 0 : (fl & 1) ? -1 : 1;
        memcpy(&f->xmax, f->h_ctl + 2, 8);
        if (f->sign < 0) {
            SC_CUDA(cudaMalloc((void **)&f->xneg, (size_t)n * 8));
            k_fl_negate<<<sm_count * 4, 256, 0, s>>>(d_x, n, f->xneg);
        }
        int per = 0;
        SC_CUDA(cudaFuncSetAttribute(k_fused_lloyd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kFlDynSmem));
        SC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_fused_lloyd, kFlThreads,
                                                              kFlDynSmem));
        f->grid = std::max(1, std::min(per, 2)) * sm_count;
        *pctx = f;
    }
    FusedLloyd *f = *pctx;
    if (f->sign == 0) return 1;
    const int64_t nch = (n + kFlChunk - 1) / kFlChunk;
    const int64_t nbuf = (n + kFlEinsumBuf - 1) / kFlEinsumBuf;
    const size_t rk = (size_t)R * k;
    // one allocation, carved
    size_t off = 0;
    auto carve = [&](size_t bytes) {
        const size_t o = off;
        off += align_up(bytes);
        return o;
    };
    const int64_t ln = nch * kFlChunk;
    const size_t o_lab = carve((size_t)3 * R * ln), o_cen = carve(3 * rk * 8),
                 o_A = carve(rk * nch * 8), o_cnt = carve(rk * nch * 4), o_pred = carve(rk * nch * 4),
                 o_M = carve(rk * nch * 16), o_MC = carve(rk * nch * 32), o_AS = carve(rk * nch * 8),
                 o_cpart = carve((size_t)R * nch * 8),
                 o_tot = carve(rk * 4), o_chg = carve((size_t)2 * R * 4), o_ctl = carve(kCtlSlots * 4),
                 o_stop = carve(R * 4), o_amb = carve(R * 4), o_rep = carve(R * 4),
                 o_fin = carve(R * 4), o_cap = carve(R * 8), o_cfr = carve(R * 8),
                 o_bp = carve((size_t)2 * R * nbuf * 8), o_cex = carve(R * 8), o_own = carve((size_t)n * 8),
                 o_gv = carve((size_t)f->grid * 8), o_gi = carve((size_t)f->grid * 8);
    if (off > f->buf_bytes) {
        if (f->buf) cudaFreeAsync(f->buf, s);
        f->buf = nullptr;
        f->buf_bytes = 0;
        SC_CUDA(cudaMallocAsync(&f->buf, off, s));
        f->buf_bytes = off;
    }
    unsigned char *B = static_cast<unsigned char *>(f->buf);
    FlArgs a;
    a.x = f->sign < 0 ? f->xneg : d_x;
    a.n = n;
    a.ln = ln;
    a.k = k;
    a.R = R;
    a.nch = (int)nch;
    a.max_iters = max_iters;
    a.nbuf = nbuf;
    a.tol = tol;
    a.delta = 2.0 * (double)(4097 + nbuf + 64 + nch / 32) * 1.1102230246251565e-16;
    a.lab = B + o_lab;
    a.cen = reinterpret_cast<double *>(B + o_cen);
    a.A = reinterpret_cast<double *>(B + o_A);
    a.cnt = reinterpret_cast<int32_t *>(B + o_cnt);
    a.pred = reinterpret_cast<int32_t *>(B + o_pred);
    a.M = reinterpret_cast<int64_t *>(B + o_M);
    a.MC = reinterpret_cast<int64_t *>(B + o_MC);
    a.AS = reinterpret_cast<double *>(B + o_AS);
    a.xmax = f->xmax;
    a.cpart = reinterpret_cast<double *>(B + o_cpart);
    a.tot = reinterpret_cast<int32_t *>(B + o_tot);
    a.changed = reinterpret_cast<int32_t *>(B + o_chg);
    a.ctl = reinterpret_cast<int32_t *>(B + o_ctl);
    a.stop = reinterpret_cast<int32_t *>(B + o_stop);
    a.amb = reinterpret_cast<int32_t *>(B + o_amb);
    a.rep = reinterpret_cast<int32_t *>(B + o_rep);
    a.final_it = reinterpret_cast<int32_t *>(B + o_fin);
    a.capprox = reinterpret_cast<double *>(B + o_cap);
    a.cfresh = reinterpret_cast<double *>(B + o_cfr);
    a.bpart = reinterpret_cast<double *>(B + o_bp);
    a.cexact = reinterpret_cast<double *>(B + o_cex);
    a.own = reinterpret_cast<double *>(B + o_own);
    a.gval = reinterpret_cast<double *>(B + o_gv);
    a.gidx = reinterpret_cast<int64_t *>(B + o_gi);
    const bool prof = getenv("SC_KMEANS_PROFILE") != nullptr;
    a.tprof = nullptr;
    if (prof) {
        SC_CUDA(cudaMallocAsync((void **)&a.tprof, 256 * 8 * 8, s));
        SC_CUDA(cudaMemsetAsync(a.tprof, 0, 256 * 8 * 8, s));
    }
    k_fl_init<<<f->grid, 256, 0, s>>>(a, d_x, f->sign < 0 ? -1.0 : 1.0, d_chosen);
    SC_CUDA(cudaGetLastError());
    void *args[] = {&a};
    SC_CUDA(cudaLaunchCooperativeKernel((const void *)k_fused_lloyd, f->grid, kFlThreads, args,
                                        kFlDynSmem, s));
    // results: control block, per-restart final iterations and exact costs, best labels
    SC_CUDA(cudaMemcpyAsync(f->h_ctl, a.ctl, kCtlSlots * 4, cudaMemcpyDeviceToHost, s));
    std::vector<int32_t> fin(R);
    std::vector<double> cex(R);
    SC_CUDA(cudaMemcpyAsync(fin.data(), a.final_it, R * 4, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaMemcpyAsync(cex.data(), a.cexact, R * 8, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaStreamSynchronize(s));
    if (prof) {
        std::vector<unsigned long long> tp(256 * 8);
        SC_CUDA(cudaMemcpy(tp.data(), a.tprof, tp.size() * 8, cudaMemcpyDeviceToHost));
        SC_CUDA(cudaFree(a.tprof));
        double acc[6] = {0, 0, 0, 0, 0, 0};
        const int its = f->h_ctl[kCtlIters];
        for (int i = 0; i <= its && i < 255; ++i)
            for (int q = 1; q < 6; ++q)
                if (tp[i * 8 + q] && tp[i * 8 + q - 1]) acc[q] += (tp[i * 8 + q] - tp[i * 8 + q - 1]) * 1e-3;
        fprintf(stderr, "[fused_lloyd] n=%lld k=%d R=%d grid=%d iterations %d: P1 %.1f us, P2 %.1f, "
                "exact/decide %.1f, P3 %.1f, P4 %.1f; final costs %.1f us; total %.1f us\n",
                (long long)n, k, R, f->grid, its, acc[1], acc[2], acc[3], acc[4], acc[5],
                (tp[255 * 8 + 1] - tp[255 * 8]) * 1e-3, (tp[255 * 8 + 1] - tp[0]) * 1e-3);
    }
    if (f->h_ctl[kCtlErr])
        return fail(SC_E_INTERNAL, "k-means cost increased (restart %d, iteration %d)",
                    f->h_ctl[kCtlErr] - 1, f->h_ctl[kCtlErrIt]);
    const int best = f->h_ctl[kCtlBest];
    SC_REQUIRE(best >= 0 && best < R, SC_E_INTERNAL, "no restart produced a finite cost");
    std::vector<uint8_t> lab8((size_t)n);
    SC_CUDA(cudaMemcpyAsync(lab8.data(), a.lab + ((size_t)(fin[best] % 3) * R + best) * ln, (size_t)n,
                            cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < n; ++i) labels_out[i] = lab8[(size_t)i];
    if (costs_out)
        for (int r = 0; r < R; ++r) costs_out[r] = cex[r];
    if (iters_out)
        for (int r = 0; r < R; ++r) iters_out[r] = fin[r] + 1;
    if (best_out) *best_out = best;
    return SC_OK;
}

}  // namespace sc
