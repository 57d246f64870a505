// sc_kmeans_fused.cu -- the exact restarted Lloyd (specluster/kmeans.py:167-215) for 1-D
// points of one sign and k <= 32, every iteration of every restart inside ONE persistent
// cooperative kernel: no host round trip, no sort, two grid barriers per iteration.
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
// Assignment.  Per restart the distinct centres are sorted; around each midpoint a band of
// half-width 8 u M^2 / gap bounds where the rounding of d2ref can decide (CenTab below).  A
// point outside every band takes its interval's centre with integer compares only; inside a
// band the two neighbours are evaluated with d2ref.
//
// Exact means without sorting.  Points are cut into chunks of 1024 consecutive indices.
// Inside one binade of the running sum every double is a multiple of its ulp u, so
// fl(s + a) = s + u * rne(a / u): a point acts on S = s/u as a translation by q or q+1
// (sc_seqsum.cuh "parity map"), except on an exact tie (a/u = q + 1/2), where the result is
// the even neighbour.  Per iteration:
//   P1   one warp per (restart, chunk): assignment, the cost terms of the previous
//        iteration, per cluster the count and an approximate sum, and -- for every cluster
//        whose running sum the previous iteration predicted to stay in one binade across the
//        chunk -- the chunk's parity map on that grid: the plain sum of the translations, or
//        an index-ordered composition if a tie occurs.  Lanes take points 32 apart, so every
//        load is coalesced and the chunk is staged by cp.async.
//   P24  one warp per (restart, cluster): an approximate prefix over the chunks gives the
//        binade predictions for the next iteration, and the EXACT walk over the chunks runs
//        alongside: maximal runs of chunks mapped on the running sum's grid advance with one
//        composed map (verified: the result must stay below the binade's top, which for a
//        monotone sum proves no intermediate left it); any other chunk holding the cluster
//        is added element by element from a staged tile (lanes own runs of 32; a run whose
//        predicted binade is the running one advances by its map, a run holding a crossing
//        adds its points one by one).  The walk writes the cluster's mean.
//   Predictions only choose between these paths; every bit comes from a verified step.  The
//   points are of one sign (x < 0 inputs run on -x: d2ref, the sums and the cost commute
//   with exact negation), so running sums are monotone.
//
// Stop decisions without the einsum chain.  The reference's cost is a sum of the terms
// t_i = fl(fl(x_i - mu)^2) in numpy's einsum order: chains of <= 4096 dependent adds per
// 8192-element buffer, then one add per buffer.  Each iteration computes instead C~, the same
// terms summed in a fixed tree order, and the proven bound |C - C~| <= delta * C~ with
// delta = 2 * (4097 + nbuf + depth(tree)) * 2^-53 (sums of the same nonnegative terms; each
// term passes through at most that many roundings).  The stop rule
// (fl(P - C) <= fl(tol * max(P, 1e-300))) and the assertion are evaluated on intervals; only
// if an interval straddles the threshold are the exact einsum-order costs of that iteration
// and of the previous one computed (same kernel, all warps).  Unchanged labels stop without a
// cost (kmeans.py:201,208), and then C == P exactly.  The costs that pick the best restart are
// always the exact einsum-order values.
//
// Speculation.  P1 of iteration it+1 also accumulates the cost terms of iteration it (the
// same pass reads x, the labels of it and the means of it), so the stop decision for it is
// taken in P24 of it+1; a restart that stops ignores the work it did for it+1.  Labels and
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
constexpr int kFlLane = 32;     // points per lane
constexpr int kFlMaxK = 32;
constexpr int kFlMaxR = 64;
constexpr int kFlMaxRK = 512;
constexpr int kFlThreads = 256;
constexpr int kFlWarps = kFlThreads / 32;
constexpr int kFlEinsumBuf = 8192;
constexpr int kSkip = kNoGrid + 1;  // chunk holds no element of the cluster
constexpr int kFlStage = 256;       // exact-cost staging window per warp
constexpr int kXsPitch = 33;        // padded tile: lane t's run of 32 at xs[t * 33 + q]
constexpr int kXsWarp = 32 * kXsPitch;
constexpr int kTileBytes = kXsWarp * 8 + kFlChunk;  // x tile + label tile, per warp (>= 12 * 32 * k)
// per-warp dynamic shared memory: the staging tile, or P1's accumulators (12 B per cluster
// and lane)
__host__ __device__ constexpr int fl_warp_bytes(int k) {
    return ((kTileBytes > 12 * 32 * k ? kTileBytes : 12 * 32 * k) + 15) / 16 * 16;
}

constexpr int kCrossTag = 1 << 20;  // pred = kCrossTag + grid: one binade crossing predicted
__device__ __forceinline__ bool is_cross(int p) { return p >= kCrossTag / 2; }
__device__ __forceinline__ bool is_grid(int p) { return p > kSkip && p < kCrossTag / 2; }

// control block (int32 slots)
enum : int {
    kCtlAmb = 0,      // some restart needs the exact costs of its last two iterations
    kCtlRepair = 1,   // some restart has an empty cluster after assignment
    kCtlErr = 2,      // cost assertion failed (kmeans.py:206): restart + 1
    kCtlErrIt = 3,
    kCtlIters = 4,    // iterations executed by the kernel
    kCtlBest = 5,
    kCtlNCross = 6,   // diagnostics: chunks added element by element
    kCtlNTie = 7,     // diagnostics: chunk maps composed in index order (ties)
    kCtlNX = 8,       // queued crossing records of the current iteration
    kCtlSlots = 12
};

struct FlArgs {
    const double *x;  // [n] points, all >= 0
    int64_t n;
    int64_t ln;       // label row stride (n rounded up to a chunk)
    int k, R, nch, max_iters;
    int64_t nbuf;
    int wd;            // doubles of dynamic shared memory per warp
    double tol, delta;
    int assert_cost;   // kmeans.py:206's assert (0: SC_KM_NO_COST_ASSERT, python -O)
    double xmax;       // max point value (rounding bands of the sorted-centre assignment)
    uint8_t *lab;      // [3][R][ln]
    double *cen;       // [3][R][k]
    double *A;         // [R][k][nch] approximate chunk sums
    int32_t *cnt;      // [R][k][nch]
    int32_t *pred2;    // [2][R][k][nch] per iteration parity: grid, kCrossTag + grid, kNoGrid, kSkip
    int32_t *chg;      // [R][nch] labels changed in the chunk by the assignment of it
    double *sfirst;    // [R][k] exact running sum after the cluster's first chunk
    double *AS;        // [R][k][nch] approximate running sum at each chunk start
    int64_t *M;        // [R][k][nch] packed parity maps (before the crossing, if any)
    int64_t *MC;       // [R][k][nch][2] crossing records: packed map after, crossing value
    uint32_t *xlist;   // [R*k*nch] queued crossing records (c << 11 | r << 5 | j)
    int32_t *rng;      // [R][k][2] first and last chunk holding the cluster
    int nbat;          // batches of 32 chunks
    int64_t *PP, *SS;  // [R][k][nch] packed prefix / suffix compositions inside the batch
    int32_t *BG;       // [R][k][nbat] batch grid (kSkip / kNoGrid if not uniform)
    int64_t *BM;       // [R][k][nbat] packed composition of the batch
    double *cpart;     // [R][nch] approximate cost partials
    int32_t *tot;      // [2][R][k] cluster sizes of even / odd iterations (atomics)
    int32_t *changed;  // [2][R]
    int32_t *ctl;      // kCtlSlots
    int32_t *stop;     // [R] sticky: restart finished
    int32_t *amb;      // [R]
    int32_t *rep;      // [R]
    int32_t *final_it; // [R]
    double *capprox;   // [R] cost of the previous decided iteration (C~ or exact)
    double *bpart;     // [2][R][nbuf] exact cost buffer partials
    double *cexact;    // [R] exact final costs
    double *own;       // [n] repair scratch
    double *gval;      // [grid] argmax partials
    int64_t *gidx;
    unsigned long long *tprof;  // optional phase timestamps [256][8] (SC_KMEANS_PROFILE)
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ uint8_t *lab_buf(const FlArgs &a, int it, int r) {
    return a.lab + ((size_t)(((it % 3) + 3) % 3) * a.R + r) * a.ln;
}
__device__ __forceinline__ int32_t *pred_buf(const FlArgs &a, int it) {
    return a.pred2 + (size_t)(it & 1) * a.R * a.k * a.nch;
}
__device__ __forceinline__ int32_t *tot_buf(const FlArgs &a, int it) {
    return a.tot + (size_t)(it & 1) * a.R * a.k;
}
__device__ __forceinline__ double *cen_buf(const FlArgs &a, int it, int r) {
    return a.cen + ((size_t)(it % 3) * a.R + r) * a.k;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
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

// fixed-order warp sums (the xor butterfly gives every lane the same bits)
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
__device__ __forceinline__ long long warp_lsum(long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// the labels of a lane's 32 points, packed 4 per word (indices are compile-time in the
// unrolled loops, so this lives in registers)
struct Lab32 {
    uint32_t w[8];
    __device__ __forceinline__ int get(int t) const { return (w[t >> 2] >> (8 * (t & 3))) & 0xff; }
    __device__ __forceinline__ void set(int t, int v) {
        w[t >> 2] = (w[t >> 2] & ~(0xffu << (8 * (t & 3)))) | ((uint32_t)v << (8 * (t & 3)));
    }
};

// The running sum s on its own grid k = grid_of(s).k: S = s / u is the significand (with the
// implicit bit; for k = 1074 the subnormal range and the first normal binade share the ulp
// 2^-1074, and S is the raw bit pattern).  Pure integer work on the walk's critical path.
__device__ __forceinline__ int64_t run_units(double s, int k) {
    return (int64_t)__double_as_longlong(s) - ((int64_t)(1074 - k) << 52);
}
__device__ __forceinline__ double run_from(int64_t S, int k) {  // S inside the grid's binade
    return __longlong_as_double(((int64_t)(1074 - k) << 52) + S);
}
// a point on grid k (k in [-971, 1074]): x * 2^k by exact power-of-two multiplications
__device__ __forceinline__ double elem_units(double x, int k) {
    if (k <= 1000) return __dmul_rn(x, __longlong_as_double((int64_t)(1023 + k) << 52));
    return __dmul_rn(__dmul_rn(x, __longlong_as_double((int64_t)(23 + k) << 52)),
                     __longlong_as_double((int64_t)(1023 + 1000) << 52));
}

// A chunk map (i0, i1) has |i1 - i0| <= 1 (after the first tie both parities of the start
// give an even value), so it packs into one word: i0 << 2 | (i1 - i0 + 1).
__device__ __forceinline__ int64_t pack_map(PMap m) { return (m.i0 << 2) | (m.i1 - m.i0 + 1); }
__device__ __forceinline__ PMap unpack_map(int64_t v) {
    const int64_t i0 = v >> 2;
    return PMap{i0, i0 + (v & 3) - 1};
}

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
    uint8_t *spos;             // [R*k] sorted position of each centre id's value
    unsigned long long *bl, *bh;  // band bounds (bits), kd-1 per restart
    int *kd;                   // distinct count, or -1: brute force
    unsigned long long *flo, *fhi;  // [R*k] by centre id: the safe interior of its interval
    uint8_t *flab;             // [R*k] by centre id: the label of that interval
};

// labels of points still inside the safe interior of their previous label's interval, or -1
__device__ __forceinline__ int assign_fast(const CenTab &T, int r, int k, double xv, int prev) {
    const unsigned long long xb = (unsigned long long)__double_as_longlong(xv);
    const int o = r * k + prev;
    return (xb > T.flo[o] && xb < T.fhi[o]) ? (int)T.flab[o] : -1;
}

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
        for (int q = j; q < k; ++q)  // every id with this value
            if (T.cen[r * k + q] == c) T.spos[r * k + q] = (uint8_t)rank;
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
    for (int t = threadIdx.x; t < rk; t += blockDim.x) {
        const int r = t / k;
        const int kd = T.kd[r];
        if (kd < 1) {
            T.flo[t] = ~0ull;  // never hits
            T.fhi[t] = 0ull;
            T.flab[t] = 0;
            continue;
        }
        const int pos = T.spos[t];
        T.flo[t] = pos > 0 ? T.bh[r * k + pos - 1] : 0ull;
        T.fhi[t] = pos < kd - 1 ? T.bl[r * k + pos] : ~0ull;
        T.flab[t] = T.sid[r * k + pos];
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------------------
// P1 for one (restart r, chunk c).  assign: new labels of iteration it.  resum: the labels of
// it are read back (after a repair).  cost: the C~ terms of iteration it-1.  Lanes take points
// 32 apart (coalesced loads, streamed 8 deep); per-cluster counts and approximate sums
// accumulate per lane in shared memory (acc[j][lane]) and are reduced per present cluster.
struct P1Mode {
    bool assign, resum, cost;
};

__device__ void p1_task(const FlArgs &a, int it, int r, int c, P1Mode md, const CenTab &T,
                        double *tile) {
    const int lane = lane_id(), k = a.k;
    const int64_t base = (int64_t)c * kFlChunk;
    const bool summ = md.assign || md.resum;
    double *accS = tile;
    int *accC = reinterpret_cast<int *>(tile + k * 32);
    if (summ)
        for (int j = 0; j < k; ++j) {
            accS[j * 32 + lane] = 0.0;
            accC[j * 32 + lane] = 0;
        }
    __syncwarp();
    const double *cr = T.cen + r * k;
    const uint8_t *lp = lab_buf(a, it + 2, r) + base;
    uint8_t *lc = lab_buf(a, it, r) + base;
    double csum = 0.0;
    int nchg = 0;
    uint32_t mask = 0, miss = 0;
    // points and labels of 8 steps in registers, the next 8 loading while these are processed
    double xn[8];
    int pn[8], cn8[8];
    auto load8 = [&](int g) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = 32 * (8 * g + u) + lane;
            const bool v = base + e < a.n;
            xn[u] = v ? __ldg(a.x + base + e) : 0.0;
            pn[u] = v ? (int)__ldcg(lp + e) : 0;
            cn8[u] = v && md.resum ? (int)__ldcg(lc + e) : 0;
        }
    };
    load8(0);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        double xc[8];
        int pc[8], cc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            xc[u] = xn[u];
            pc[u] = pn[u];
            cc[u] = cn8[u];
        }
        if (g < 3) load8(g + 1);
        int fast[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) fast[u] = md.assign ? assign_fast(T, r, k, xc[u], pc[u]) : cc[u];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int q = 8 * g + u;
            const int e = 32 * q + lane;
            if (base + e < a.n) {
                const double xv = xc[u];
                const int pl = pc[u];
                if (md.cost) {
                    const double d = __dsub_rn(xv, cr[pl]);
                    csum = __dadd_rn(csum, __dmul_rn(d, d));
                }
                if (summ) {
                    const int lb = fast[u];
                    if (lb < 0) {  // searched after the loop, so lanes do not diverge here
                        miss |= 1u << q;
                        continue;
                    }
                    if (md.assign) lc[e] = (uint8_t)lb;
                    nchg += lb != pl;
                    mask |= 1u << lb;
                    accS[lb * 32 + lane] += xv;
                    accC[lb * 32 + lane] += 1;
                }
            }
        }
    }
    while (miss) {  // the points that left the safe interior of their previous label's interval
        const int q = __ffs(miss) - 1;
        miss &= miss - 1;
        const int e = 32 * q + lane;
        const double xv = __ldg(a.x + base + e);
        const int pl = __ldcg(lp + e);
        const int lb = assign_one(T, r, k, xv);
        lc[e] = (uint8_t)lb;
        nchg += lb != pl;
        mask |= 1u << lb;
        accS[lb * 32 + lane] += xv;
        accC[lb * 32 + lane] += 1;
    }
    if (md.cost) {
        csum = warp_sum(csum);
        if (lane == 0) __stcg(a.cpart + (size_t)r * a.nch + c, csum);
    }
    if (!summ) return;
    __syncwarp();
    uint32_t wm = mask;
#pragma unroll
    for (int o = 16; o; o >>= 1) wm |= __shfl_xor_sync(0xffffffffu, wm, o);
    const size_t ob = (size_t)r * k * a.nch + c;  // + j * nch
    if (lane < k && !((wm >> lane) & 1u)) {
        __stcg(a.A + ob + (size_t)lane * a.nch, 0.0);
        __stcg(a.cnt + ob + (size_t)lane * a.nch, 0);
    }
    for (uint32_t b = wm; b; b &= b - 1) {
        const int j = __ffs(b) - 1;
        const double sj = warp_sum(accS[j * 32 + lane]);
        const int cj = warp_isum(accC[j * 32 + lane]);
        if (lane == 0) {
            __stcg(a.A + ob + (size_t)j * a.nch, sj);
            __stcg(a.cnt + ob + (size_t)j * a.nch, cj);
            atomicAdd(tot_buf(a, it) + (size_t)r * k + j, cj);
        }
    }
    nchg = warp_isum(nchg);
    if (lane == 0) {
        if (nchg) atomicAdd(a.changed + (it % 3) * a.R + r, nchg);
        __stcg(a.chg + (size_t)r * a.nch + c, nchg);
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------------------
// P2 for one (r, j): approximate prefix over the chunks -> per chunk the binade the exact
// running sum is expected in (pred), or one predicted crossing into the next binade (pred =
// kCrossTag + grid; the pair is queued for a crossing record); the approximate start of each
// chunk (AS).
__device__ void p2_task(const FlArgs &a, int it, int r, int j) {
    const int lane = lane_id();
    int32_t *pred = pred_buf(a, it);
    const size_t base = ((size_t)r * a.k + j) * a.nch;
    const double lo_f = 1.0 - 1.0 / 1048576.0, hi_f = 1.0 + 1.0 / 1048576.0;
    double carry = 0.0;
    int first = a.nch, last = -1;
    constexpr int kU = 4;  // batches per group; the next group loads during this one
    double avn[kU];
    int cnn[kU];
    auto fetch = [&](int c00) {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int c = c00 + 32 * u + lane;
            avn[u] = c < a.nch ? __ldcg(a.A + base + c) : 0.0;
            cnn[u] = c < a.nch ? __ldcg(a.cnt + base + c) : 0;
        }
    };
    fetch(0);
    for (int c00 = 0; c00 < a.nch; c00 += 32 * kU) {
        double av[kU];
        int cn[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            av[u] = avn[u];
            cn[u] = cnn[u];
        }
        fetch(c00 + 32 * kU);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int c = c00 + 32 * u + lane;
            if (!__any_sync(0xffffffffu, cn[u] != 0)) {  // no point of the cluster in the batch
                if (c < a.nch) {
                    __stcg(pred + base + c, kSkip);
                    __stcg(a.AS + base + c, carry);
                }
                continue;
            }
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
                __stcg(pred + base + c, kp);
                __stcg(a.AS + base + c, st);
                if (is_cross(kp)) {
                    const int slot = atomicAdd(a.ctl + kCtlNX, 1);
                    a.xlist[slot] = ((uint32_t)c << 11) | ((uint32_t)r << 5) | (uint32_t)j;
                }
            }
            carry += __shfl_sync(0xffffffffu, incl, 31);
            const unsigned have = __ballot_sync(0xffffffffu, c < a.nch && cn[u] != 0);
            if (have) {
                first = min(first, c00 + 32 * u + __ffs(have) - 1);
                last = c00 + 32 * u + 31 - __clz(have);
            }
        }
    }
    if (lane == 0) {
        a.rng[2 * ((size_t)r * a.k + j)] = first;
        a.rng[2 * ((size_t)r * a.k + j) + 1] = last;
    }
}

// ---------------------------------------------------------------------------------------
// P3a for one (r, chunk): parity maps of the clusters predicted to stay in one binade across
// the chunk: each point's translation q or q+1 on the predicted grid, summed per lane and
// cluster in shared memory and reduced; a tie (a/u = q + 1/2) makes the parity matter, and
// then the cluster's map is composed in index order (q-major, lane-minor).
__device__ void p3a_task(const FlArgs &a, int it, int r, int c, int *spred, double *tile) {
    const int lane = lane_id(), k = a.k;
    const int64_t base = (int64_t)c * kFlChunk;
    const size_t ob = (size_t)r * k * a.nch + c;
    int32_t *pred = pred_buf(a, it);
    int pj = kSkip;
    bool keep = false;  // same points and same grid as the last iteration: the map stands
    if (lane < k && __ldcg(a.cnt + ob + (size_t)lane * a.nch)) {
        pj = __ldcg(pred + ob + (size_t)lane * a.nch);
        keep = it > 0 && __ldcg(a.chg + (size_t)r * a.nch + c) == 0 &&
               __ldcg(pred_buf(a, it - 1) + ob + (size_t)lane * a.nch) == pj;
    }
    const uint32_t want = __ballot_sync(0xffffffffu, lane < k && is_grid(pj) && !keep);
    if (!want) return;
    if (lane < k) spred[lane] = pj;
    long long *accQ = reinterpret_cast<long long *>(tile);
    for (uint32_t b = want; b; b &= b - 1) accQ[(__ffs(b) - 1) * 32 + lane] = 0;
    __syncwarp();
    const uint8_t *lc = lab_buf(a, it, r) + base;
    uint32_t tmask = 0, hmask = 0;  // clusters with a tie / with a point beyond the grid
    uint32_t oddq = 0, tieq = 0;    // per step q: translation parity, tie
    Lab32 L;
#pragma unroll
    for (int q = 0; q < 8; ++q) L.w[q] = 0xffffffffu;  // 255: no point
    double xn[8];
    int ln8[8];
    auto load8 = [&](int g) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = 32 * (8 * g + u) + lane;
            const bool v = base + e < a.n;
            xn[u] = v ? __ldg(a.x + base + e) : 0.0;
            ln8[u] = v ? (int)__ldcg(lc + e) : 255;
        }
    };
    load8(0);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        double xc[8];
        int lcu[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            xc[u] = xn[u];
            lcu[u] = ln8[u];
        }
        if (g < 3) load8(g + 1);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int q = 8 * g + u;
            const int lb = lcu[u];
            if (lb == 255) continue;
            L.set(q, lb);
            if ((want >> lb) & 1u) {
                // translation on the grid: q or q+1; on a tie d = q and the parity decides
                const double v = elem_units(xc[u], spred[lb]);
                int64_t d = 0;
                int tie = 0;
                if (!(v <= 4.5e15)) {
                    hmask |= 1u << lb;
                } else {
                    const double fl = floor(v);
                    const double f = v - fl;
                    d = (int64_t)fl + (f > 0.5);
                    tie = f == 0.5;
                }
                tmask |= (uint32_t)tie << lb;
                oddq |= (uint32_t)(d & 1) << q;
                tieq |= (uint32_t)tie << q;
                accQ[lb * 32 + lane] += d;
            }
        }
    }
    __syncwarp();
    uint32_t wt = tmask, wh = hmask;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        wt |= __shfl_xor_sync(0xffffffffu, wt, o);
        wh |= __shfl_xor_sync(0xffffffffu, wh, o);
    }
    for (uint32_t b = want; b; b &= b - 1) {
        const int j = __ffs(b) - 1;
        const size_t oj = ob + (size_t)j * a.nch;
        if ((wh >> j) & 1u) {  // a point beyond the predicted binade: the walk adds the chunk
            if (lane == 0) __stcg(pred + oj, kNoGrid);
            continue;
        }
        const long long D = warp_lsum(accQ[j * 32 + lane]);
        long long C0 = 0, C1 = 0;
        if ((wt >> j) & 1u) {
            // A tie maps S to the even one of S + q, S + q + 1, so it adds (S + q) & 1 and leaves
            // an even value.  Track the running parity from an even (0) and an odd (1) start in
            // index order (step-major, lane-minor) with ballots; only parities matter.
            if (lane == 0 && a.tprof) atomicAdd(a.ctl + kCtlNTie, 1);
            int cur0 = 0, cur1 = 1;
#pragma unroll
            for (int q = 0; q < kFlLane; ++q) {
                const bool in = L.get(q) == j;
                const unsigned tb = __ballot_sync(0xffffffffu, in && ((tieq >> q) & 1u));
                const unsigned ob2 = __ballot_sync(0xffffffffu, in && ((oddq >> q) & 1u) && !((tieq >> q) & 1u));
                if (!tb) {
                    const int pp = __popc(ob2) & 1;
                    cur0 ^= pp;
                    cur1 ^= pp;
                    continue;
                }
                const unsigned tq = __ballot_sync(0xffffffffu, in && ((tieq >> q) & 1u) && ((oddq >> q) & 1u));
                unsigned done = 0;
                for (unsigned t = tb; t; t &= t - 1) {
                    const int ln = __ffs(t) - 1;
                    const unsigned below = ((1u << ln) - 1u) & ~done;
                    const int pp = __popc(ob2 & below) & 1;
                    cur0 ^= pp;
                    cur1 ^= pp;
                    const int qp = (tq >> ln) & 1;
                    C0 += (cur0 + qp) & 1;
                    C1 += (cur1 + qp) & 1;
                    cur0 = cur1 = 0;  // the result of a tie is even
                    done = (ln == 31) ? 0xffffffffu : ((2u << ln) - 1u);
                }
                const int pp = __popc(ob2 & ~done) & 1;
                cur0 ^= pp;
                cur1 ^= pp;
            }
        }
        if (lane == 0) {
            if (D + 2 >= (int64_t(1) << 53)) __stcg(pred + oj, kNoGrid);  // cannot stay in a binade
            else __stcg(a.M + oj, pack_map(PMap{D + C0, D + C1}));
        }
    }
    __syncwarp();
}

// stage chunk c with lanes owning runs of 32 consecutive points: xs[t * 33 + q] and the run's
// label bytes at lb[32 t + q] (cp.async, zeros / no labels past n)
__device__ __forceinline__ void stage_runs(const FlArgs &a, int it, int r, int c, double *tile) {
    const int lane = lane_id();
    double *xs = tile;
    uint32_t *lb = reinterpret_cast<uint32_t *>(tile + kXsWarp);
    const int64_t base = (int64_t)c * kFlChunk;
    const uint32_t *src = reinterpret_cast<const uint32_t *>(lab_buf(a, it, r) + base);
    // coalesced loads, all 32 + 8 in flight, then the padded stores
    double v[32];
    uint32_t w[8];
    if (base + kFlChunk <= a.n) {
#pragma unroll
        for (int u = 0; u < 32; ++u) v[u] = __ldg(a.x + base + 32 * u + lane);
    } else {
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            const int64_t i = base + 32 * u + lane;
            v[u] = i < a.n ? __ldg(a.x + i) : 0.0;
        }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) w[u] = __ldcg(src + 32 * u + lane);
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 32; ++u) xs[u * kXsPitch + lane] = v[u];
#pragma unroll
    for (int u = 0; u < 8; ++u) lb[32 * u + lane] = w[u];
    __syncwarp();
}

// P3b for one queued (r, j, chunk) with a predicted crossing: the point whose add crosses into
// the next binade (found on an approximate running sum with a relative margin of 2^-24, else
// the chunk is left to the walk), the map of the points before it and the map after it.
__device__ void p3b_task(const FlArgs &a, int it, uint32_t item, double *tile) {
    const int lane = lane_id();
    const int j = item & 31, r = (item >> 5) & 63, c = (int)(item >> 11);
    if (__ldcg(a.stop + r)) return;
    const int k = a.k;
    const size_t o = ((size_t)r * k + j) * a.nch + c;
    int32_t *pred = pred_buf(a, it);
    const int p = __ldcg(pred + o);
    const double as0 = __ldcg(a.AS + o);
    stage_runs(a, it, r, c, tile);
    const int64_t i0 = (int64_t)c * kFlChunk + (int64_t)lane * kFlLane;
    const int m = (int)max((int64_t)0, min((int64_t)kFlLane, a.n - i0));
    const double *xr = tile + lane * kXsPitch;
    const uint8_t *lr = reinterpret_cast<const uint8_t *>(tile + kXsWarp) + lane * kFlLane;
    uint32_t bits = 0;
    double as = 0.0;
#pragma unroll
    for (int t = 0; t < kFlLane; ++t)
        if (t < m && lr[t] == j) {
            bits |= 1u << t;
            as += xr[t];
        }
    double incl = as;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double ov = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += ov;
    }
    const int g1 = p - kCrossTag, g2 = g1 - 1;
    const double B = scalbn(1.0, 53 - g1);  // bottom of the next binade
    const double mlo = 1.0 - 1.0 / 16777216.0, mhi = 1.0 + 1.0 / 16777216.0;
    const double st = as0 + (incl - as), en = as0 + incl;
    PMap m1 = pmap_id(), m2 = pmap_id();
    double ac = 0.0;
    int role;  // 0 before, 2 after, 1 holds the crossing, 3 undecidable
    if (!bits || en < B * mlo) role = 0;
    else if (st >= B * mhi) role = 2;
    else if (st < B * mlo) role = 1;
    else role = 3;
    if (role == 0) {
        for (uint32_t b = bits; b; b &= b - 1) m1 = pmap_then(m1, pmap_elem(elem_units(xr[__ffs(b) - 1], g1)));
    } else if (role == 2) {
        for (uint32_t b = bits; b; b &= b - 1) m2 = pmap_then(m2, pmap_elem(elem_units(xr[__ffs(b) - 1], g2)));
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
                m1 = pmap_then(m1, pmap_elem(elem_units(xv, g1)));
            } else {
                m2 = pmap_then(m2, pmap_elem(elem_units(xv, g2)));
            }
            rr = nr;
        }
        if (!phase) role = 3;
    }
    const unsigned holders = __ballot_sync(0xffffffffu, role == 1);
    m1 = warp_reduce_pmap(m1);
    m2 = warp_reduce_pmap(m2);
    const int64_t lim53 = int64_t(1) << 53;
    const bool ok = !__any_sync(0xffffffffu, role == 3) && __popc(holders) == 1 &&
                    __shfl_sync(0xffffffffu, (int)(m1.i0 >= 0 && m1.i0 < lim53 && m1.i1 >= 0 &&
                                                   m1.i1 < lim53 && m2.i0 >= 0 && m2.i0 < lim53 &&
                                                   m2.i1 >= 0 && m2.i1 < lim53), 0);
    const double acv = __shfl_sync(0xffffffffu, ac, holders ? __ffs(holders) - 1 : 0);
    if (lane == 0) {
        if (ok) {
            __stcg(a.M + o, pack_map(m1));
            __stcg(a.MC + 2 * o, pack_map(m2));
            __stcg(reinterpret_cast<double *>(a.MC) + 2 * o + 1, acv);
        } else {
            __stcg(pred + o, kNoGrid);  // the walk adds this chunk element by element
        }
    }
    __syncwarp();
}

// Exact addition of cluster j's points of chunk c to the running sum s (no usable record):
// lanes own runs of 32 consecutive points; each lane predicts the binade of its run from s plus
// an approximate prefix and builds its run's map; the warp then advances over maximal runs of
// lanes on the running sum's grid with one composed map, and adds a lane's run element by
// element where a crossing falls inside it.
__device__ __forceinline__ unsigned long long gtimer();
__device__ double cross_chunk_impl(const FlArgs &a, int it, int r, int j, int c, double s, double *tile);
__device__ double cross_chunk(const FlArgs &a, int it, int r, int j, int c, double s, double *tile) {
    const unsigned long long t0 = a.tprof ? gtimer() : 0;
    const double v = cross_chunk_impl(a, it, r, j, c, s, tile);
    if (a.tprof && lane_id() == 0) atomicAdd(a.tprof + 256 * 8 + 3, gtimer() - t0);
    return v;
}
__device__ double cross_chunk_impl(const FlArgs &a, int it, int r, int j, int c, double s, double *tile) {
    const int lane = lane_id();
    if (lane == 0 && a.tprof) atomicAdd(a.ctl + kCtlNCross, 1);
    stage_runs(a, it, r, c, tile);
    const int64_t i0 = (int64_t)c * kFlChunk + (int64_t)lane * kFlLane;
    const int m = (int)max((int64_t)0, min((int64_t)kFlLane, a.n - i0));
    const double *xr = tile + lane * kXsPitch;
    const uint8_t *lr = reinterpret_cast<const uint8_t *>(tile + kXsWarp) + lane * kFlLane;
    uint32_t bits = 0;
    double as = 0.0;
#pragma unroll
    for (int t = 0; t < kFlLane; ++t)
        if (t < m && lr[t] == j) {
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
        if (g != kNoGrid)
            for (uint32_t b = bits; b; b &= b - 1) lm = pmap_then(lm, pmap_elem(elem_units(xr[__ffs(b) - 1], g)));
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
            const int64_t S1 = pmap_apply(bm, run_units(s, gs.k));
            if (S1 < gs.top) {
                s = run_from(S1, gs.k);
                L = L2;
                continue;
            }
        }
        double v = s;  // lane L element by element (loads first, then the dependent adds)
        if (lane == L) {
            double xv[kFlLane];
#pragma unroll
            for (int t = 0; t < kFlLane; ++t) xv[t] = xr[t];
#pragma unroll
            for (int t = 0; t < kFlLane; ++t)
                if ((bits >> t) & 1u) v = __dadd_rn(v, xv[t]);
        }
        s = __shfl_sync(0xffffffffu, v, L);
        L += 1;
    }
    __syncwarp();
    return s;
}

// P3c for one (r, j): the cluster's first chunk, from the exact running value 0 (binade
// crossings at every doubling of the sum fall here), added off the walk's critical path
__device__ void p3c_task(const FlArgs &a, int it, int r, int j, double *tile) {
    const int c = __ldcg(a.rng + 2 * ((size_t)r * a.k + j));
    double s = 0.0;
    if (c < a.nch) s = cross_chunk(a, it, r, j, c, 0.0, tile);
    if (lane_id() == 0) __stcg(a.sfirst + (size_t)r * a.k + j, s);
}

// P4 for one (r, j): the exact walk over the chunks, 32 at a time with 4 batches of records in
// flight: maximal runs of chunks on the running sum's grid advance with one composed map, a
// predicted crossing with its two maps and one real add of the crossing point, anything else
// element by element (cross_chunk).  Every step is verified against the exact running value.
// Writes the cluster's mean for iteration it+1.
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// P3.5 for one (r, j, batch of 32 chunks): off the walk's critical path, the batch's common
// grid (when every chunk holding the cluster is mapped on one grid) with the composition of
// all its chunks, and per chunk the composition of the batch's chunks up to it (prefix) and
// from it to the batch end (suffix) -- the walk's runs start at a batch start or end at a batch
// end except between two crossings.
__device__ void p35_task(const FlArgs &a, int it, int r, int j, int b) {
    const int lane = lane_id();
    const size_t base = ((size_t)r * a.k + j) * a.nch;
    const int c = 32 * b + lane;
    const int32_t *pred = pred_buf(a, it);
    const int cfirst = __ldcg(a.rng + 2 * ((size_t)r * a.k + j));
    int p = kSkip;
    PMap m = pmap_id();
    if (c < a.nch && c > cfirst) {
        p = __ldcg(pred + base + c);
        if (is_grid(p)) m = unpack_map(__ldcg(a.M + base + c));
    }
    const unsigned have = __ballot_sync(0xffffffffu, p != kSkip);
    const int g0 = __shfl_sync(0xffffffffu, p, have ? __ffs(have) - 1 : 0);
    const bool uni = __all_sync(0xffffffffu, p == kSkip || (is_grid(p) && p == g0));
    // inclusive prefix (lane order) and suffix compositions
    PMap pre = m, suf = m;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        PMap o;
        o.i0 = __shfl_up_sync(0xffffffffu, pre.i0, d);
        o.i1 = __shfl_up_sync(0xffffffffu, pre.i1, d);
        if (lane >= d) pre = pmap_then(o, pre);
        PMap w;
        w.i0 = __shfl_down_sync(0xffffffffu, suf.i0, d);
        w.i1 = __shfl_down_sync(0xffffffffu, suf.i1, d);
        if (lane + d < 32) suf = pmap_then(suf, w);
    }
    if (c < a.nch) {
        __stcg(a.PP + base + c, pack_map(pre));
        __stcg(a.SS + base + c, pack_map(suf));
    }
    if (lane == 31) {
        const size_t ob = ((size_t)r * a.k + j) * a.nbat + b;
        __stcg(a.BG + ob, !have ? kSkip : (uni ? g0 : kNoGrid));
        __stcg(a.BM + ob, pack_map(pre));
    }
}

// P4 for one (r, j): the exact walk over the chunks.  Per batch of 32: on the running sum's grid
// in one step (P3.5's composition), else runs of mapped chunks with one prefix / suffix
// composition each, a predicted crossing with its two maps and one real add of the crossing
// point, anything else element by element (cross_chunk).  Every step is verified against the
// exact running value.  Writes the cluster's mean for iteration it+1.
__device__ void p4_task(const FlArgs &a, int it, int r, int j, double *tile) {
    const int lane = lane_id();
    const unsigned long long t_start = a.tprof ? gtimer() : 0;
    const size_t base = ((size_t)r * a.k + j) * a.nch;
    const size_t bb = ((size_t)r * a.k + j) * a.nbat;
    const int32_t *pred = pred_buf(a, it);
    const int cfirst = __ldcg(a.rng + 2 * ((size_t)r * a.k + j));
    const int clast = __ldcg(a.rng + 2 * ((size_t)r * a.k + j) + 1);
    double s = __ldcg(a.sfirst + (size_t)r * a.k + j);  // the first chunk was added in P3
    const int b_beg = (cfirst + 1) / 32, b_end = clast / 32 + 1;
    for (int b0 = b_beg; b0 < b_end; b0 += 32) {
        // batch summaries of up to 32 batches, one per lane
        const int bl = b0 + lane;
        const int bg_l = bl < b_end ? __ldcg(a.BG + bb + bl) : kSkip;
        const int64_t bm_l = bl < b_end ? __ldcg(a.BM + bb + bl) : 1;
        const int nb = min(32, b_end - b0);
        for (int q = 0; q < nb; ++q) {
            const int bg = __shfl_sync(0xffffffffu, bg_l, q);
            if (bg == kSkip) continue;
            {
                const Grid gs = grid_of(s);
                if (bg == gs.k) {
                    const int64_t S1 = pmap_apply(unpack_map(__shfl_sync(0xffffffffu, bm_l, q)), run_units(s, gs.k));
                    if (S1 < gs.top) {
                        s = run_from(S1, gs.k);
                        continue;
                    }
                }
            }
            // chunk by chunk inside batch b
            const int b = b0 + q;
            const int c0 = 32 * b, c = c0 + lane;
            const int lim = min(32, a.nch - c0);
            int p = kSkip;
            int64_t mw = 1, pp = 1, ss = 1, m2w = 1;
            double ac = 0.0;
            if (c < a.nch && c > cfirst) {
                p = __ldcg(pred + base + c);
                mw = __ldcg(a.M + base + c);
                pp = __ldcg(a.PP + base + c);
                ss = __ldcg(a.SS + base + c);
                m2w = __ldcg(a.MC + 2 * (base + c));
                ac = __ldcg(reinterpret_cast<const double *>(a.MC) + 2 * (base + c) + 1);
            }
            int L = 0;
            while (L < lim) {
                const Grid gs = grid_of(s);
                const bool ok = p == kSkip || p == gs.k;
                const unsigned badm = __ballot_sync(0xffffffffu, !ok && lane >= L && lane < lim);
                const int L2 = badm ? __ffs(badm) - 1 : lim;
                if (L2 > L) {
                    if (__any_sync(0xffffffffu, lane >= L && lane < L2 && p != kSkip)) {
                        PMap bm;
                        if (L == 0) {
                            bm = unpack_map(__shfl_sync(0xffffffffu, pp, L2 - 1));
                        } else if (L2 == lim) {
                            bm = unpack_map(__shfl_sync(0xffffffffu, ss, L));
                        } else {
                            PMap pm = (lane >= L && lane < L2 && p != kSkip) ? unpack_map(mw) : pmap_id();
                            pm = warp_reduce_pmap(pm);
                            bm = PMap{__shfl_sync(0xffffffffu, pm.i0, 0), __shfl_sync(0xffffffffu, pm.i1, 0)};
                        }
                        const int64_t S1 = pmap_apply(bm, run_units(s, gs.k));
                        if (S1 >= gs.top) {  // left the binade inside the run: first chunk by hand
                            s = cross_chunk(a, it, r, j, c0 + L, s, tile);
                            L += 1;
                            continue;
                        }
                        s = run_from(S1, gs.k);
                    }
                    L = L2;
                    continue;
                }
                // chunk L is off the running grid
                const int pL = __shfl_sync(0xffffffffu, p, L);
                bool done = false;
                if (is_cross(pL) && pL - kCrossTag == gs.k) {
                    const int64_t w1 = __shfl_sync(0xffffffffu, mw, L);
                    const int64_t w2 = __shfl_sync(0xffffffffu, m2w, L);
                    const double acl = __shfl_sync(0xffffffffu, ac, L);
                    const int g2l = gs.k - 1;
                    const int64_t S1 = pmap_apply(unpack_map(w1), run_units(s, gs.k));
                    if (S1 < gs.top) {
                        const double s2 = __dadd_rn(run_from(S1, gs.k), acl);
                        const Grid g2s = grid_of(s2);
                        if (g2s.k == g2l) {
                            const int64_t S2 = pmap_apply(unpack_map(w2), run_units(s2, g2l));
                            if (S2 < g2s.top) {
                                s = run_from(S2, g2l);
                                done = true;
                            }
                        }
                    }
                }
                if (!done) s = cross_chunk(a, it, r, j, c0 + L, s, tile);
                L += 1;
            }
        }
    }
    if (lane == 0) {
        const int t = __ldcg(tot_buf(a, it) + (size_t)r * a.k + j);
        __stcg(cen_buf(a, it + 1, r) + j, t > 0 ? __ddiv_rn(s, (double)t) : 0.0);
        if (a.tprof) {  // diagnostics: longest walk, latest walk end
            const unsigned long long t_end = gtimer();
            atomicMax(a.tprof + 256 * 8 + 0, t_end - t_start);
            atomicMax(a.tprof + 256 * 8 + 1, t_end - a.tprof[(size_t)min(it, 255) * 8 + 4]);
            atomicAdd(a.tprof + 256 * 8 + 2, t_end - t_start);
        }
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
// (kmeans.py:151-164).  Grid-uniform; the caller redoes the restart's chunk summaries.
__device__ void repair_restart(const FlArgs &a, cg::grid_group &grid, int it, int r, const CenTab &T) {
    const int k = a.k;
    uint8_t *lab = lab_buf(a, it, r);
    const double *cr = T.cen + r * k;
    // the empties, listed once (np.flatnonzero(counts == 0) before the loop)
    uint32_t empties = 0;
    for (int j = 0; j < k; ++j)
        if (__ldcg(tot_buf(a, it) + (size_t)r * k + j) == 0) empties |= 1u << j;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < a.n; i += nth) {
        const double xv = __ldg(a.x + i);
        const double cl = cr[__ldcg(lab + i)];
        const double xx = __dmul_rn(xv, xv), tx = __dmul_rn(2.0, xv);
        const double v = __dadd_rn(__dsub_rn(xx, __dmul_rn(tx, cl)), __dmul_rn(cl, cl));
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
    // fresh counters for the redone summaries
    if (blockIdx.x == 0 && threadIdx.x < k) tot_buf(a, it)[(size_t)r * k + threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.changed[(it % 3) * a.R + r] = 0;
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
    __shared__ uint8_t ssid[kFlMaxRK], sspos[kFlMaxRK], sflab[kFlMaxRK];
    __shared__ unsigned long long sflo[kFlMaxRK], sfhi[kFlMaxRK];
    __shared__ int skd[kFlMaxR];
    __shared__ int spred_all[kFlWarps][kFlMaxK];
    __shared__ int act[kFlMaxR];
    __shared__ int nact_s, any_s;
    extern __shared__ double fl_dyn[];  // per warp: a.wd doubles (tiles / accumulators)
    CenTab T{scen, ssv, ssid, sspos, sbl, sbh, skd, sflo, sfhi, sflab};
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int gw = blockIdx.x * kFlWarps + warp, nw = gridDim.x * kFlWarps;
    double *tile = fl_dyn + (size_t)warp * a.wd;
    int *spred = spred_all[warp];
    const int R = a.R, k = a.k, rk = R * k;
    auto load_active = [&]() {
        __syncthreads();
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
        // centres of iteration it (= means of it-1)
        for (int t = threadIdx.x; t < rk; t += blockDim.x) scen[t] = __ldcg(a.cen + (size_t)(it % 3) * rk + t);
        if (assign) build_tables(T, R, k, a.xmax);
        __syncthreads();
        const int nact = nact_s;
        // ---- P1: assignment of it, C~ terms of it-1
        {
            const P1Mode md{assign, false, cost};
            const unsigned long long w0 = a.tprof ? gtimer() : 0;
            int ntask = 0;
            for (int t = gw; t < nact * a.nch; t += nw, ++ntask) {
                const unsigned long long t0 = a.tprof ? gtimer() : 0;
                p1_task(a, it, act[t / a.nch], t % a.nch, md, T, tile);
                if (a.tprof && lane == 0) {
                    const unsigned long long dt = gtimer() - t0;
                    atomicAdd(a.tprof + 256 * 8 + 7, dt);
                    atomicMax(a.tprof + 256 * 8 + 8, dt);
                }
            }
            if (a.tprof && lane == 0) {
                atomicMax(a.tprof + 256 * 8 + 9, gtimer() - w0);
                atomicMax(a.tprof + 256 * 8 + 10, (unsigned long long)ntask);
                atomicMax(a.tprof + 256 * 8 + 11, gtimer() - a.tprof[(size_t)min(it, 255) * 8 + 0]);
            }
        }
        grid.sync();
        tmark(a, it, 1);
        // ---- empty clusters (rare): repair, then the restart's summaries again
        if (assign) {
            if (threadIdx.x == 0) {
                int any = 0;
                for (int q = 0; q < nact; ++q)
                    for (int j = 0; j < k; ++j) any |= __ldcg(tot_buf(a, it) + (size_t)act[q] * k + j) == 0;
                any_s = any;  // every block computes the same value
            }
            __syncthreads();
            if (any_s) {
                for (int q = 0; q < nact; ++q) {
                    const int r = act[q];
                    int emp = 0;
                    for (int j = 0; j < k; ++j) emp |= __ldcg(tot_buf(a, it) + (size_t)r * k + j) == 0;
                    if (!emp) continue;  // uniform: tot of r only changes inside its own repair
                    repair_restart(a, grid, it, r, T);
                    const P1Mode md{false, true, false};
                    for (int c = gw; c < a.nch; c += nw) p1_task(a, it, r, c, md, T, tile);
                    grid.sync();
                }
            }
        }
        // ---- P2: binade predictions of it; decision for it-1 (task index j == k)
        for (int t = gw; t < nact * (k + 1); t += nw) {
            const int r = act[t / (k + 1)], j = t % (k + 1);
            if (j < k) {
                if (assign) p2_task(a, it, r, j);
                if (j == 0 && lane == 0) a.changed[((it + 1) % 3) * R + r] = 0;
                if (lane == 0) tot_buf(a, it + 1)[(size_t)r * k + j] = 0;  // for P1 of it+1
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
            const bool unchanged = fin && __ldcg(a.changed + (d_it % 3) * R + r) == 0;
            int stop = 0, amb = 0;
            if (unchanged) {
                stop = 1;
            } else if (fin) {
                int bad = 0;
                const int sg = certify(P, cs, a.tol, a.delta, &bad);
                // (a sure failure is confirmed exactly; without the assert only the stop
                // decision matters: a cost increase stops, kmeans.py:207)
                if (sg < 0 || (a.assert_cost && bad != 0)) amb = 1;
                else stop = sg;
            }
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
            exact_partials(a, a.amb, it - 1, 0, tile, gw, nw);
            exact_partials(a, a.amb, it - 2, 1, tile, gw, nw);
            grid.sync();
            if (blockIdx.x == 0 && threadIdx.x < R) {
                const int r = threadIdx.x;
                if (a.amb[r]) {
                    const double C = exact_combine(a, 0, r), P = exact_combine(a, 1, r);
                    int bad = 0;
                    const int stop = decide_exact(P, C, a.tol, &bad);
                    if (bad && a.assert_cost) {
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
        load_active();
        if (!assign || nact_s == 0) break;
        tmark(a, it, 3);
        // ---- P3: chunk maps (a) and crossing records (b)
        {
            // the long first-chunk tasks first, then the crossing records, then the maps
            const int na = nact_s, nfirst = na * k, nsteady = na * a.nch;
            const int nx = __ldcg(a.ctl + kCtlNX);
            const unsigned long long w0 = a.tprof ? gtimer() : 0;
            for (int t = gw; t < nfirst + nx + nsteady; t += nw) {
                const unsigned long long t0 = a.tprof ? gtimer() : 0;
                int kind;
                if (t < nfirst) {
                    p3c_task(a, it, act[t / k], t % k, tile);
                    kind = 0;
                } else if (t < nfirst + nx) {
                    p3b_task(a, it, __ldcg(a.xlist + (t - nfirst)), tile);
                    kind = 1;
                } else {
                    p3a_task(a, it, act[(t - nfirst - nx) / a.nch], (t - nfirst - nx) % a.nch, spred, tile);
                    kind = 2;
                }
                if (a.tprof && lane == 0) {
                    const unsigned long long dt = gtimer() - t0;
                    atomicAdd(a.tprof + 258 * 8 + kind, dt);
                    atomicMax(a.tprof + 258 * 8 + 3 + kind, dt);
                    atomicAdd(a.tprof + 259 * 8 + kind, 1ull);
                }
            }
            if (a.tprof && lane == 0) atomicMax(a.tprof + 259 * 8 + 3, gtimer() - w0);
        }
        grid.sync();
        // ---- P3.5: batch compositions
        for (int t = gw; t < nact_s * k * a.nbat; t += nw) {
            const int rj = t / a.nbat;
            p35_task(a, it, act[rj / k], rj % k, t % a.nbat);
        }
        grid.sync();
        tmark(a, it, 4);
        // ---- P4: exact walks -> means of it
        for (int t = gw; t < nact_s * k; t += nw) p4_task(a, it, act[t / k], t % k, tile);
        if (blockIdx.x == 0 && threadIdx.x == 0) a.ctl[kCtlNX] = 0;
        grid.sync();
        tmark(a, it, 5);
    }
    tmark(a, 255, 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) a.ctl[kCtlIters] = it;
    if (__ldcg(a.ctl + kCtlErr)) return;
    // ---- exact final costs of every restart, best = first strictly smallest
    int32_t *all = a.amb;  // reused as "every restart" flags
    if (blockIdx.x == 0 && threadIdx.x < R) all[threadIdx.x] = 1;
    grid.sync();
    exact_partials(a, all, -1, 0, tile, gw, nw);
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
        a.changed[2 * a.R + t] = 0;
    }
    for (int64_t t = tid; t < kCtlSlots; t += nth) a.ctl[t] = 0;
    for (int64_t t = tid; t < 2 * rk; t += nth) a.tot[t] = 0;
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
                    bool assert_cost, int64_t *labels_out, double *costs_out, int32_t *iters_out,
                    int32_t *best_out) {
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
        *pctx = f;
    }
    FusedLloyd *f = *pctx;
    if (f->sign == 0) return 1;
    const int dyn = kFlWarps * fl_warp_bytes(k);
    {
        int per = 0;
        SC_CUDA(cudaFuncSetAttribute(k_fused_lloyd, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
        SC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_fused_lloyd, kFlThreads, dyn));
        SC_REQUIRE(per >= 1, SC_E_INTERNAL, "fused k-means kernel does not fit on an SM");
        f->grid = std::min(per, 2) * sm_count;
    }
    const int64_t nch = (n + kFlChunk - 1) / kFlChunk;
    const int64_t nbuf = (n + kFlEinsumBuf - 1) / kFlEinsumBuf;
    const int64_t nbat = (nch + 31) / 32;
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
                 o_A = carve(rk * nch * 8), o_cnt = carve(rk * nch * 4), o_p = carve(2 * rk * nch * 4), o_chg2 = carve((size_t)R * nch * 4), o_sf = carve(rk * 8),
                 o_AS = carve(rk * nch * 8), o_M = carve(rk * nch * 8), o_MC = carve(rk * nch * 16),
                 o_xl = carve(rk * nch * 4), o_rng = carve(rk * 8), o_PP = carve(rk * nch * 8), o_SS = carve(rk * nch * 8),
                 o_BG = carve(rk * nbat * 4), o_BM = carve(rk * nbat * 8),
                 o_cpart = carve((size_t)R * nch * 8), o_tot = carve(2 * rk * 4),
                 o_chg = carve((size_t)3 * R * 4), o_ctl = carve(kCtlSlots * 4),
                 o_stop = carve(R * 4), o_amb = carve(R * 4), o_rep = carve(R * 4),
                 o_fin = carve(R * 4), o_cap = carve(R * 8), o_bp = carve((size_t)2 * R * nbuf * 8),
                 o_cex = carve(R * 8), o_own = carve((size_t)n * 8), o_gv = carve((size_t)f->grid * 8),
                 o_gi = carve((size_t)f->grid * 8);
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
    a.wd = fl_warp_bytes(k) / 8;
    a.tol = tol;
    a.assert_cost = assert_cost ? 1 : 0;
    a.delta = 2.0 * (double)(4097 + nbuf + 64 + nch / 32) * 1.1102230246251565e-16;
    a.lab = B + o_lab;
    a.cen = reinterpret_cast<double *>(B + o_cen);
    a.A = reinterpret_cast<double *>(B + o_A);
    a.cnt = reinterpret_cast<int32_t *>(B + o_cnt);
    a.pred2 = reinterpret_cast<int32_t *>(B + o_p);
    a.chg = reinterpret_cast<int32_t *>(B + o_chg2);
    a.sfirst = reinterpret_cast<double *>(B + o_sf);
    a.AS = reinterpret_cast<double *>(B + o_AS);
    a.MC = reinterpret_cast<int64_t *>(B + o_MC);
    a.xlist = reinterpret_cast<uint32_t *>(B + o_xl);
    a.rng = reinterpret_cast<int32_t *>(B + o_rng);
    a.nbat = (int)nbat;
    a.PP = reinterpret_cast<int64_t *>(B + o_PP);
    a.SS = reinterpret_cast<int64_t *>(B + o_SS);
    a.BG = reinterpret_cast<int32_t *>(B + o_BG);
    a.BM = reinterpret_cast<int64_t *>(B + o_BM);
    a.M = reinterpret_cast<int64_t *>(B + o_M);
    a.cpart = reinterpret_cast<double *>(B + o_cpart);
    a.tot = reinterpret_cast<int32_t *>(B + o_tot);
    a.changed = reinterpret_cast<int32_t *>(B + o_chg);
    a.ctl = reinterpret_cast<int32_t *>(B + o_ctl);
    a.stop = reinterpret_cast<int32_t *>(B + o_stop);
    a.amb = reinterpret_cast<int32_t *>(B + o_amb);
    a.rep = reinterpret_cast<int32_t *>(B + o_rep);
    a.final_it = reinterpret_cast<int32_t *>(B + o_fin);
    a.capprox = reinterpret_cast<double *>(B + o_cap);
    a.bpart = reinterpret_cast<double *>(B + o_bp);
    a.cexact = reinterpret_cast<double *>(B + o_cex);
    a.own = reinterpret_cast<double *>(B + o_own);
    a.gval = reinterpret_cast<double *>(B + o_gv);
    a.xmax = f->xmax;
    a.gidx = reinterpret_cast<int64_t *>(B + o_gi);
    const bool prof = getenv("SC_KMEANS_PROFILE") != nullptr;
    a.tprof = nullptr;
    if (prof) {
        SC_CUDA(cudaMallocAsync((void **)&a.tprof, 260 * 8 * 8, s));
        SC_CUDA(cudaMemsetAsync(a.tprof, 0, 260 * 8 * 8, s));
    }
    k_fl_init<<<f->grid, 256, 0, s>>>(a, d_x, f->sign < 0 ? -1.0 : 1.0, d_chosen);
    SC_CUDA(cudaGetLastError());
    void *args[] = {&a};
    SC_CUDA(cudaLaunchCooperativeKernel((const void *)k_fused_lloyd, f->grid, kFlThreads, args,
                                        dyn, s));
    // results: control block, per-restart final iterations and exact costs, best labels
    SC_CUDA(cudaMemcpyAsync(f->h_ctl, a.ctl, kCtlSlots * 4, cudaMemcpyDeviceToHost, s));
    std::vector<int32_t> fin(R);
    std::vector<double> cex(R);
    SC_CUDA(cudaMemcpyAsync(fin.data(), a.final_it, R * 4, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaMemcpyAsync(cex.data(), a.cexact, R * 8, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaStreamSynchronize(s));
    if (prof) {
        std::vector<unsigned long long> tp(260 * 8);
        SC_CUDA(cudaMemcpy(tp.data(), a.tprof, tp.size() * 8, cudaMemcpyDeviceToHost));
        SC_CUDA(cudaFree(a.tprof));
        double acc[6] = {0, 0, 0, 0, 0, 0};
        const int its = f->h_ctl[kCtlIters];
        for (int i = 0; i <= its && i < 255; ++i)
            for (int q = 1; q < 6; ++q)
                if (tp[i * 8 + q] && tp[i * 8 + q - 1]) acc[q] += (tp[i * 8 + q] - tp[i * 8 + q - 1]) * 1e-3;
        fprintf(stderr, "[fused_lloyd] n=%lld k=%d R=%d grid=%d iterations %d: P1 %.1f us, P2 %.1f, "
                "exact decisions %.1f, P3 %.1f, P4 %.1f; final costs %.1f us; total %.1f us; "
                "element-wise chunks %d, ordered maps %d\n",
                (long long)n, k, R, f->grid, its, acc[1], acc[2], acc[3], acc[4], acc[5],
                (tp[255 * 8 + 1] - tp[255 * 8]) * 1e-3, (tp[255 * 8 + 1] - tp[0]) * 1e-3,
                f->h_ctl[kCtlNCross], f->h_ctl[kCtlNTie]);
        fprintf(stderr, "[fused_lloyd] walks: longest %.1f us, latest end after P3 %.1f us, total %.1f us, "
                "in element-wise chunks %.1f us; batches in one step %llu, stepped %llu, steps %llu\n",
                tp[256 * 8] * 1e-3, tp[256 * 8 + 1] * 1e-3, tp[256 * 8 + 2] * 1e-3, tp[256 * 8 + 3] * 1e-3,
                tp[256 * 8 + 4], tp[256 * 8 + 5], tp[256 * 8 + 6]);
        for (int kind = 0; kind < 3; ++kind)
            fprintf(stderr, "[fused_lloyd] P3 %s: %llu tasks, mean %.2f us, max %.2f us\n",
                    kind == 0 ? "first chunks" : kind == 1 ? "crossing records" : "chunk maps",
                    tp[259 * 8 + kind], tp[258 * 8 + kind] * 1e-3 / std::max(1ull, tp[259 * 8 + kind]),
                    tp[258 * 8 + 3 + kind] * 1e-3);
        fprintf(stderr, "[fused_lloyd] P3 max per-warp time %.2f us\n", tp[259 * 8 + 3] * 1e-3);
        fprintf(stderr, "[fused_lloyd] P1 tasks: mean %.2f us, max %.2f us; max per-warp P1 time %.2f us, "
                "max tasks per warp %llu, max P1 end since iteration start %.2f us\n",
                tp[256 * 8 + 7] * 1e-3 / (41.0 * 9770), tp[256 * 8 + 8] * 1e-3, tp[256 * 8 + 9] * 1e-3,
                tp[256 * 8 + 10], tp[256 * 8 + 11] * 1e-3);
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
    widen_labels(lab8.data(), labels_out, n);
    if (costs_out)
        for (int r = 0; r < R; ++r) costs_out[r] = cex[r];
    if (iters_out)
        for (int r = 0; r < R; ++r) iters_out[r] = fin[r] + 1;
    if (best_out) *best_out = best;
    return SC_OK;
}

}  // namespace sc
