// sc_kmeans.cu -- 1-D k-means on the embedding f (K4): a bit-exact device replica of the
// reference's restarted Lloyd (specluster/kmeans.py:167-215), all restarts batched.
//
// Exactness contract, element by element:
//   distances      _sq_dists_to (kmeans.py:106-113): ((x*x) - ((2x)*c)) + (c*c), clip 0,
//                  every op separately rounded (d2ref in sc_common.cuh)
//   argmin         lowest index among equal distances (kmeans.py:199)
//   empty repair   _repair_empty (kmeans.py:151-164): clusters empty after assignment, in
//                  increasing order, take the first point of maximal own-distance
//   means          np.add.at (kmeans.py:89): per cluster, left-to-right sum in point index
//                  order -- reproduced by a stable radix sort on the label followed by an
//                  ordered segmented sum -- then sum / count
//   cost           kmeans_cost (kmeans.py:96-103): numpy einsum("ij,ij->") on (n,1): 8192-
//                  element buffers, two lanes, 8-element steps in order 6|7,4|5,2|3,0|1
//   seeding        _kmeans_pp_indices (kmeans.py:121-137): cumsum is sequential (np.cumsum),
//                  searchsorted(..., 'right'), clipped; draws replayed by the host
//   stop rules     kmeans.py:202-210 (evaluated on the host in the same double arithmetic)
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cstring>
#include <mutex>
#include <vector>

#include "sc_common.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#include "sc_seqsum.cuh"

namespace sc {
struct FusedLloyd;  // sc_kmeans_fused.cu
bool fused_lloyd_eligible(int l, int k, int R, int64_t n);
// sc_kmeans_small.cu: one CTA per restart for n <= 4096
bool small_kmeans_eligible(int l, int k, int64_t n);
int32_t small_kpp(int device, cudaStream_t s, const double *d_x, int64_t n, int k, int R,
                  const int32_t *d_start, const double *d_u, int64_t *d_chosen, int32_t *d_degen);
int32_t small_lloyd(cudaStream_t s, const double *d_x, int64_t n, int k, int R,
                    const int64_t *d_chosen, int max_iters, double tol, bool assert_cost,
                    int32_t *d_lab, double *d_cost, int32_t *d_iters, int32_t *d_err,
                    int64_t *labels_out, double *costs_out, int32_t *iters_out, int32_t *best_out);
int32_t fused_lloyd(FusedLloyd **pctx, int device, int sm_count, cudaStream_t s, const double *d_x,
                    int64_t n, int k, int R, const int64_t *d_chosen, int max_iters, double tol,
                    bool assert_cost, int64_t *labels_out, double *costs_out, int32_t *iters_out,
                    int32_t *best_out);
void fused_lloyd_free(FusedLloyd *f);
const double *graph_f_device(sc_graph *g);
int64_t graph_n(const sc_graph *g);
int graph_device(const sc_graph *g);
}  // namespace sc

struct sc_kmeans {
    int device = 0;
    int sm_count = 148;
    int64_t n = 0;
    int l = 1;                     // point dimension; d_x is [n][l] row-major
    double *d_x = nullptr;
    int32_t *d_idx = nullptr, *d_idx_alt = nullptr;  // [R*n] sort payload when l > 1
    cudaStream_t stream = nullptr;
    cudaStream_t stream2 = nullptr;  // Lloyd: cost of iteration it beside main(it+1)
    cudaEvent_t ev_main = nullptr, ev_cost = nullptr;
    double *h_cost = nullptr;        // pinned [2][R]
    int32_t *h_changed = nullptr;    // pinned [2][R]
    int32_t *h_act = nullptr;        // pinned [2][2R]: active flags + compacted list per parity
    int cap_host_r = 0;
    bool assert_cost = true;         // kmeans.py:206's assert (off: SC_KM_NO_COST_ASSERT)
    sc::FusedLloyd *fused = nullptr;  // persistent exact Lloyd (1-D, one sign, k <= 32)
    unsigned char *h_block = nullptr;  // owned pinned block behind h_cost/h_changed/h_act
    size_t h_block_bytes = 0;
    // workspaces (grown on demand)
    int cap_r = 0, cap_k = 0;
    double *d_best = nullptr;      // [R][n] k-means++ D^2 weights
    int32_t *d_lab[2] = {nullptr, nullptr};  // [R][n] labels (current / previous)
    int32_t *d_keys = nullptr;     // [R*n] sort keys (r*k + label)
    int32_t *d_keys_alt = nullptr;
    double *d_vals = nullptr;      // [R*n] sorted points
    double *d_vals_alt = nullptr;
    void *d_cub = nullptr;
    size_t cub_bytes = 0;
    int64_t *d_chosen = nullptr;   // [R][k]
    double *d_u = nullptr;         // [R][k-1]
    int32_t *d_start = nullptr;    // [R]
    int32_t *d_degen = nullptr;    // [R]
    double *d_cen = nullptr;       // [R][k]
    double *d_scen = nullptr;      // [R][k] centers sorted ascending (sorted assignment)
    int32_t *d_sidx = nullptr;     // [R][k] their original indices
    double *d_cmax = nullptr;      // [R] max |center|
    int32_t *d_elist = nullptr;    // [R][k] empty clusters (cooperative repair)
    int32_t *d_mlist = nullptr;    // [R]
    double *d_pval = nullptr;      // [R][grid] partial argmax
    int64_t *d_pidx = nullptr;
    int coop_grid = 0;
    int32_t *d_cnt = nullptr;      // [R][k]
    int64_t *d_seg = nullptr;      // [R*k + 1] segment offsets into the sorted arrays
    double *d_part = nullptr;      // [R][nchunks][2] einsum lane partials
    double *d_cost = nullptr;      // [R]
    int32_t *d_changed = nullptr;  // [R]
    int32_t *d_active = nullptr;   // [R]
    int32_t *d_empty = nullptr;    // [R]
    // exact sequential-sum workspaces (sc_seqsum.cuh)
    int64_t cap_chunks = 0;
    double *d_A = nullptr, *d_vmax = nullptr, *d_cstart = nullptr, *d_total = nullptr;
    double *d_a64 = nullptr;  // fp64 chunk sums of the k-means++ weights (certified fast draw)
    int32_t *d_kpred = nullptr, *d_neg = nullptr, *d_round_on = nullptr, *d_on = nullptr;
    int64_t *d_q0 = nullptr, *d_q1 = nullptr, *d_cofs = nullptr, *d_nchunks = nullptr;
    int64_t *d_segkpp = nullptr;   // [R+1] restart segments over d_best
    int64_t *d_sq0 = nullptr, *d_sq1 = nullptr;  // super-chunk maps
    double *d_svmax = nullptr;
    int32_t *d_skp = nullptr;
    int32_t *d_kmap = nullptr;     // [chunks] grid the chunk map in d_q0/d_q1 was built on
    double *d_sstart = nullptr;    // [supers] k-means++: exact running sum at super starts
    int32_t *d_sflag = nullptr;
};

namespace sc {

// Pool of page-locked blocks shared by all k-means contexts of the process.  A block is
// owned by exactly one context between pinned_take and pinned_give.
std::mutex g_pinned_mu;
std::vector<std::pair<size_t, unsigned char *>> g_pinned_free;

unsigned char *pinned_take(size_t need) {
    {
        std::lock_guard<std::mutex> lk(g_pinned_mu);
        size_t best = g_pinned_free.size();
        for (size_t i = 0; i < g_pinned_free.size(); ++i)
            if (g_pinned_free[i].first >= need &&
                (best == g_pinned_free.size() || g_pinned_free[i].first < g_pinned_free[best].first))
                best = i;
        if (best < g_pinned_free.size()) {
            unsigned char *p = g_pinned_free[best].second;
            g_pinned_free.erase(g_pinned_free.begin() + best);
            return p;
        }
    }
    unsigned char *p = nullptr;
    if (cudaMallocHost((void **)&p, need) != cudaSuccess) return nullptr;
    return p;
}

void pinned_give(unsigned char *p, size_t bytes) {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    g_pinned_free.emplace_back(bytes, p);
}

constexpr int kEinsumBuf = 8192;  // numpy nditer buffer size (elements)

// _sq_dists_to for one point / one center of dimension l (kmeans.py:106-113):
// (sum x^2 - 2 sum x*c) + sum c^2, clipped at 0, each sum left to right, every operation
// separately rounded.  For l = 1 it equals d2ref bit for bit (2.0*(x*c) == (2x)*c).  The
// reference evaluates the middle term with BLAS (dgemm/dgemv), whose summation order is
// CPU-specific, so for l > 1 labels agree with the reference up to exact ties only.
__device__ __forceinline__ double d2nd(const double *__restrict__ x, const double *__restrict__ c,
                                       int l) {
    if (l == 1) return d2ref(x[0], c[0]);
    double xx = 0.0, xc = 0.0, cc = 0.0;
    for (int q = 0; q < l; ++q) {
        xx = __dadd_rn(xx, __dmul_rn(x[q], x[q]));
        xc = __dadd_rn(xc, __dmul_rn(x[q], c[q]));
        cc = __dadd_rn(cc, __dmul_rn(c[q], c[q]));
    }
    const double v = __dadd_rn(__dsub_rn(xx, __dmul_rn(2.0, xc)), cc);
    return v < 0.0 ? 0.0 : v;
}

// ---------------------------------------------------------------------------
// Segmented exact sequential sums (sc_seqsum.cuh) over a batch of segments.
//
// Segment s covers elements [seg_off[s], seg_off[s+1]) of vals and chunks
// [cofs[s], cofs[s+1]) (kSeqChunk elements per chunk).  Segments whose `on` flag is 0 are
// skipped (finished restarts).

struct SegView {
    const double *vals;
    const int64_t *seg_off;  // S + 1
    const int64_t *cofs;     // S + 1
    int S;
    const int32_t *on;       // per group of `on_div` segments (nullable = all on)
    int on_div;
};

struct SeqWork {
    double *A;        // approximate chunk sums
    double *vmax;     // chunk max element
    int32_t *kpred;   // predicted grid exponent per chunk (kNoGrid = step it)
    int64_t *q0, *q1; // chunk parity map
    double *cstart;   // exact running sum at each chunk start
    int32_t *neg;     // per segment flags: 1 negative, 2 positive, 4 non-finite element
    double *total;    // per segment exact total
    // super-chunks: kSuper consecutive chunks (aligned to the global chunk index) composed
    // into one map when they all lie in one segment on one predicted grid
    int64_t *sq0, *sq1;
    double *svmax;
    int32_t *skp;     // common predicted grid, or kNoGrid (walk the chunks one by one)
    // k-means++ search by super-chunk (compose mode 2): exact running sum at every super
    // start, and whether the super was advanced whole (1: its chunk starts follow from the
    // chunk maps) or chunk by chunk (0: cstart holds them)
    double *sstart = nullptr;
    int32_t *sflag = nullptr;
};

constexpr int kSuper = 32;
constexpr int kNoMap = 0x7f7f7f7f;  // k-means++ kmap: no valid chunk map (no grid exponent)
constexpr int kMaxKppR = 64;        // restarts of the one-pass k-means++ round
// stride of a restart's k-means++ weights: n rounded up to whole super-chunks
constexpr int64_t kppStrideAlign = (int64_t)kSuper * kSeqChunk;
__host__ __device__ __forceinline__ int64_t kpp_stride(int64_t n) {
    return (n + kppStrideAlign - 1) / kppStrideAlign * kppStrideAlign;
}

__device__ __forceinline__ int seg_of_chunk(const SegView &v, int64_t c) {
    int lo = 0, hi = v.S;  // cofs[lo] <= c < cofs[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (v.cofs[mid] <= c) lo = mid;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ bool seg_on(const SegView &v, int s) {
    return v.on == nullptr || v.on[s / v.on_div] != 0;
}

// load the chunk's elements 8 per lane, lane-contiguous; returns the element count
__device__ __forceinline__ int load_chunk(const SegView &v, int s, int64_t c,
                                          double (&a)[kSeqPerLane], int64_t &first) {
    const int lane = threadIdx.x & 31;
    const int64_t lo = v.seg_off[s] + (c - v.cofs[s]) * kSeqChunk;
    const int64_t hi = min(lo + kSeqChunk, v.seg_off[s + 1]);
    first = lo;
#pragma unroll
    for (int t = 0; t < kSeqPerLane; ++t) {
        const int64_t j = lo + lane * kSeqPerLane + t;
        a[t] = j < hi ? v.vals[j] : 0.0;
    }
    return int(hi - lo);
}

__global__ void k_seq_summarize(SegView v, SeqWork w, const int64_t *__restrict__ pn) {
    const int64_t nchunks = *pn;
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = wid; c < nchunks; c += nw) {
        const int s = seg_of_chunk(v, c);
        if (!seg_on(v, s)) continue;
        double a[kSeqPerLane];
        int64_t first;
        const int m = load_chunk(v, s, c, a, first);
        double sum = 0.0, mx = 0.0;
        int fl = 0;
#pragma unroll
        for (int t = 0; t < kSeqPerLane; ++t) {
            if (lane * kSeqPerLane + t < m) {
                sum += a[t];
                mx = fmax(mx, a[t]);
                fl |= (a[t] < 0.0) | ((a[t] > 0.0) << 1) | ((!isfinite(a[t])) << 2);
            }
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            sum += __shfl_xor_sync(0xffffffffu, sum, d);
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
            fl |= __shfl_xor_sync(0xffffffffu, fl, d);
        }
        if (lane == 0) {
            w.A[c] = sum;
            w.vmax[c] = mx;
            if (fl) atomicOr(&w.neg[s], fl);
        }
    }
}

// one warp per segment: approximate chunk starts -> predicted grid per chunk.  Chunk data
// are read 256 at a time (8 independent loads per lane) so the walk pays one memory latency
// per 256 chunks.
// A segment whose elements are all <= 0 is summed as the negation of its negated elements
// (round-to-nearest-even is symmetric: fl(-x + -y) = -fl(x + y)), so it takes the fast
// path too; only mixed-sign or non-finite segments are added element by element.
__device__ __forceinline__ bool seg_slow(int f) { return (f & 4) || ((f & 1) && (f & 2)); }
__device__ __forceinline__ bool seg_flipped(int f) { return !seg_slow(f) && (f & 1); }

// one warp per chunk of a flipped segment: negate its elements in place and re-summarise
__global__ void k_seq_flip(SegView v, SeqWork w, const int64_t *__restrict__ pn) {
    const int64_t nchunks = *pn;
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double *vals = const_cast<double *>(v.vals);
    for (int64_t c = wid; c < nchunks; c += nw) {
        const int s = seg_of_chunk(v, c);
        if (!seg_on(v, s) || !seg_flipped(w.neg[s])) continue;
        const int64_t lo = v.seg_off[s] + (c - v.cofs[s]) * kSeqChunk;
        const int64_t hi = min(lo + kSeqChunk, v.seg_off[s + 1]);
        double sum = 0.0, mx = 0.0;
        for (int64_t j = lo + lane; j < hi; j += 32) {
            const double a = -vals[j];
            vals[j] = a;
            sum += a;
            mx = fmax(mx, a);
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            sum += __shfl_xor_sync(0xffffffffu, sum, d);
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        }
        if (lane == 0) {
            w.A[c] = sum;
            w.vmax[c] = mx;
        }
    }
}

constexpr int kPredictWarps = 8;

// one CTA per segment: each warp takes a contiguous share of the segment's chunks, the
// warps' approximate totals are scanned in shared memory, then every warp walks its share
// from its carry (approximate prefixes: they only steer the prediction, compose re-checks)
template <int PW = kPredictWarps>
__global__ void __launch_bounds__(32 * PW) k_seq_predict(SegView v, SeqWork w) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int s = blockIdx.x;
    if (s >= v.S || !seg_on(v, s)) return;
    const int64_t c0s = v.cofs[s], c1s = v.cofs[s + 1];
    const int64_t per = ((c1s - c0s + PW - 1) / PW + 31) / 32 * 32;
    const int64_t c0 = min(c1s, c0s + wid * per), c1 = min(c1s, c0 + per);
    __shared__ double part[PW];
    double tot = 0.0;
    for (int64_t c = c0 + lane; c < c1; c += 32) tot += w.A[c];
#pragma unroll
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0) part[wid] = tot;
    __syncthreads();
    double carry = 0.0;
    for (int q = 0; q < wid; ++q) carry += part[q];
    const double lo_f = 1.0 - 1.0 / 1048576.0, hi_f = 1.0 + 1.0 / 1048576.0;
    for (int64_t blk = c0; blk < c1; blk += 256) {
        double A[8], V[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const int64_t c = blk + 32 * t + lane;
            A[t] = c < c1 ? w.A[c] : 0.0;
            V[t] = c < c1 ? w.vmax[c] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            double incl = A[t];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double o = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += o;
            }
            const double P = carry + (incl - A[t]);
            const int64_t c = blk + 32 * t + lane;
            if (c < c1) {
                int kp = kNoGrid;
                const double plo = P * lo_f, phi = (P + A[t] + V[t]) * hi_f;
                if (plo >= 2.2250738585072014e-308) {
                    const Grid ga = grid_of(plo), gb = grid_of(phi);
                    if (ga.k == gb.k) kp = ga.k;
                }
                w.kpred[c] = kp;
            }
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
}

// one warp per chunk: parity map of the chunk on its predicted grid
__global__ void k_seq_chunkmap(SegView v, SeqWork w, const int64_t *__restrict__ pn) {
    const int64_t nchunks = *pn;
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = wid; c < nchunks; c += nw) {
        const int kp = w.kpred[c];
        if (kp == kNoGrid) continue;
        const int s = seg_of_chunk(v, c);
        if (!seg_on(v, s)) continue;
        double a[kSeqPerLane];
        int64_t first;
        const int m = load_chunk(v, s, c, a, first);
        PMap lm = pmap_id();
#pragma unroll
        for (int t = 0; t < kSeqPerLane; ++t)
            if (lane * kSeqPerLane + t < m) lm = pmap_then(lm, pmap_elem(to_units(a[t], kp)));
        const PMap tot = warp_scan_pmap(lm);
        if (lane == 31) {
            w.q0[c] = tot.i0;
            w.q1[c] = tot.i1;
        }
    }
}

// one warp per super-chunk: compose its 32 chunk maps (lane = chunk) when they share one
// segment and one predicted grid
__global__ void k_seq_superize(SegView v, SeqWork w, const int64_t *__restrict__ pn) {
    const int64_t nchunks = *pn;
    const int64_t nsup = (nchunks + kSuper - 1) / kSuper;
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t g = wid; g < nsup; g += nw) {
        const int64_t c = g * kSuper + lane;
        const bool full = (g + 1) * kSuper <= nchunks;
        int kp = kNoGrid;
        PMap m = pmap_id();
        double vm = 0.0;
        if (full) {
            kp = w.kpred[c];
            m = PMap{w.q0[c], w.q1[c]};
            vm = w.vmax[c];
        }
        int ok = full && kp != kNoGrid;
        const int kp0 = __shfl_sync(0xffffffffu, kp, 0);
        ok = __all_sync(0xffffffffu, ok && kp == kp0);
        if (ok && lane == 0) {
            const int s0 = seg_of_chunk(v, g * kSuper);
            ok = seg_on(v, s0) && v.cofs[s0 + 1] >= (g + 1) * kSuper;
        }
        ok = __shfl_sync(0xffffffffu, ok, 0);
        const PMap tot = warp_scan_pmap(m);
#pragma unroll
        for (int o = 16; o; o >>= 1) vm = fmax(vm, __shfl_xor_sync(0xffffffffu, vm, o));
        if (lane == 31) {
            w.skp[g] = ok ? kp0 : kNoGrid;
            w.sq0[g] = tot.i0;
            w.sq1[g] = tot.i1;
            w.svmax[g] = vm;
        }
    }
}

// one warp per segment: exact composition of the chunk maps (see sc_seqsum.cuh).  Each
// warp stages 256 chunks' maps in its slice of shared memory (one memory latency per 256
// chunks), then advances up to 32 chunks per step; a chunk whose exact start contradicts its
// prediction is stepped element by element.
constexpr int kMetaBlk = 256;
constexpr int kComposeWarps = 4;
constexpr size_t kComposeSmem =
    (size_t)kComposeWarps * (kMetaBlk * (8 + 8 + 8 + 4) + kSeqChunk * 8);

__global__ void __launch_bounds__(32 * kComposeWarps) k_seq_compose(SegView v, SeqWork w,
                                                                  int want_cstart) {
    extern __shared__ unsigned char cm_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int s = blockIdx.x * kComposeWarps + wib;
    if (s >= v.S || !seg_on(v, s)) return;
    int64_t *sq0 = reinterpret_cast<int64_t *>(cm_raw) + wib * kMetaBlk;
    int64_t *sq1 = reinterpret_cast<int64_t *>(cm_raw) + (kComposeWarps + wib) * kMetaBlk;
    double *svm = reinterpret_cast<double *>(cm_raw) + (2 * kComposeWarps + wib) * kMetaBlk;
    int32_t *skp = reinterpret_cast<int32_t *>(reinterpret_cast<double *>(cm_raw) +
                                               3 * kComposeWarps * kMetaBlk) + wib * kMetaBlk;
    double *sbuf = reinterpret_cast<double *>(cm_raw + (size_t)kComposeWarps * kMetaBlk * 28) +
                   wib * kSeqChunk;
    const int64_t c0 = v.cofs[s], c1 = v.cofs[s + 1];
    double run = 0.0;
    const int sflags = w.neg[s];
    const double sgn = seg_flipped(sflags) ? -1.0 : 1.0;  // flipped: negated elements
    if (seg_slow(sflags)) {
        // mixed signs or non-finite elements: plain sequential sum
        for (int64_t c = c0; c < c1; ++c) {
            double a[kSeqPerLane];
            int64_t first;
            const int m = load_chunk(v, s, c, a, first);
            if (lane == 0) w.cstart[c] = run;
            warp_step_seq(a, m, run, 0.0, false, sbuf);
        }
        if (lane == 0) w.total[s] = run;
        return;
    }
    int64_t c = c0, blk = -1, blk_end = -1;
    // super metadata of the next 32 supers, loaded one step ahead (a full super step then
    // costs one memory latency less)
    int64_t pfG = -1;
    int pf_kp = kNoGrid;
    int64_t pf_q0 = 0, pf_q1 = 0;
    double pf_vm = 0.0;
    auto super_meta = [&](int64_t G0) {
        const int64_t Gl = G0 + lane;
        if ((Gl + 1) * kSuper <= c1) {
            pf_kp = w.skp[Gl];
            pf_q0 = w.sq0[Gl];
            pf_q1 = w.sq1[Gl];
            pf_vm = w.svmax[Gl];
        }
        pfG = G0;
    };
    while (c < c1) {
        if ((c & (kSuper - 1)) == 0 && c + kSuper <= c1) {
            // super step: up to 32 super-chunks (1024 chunks) on the current grid at once
            const Grid g = grid_of(run);
            const int64_t S0 = (int64_t)to_units(run, g.k);
            const int64_t G = c / kSuper + lane;
            const bool valid = (G + 1) * kSuper <= c1;
            if (pfG != c / kSuper) super_meta(c / kSuper);
            const int m_kp = pf_kp;
            const int64_t m_q0 = pf_q0, m_q1 = pf_q1;
            const double m_vm = pf_vm;
            super_meta(c / kSuper + 32);  // in flight during this step
            bool ok = false;
            PMap m = pmap_id();
            double vmu = 0.0;
            if (valid && g.top == (int64_t(1) << 53) && m_kp == g.k) {
                m = PMap{m_q0, m_q1};
                vmu = to_units(m_vm, g.k);
                ok = true;
            } else if (valid && m_vm == 0.0) {
                ok = true;  // all zeros (elements are >= 0 here): fl(s + 0) = s, any grid
            }
            const PMap excl = warp_exclusive(warp_scan_pmap(m));
            const int64_t Sl = pmap_apply(excl, S0);
            if (ok) {
                const int64_t qmax = max(m.i0, m.i1);
                ok = (double)(g.top - Sl - qmax) >= vmu && Sl + qmax <= g.top;
            }
            const unsigned badm = __ballot_sync(0xffffffffu, valid && !ok);
            const unsigned valm = __ballot_sync(0xffffffffu, valid);
            const int Lb = badm ? __ffs(badm) - 1 : 32;
            const int nadv = min(Lb, __popc(valm));
            if (want_cstart == 2 && lane < nadv) {
                w.sstart[G] = sgn * from_units(Sl, g.k);
                w.sflag[G] = 1;
            }
            if (want_cstart == 1 && lane < nadv) {
                // exact start of every chunk of this super-chunk (for the k-means++ search);
                // the chunk maps are fetched 8 at a time so a step pays 4 memory latencies
                int64_t S = Sl;
                const int64_t cb = G * kSuper;
                for (int t0 = 0; t0 < kSuper; t0 += 8) {
                    int64_t a0[8], a1[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        a0[u] = w.q0[cb + t0 + u];
                        a1[u] = w.q1[cb + t0 + u];
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        w.cstart[cb + t0 + u] = sgn * from_units(S, g.k);
                        S = pmap_apply(PMap{a0[u], a1[u]}, S);
                    }
                }
            }
            if (nadv > 0) {
                const int64_t Send = __shfl_sync(0xffffffffu, pmap_apply(m, Sl), nadv - 1);
                run = from_units(Send, g.k);
                c += (int64_t)nadv * kSuper;
                continue;
            }
            // the first super-chunk needs the chunk walk (grid change or non-uniform)
        }
        if (c >= blk_end) {
            blk = c;
            blk_end = min(c + kMetaBlk, c1);
            __syncwarp();
            for (int t = lane; t < kMetaBlk; t += 32) {
                const int64_t cc = blk + t;
                if (cc < blk_end) {
                    sq0[t] = w.q0[cc];
                    sq1[t] = w.q1[cc];
                    svm[t] = w.vmax[cc];
                    skp[t] = w.kpred[cc];
                }
            }
            __syncwarp();
        }
        const Grid g = grid_of(run);
        const int64_t S0 = (int64_t)to_units(run, g.k);
        const int64_t cl = c + lane;
        const bool valid = cl < blk_end && cl < (c / kSuper + 1) * kSuper;
        bool ok = false;
        PMap m = pmap_id();
        double vmu = 0.0;
        if (valid && g.top == (int64_t(1) << 53) && skp[cl - blk] == g.k) {
            m = PMap{sq0[cl - blk], sq1[cl - blk]};
            vmu = to_units(svm[cl - blk], g.k);
            ok = true;
        } else if (valid && svm[cl - blk] == 0.0) {
            ok = true;  // all zeros: identity (a long zero prefix keeps the sum at 0, whose
                        // subnormal grid no chunk map is built on)
        }
        const PMap excl = warp_exclusive(warp_scan_pmap(m));
        const int64_t Sl = pmap_apply(excl, S0);
        if (ok) {
            const int64_t qmax = max(m.i0, m.i1);
            ok = (double)(g.top - Sl - qmax) >= vmu && Sl + qmax <= g.top;
        }
        const unsigned badm = __ballot_sync(0xffffffffu, valid && !ok);
        const unsigned valm = __ballot_sync(0xffffffffu, valid);
        const int Lb = badm ? __ffs(badm) - 1 : 32;   // first chunk to step
        const int Le = __popc(valm);                  // valid lanes form a prefix
        const int nadv = min(Lb, Le);
        if (want_cstart && lane < nadv) w.cstart[cl] = sgn * from_units(Sl, g.k);
        if (want_cstart == 2 && lane < nadv && (cl & (kSuper - 1)) == 0) {
            w.sstart[cl / kSuper] = sgn * from_units(Sl, g.k);
            w.sflag[cl / kSuper] = 0;
        }
        if (nadv > 0) {
            const int64_t Send = __shfl_sync(0xffffffffu, pmap_apply(m, Sl), nadv - 1);
            run = from_units(Send, g.k);
            c += nadv;
        }
        if (Lb < Le) {
            // step chunk c element by element
            if (want_cstart && lane == 0) w.cstart[c] = sgn * run;
            if (want_cstart == 2 && lane == 0 && (c & (kSuper - 1)) == 0) {
                w.sstart[c / kSuper] = sgn * run;
                w.sflag[c / kSuper] = 0;
            }
            double a[kSeqPerLane];
            int64_t first;
            const int mcount = load_chunk(v, s, c, a, first);
            warp_step_seq(a, mcount, run, 0.0, false, sbuf);
            ++c;
        }
    }
    if (lane == 0) w.total[s] = sgn * run;
}

// ---------------------------------------------------------------------------
// k-means++

// best[r][j] = min over chosen[r][0..start_r-1] of d2(x_j, x[chosen])
__global__ void k_kpp_init(const double *__restrict__ x, int64_t n, int l, int k,
                           const int64_t *__restrict__ chosen, const int32_t *__restrict__ start,
                           const int32_t *__restrict__ on, double *__restrict__ best,
                           int32_t *__restrict__ kpred, int64_t cps) {
    const int r = blockIdx.y;
    if (!on[r]) return;
    const int s = start[r];
    const int64_t nb = kpp_stride(n);
    double *b = best + (int64_t)r * nb;
    const int64_t *ch = chosen + (int64_t)r * k;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nb;
         j += (int64_t)gridDim.x * blockDim.x) {
        double v = 0.0;  // padding past n stays 0 (adds nothing to any running sum)
        if (j < n) {
            const double *xj = x + j * l;
            v = d2nd(xj, x + ch[0] * l, l);
            for (int i = 1; i < s; ++i) v = fmin(v, d2nd(xj, x + ch[i] * l, l));
        }
        b[j] = v;
        if (j < cps) kpred[(int64_t)r * cps + j] = kNoGrid;  // no speculative grid yet
    }
}


// k-means++ round i, fused with the seqsum summary of the D^2 weights: one warp per
// 256-weight chunk lowers best[] by the distance to the center chosen in round i-1 (when
// this restart has one) and records the chunk's approximate sum and max for the prediction
// (k_seq_summarize's output), so the weights are read once per round instead of twice
__global__ void k_kpp_update_sum(const double *__restrict__ x, int64_t n, int l, int k, int i,
                                 const int64_t *__restrict__ chosen,
                                 const int32_t *__restrict__ start, const int32_t *__restrict__ on,
                                 const int32_t *__restrict__ round_on, double *__restrict__ best,
                                 SeqWork w, int64_t cps, int R) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = wid; c < (int64_t)R * cps; c += nw) {
        const int r = (int)(c / cps);
        if (!round_on[r]) continue;
        const bool upd = on[r] && i - 1 >= start[r];
        const double *cn = upd ? x + chosen[(int64_t)r * k + i - 1] * l : nullptr;
        double *b = best + (int64_t)r * kpp_stride(n);
        const int64_t j0 = (c - (int64_t)r * cps) * kSeqChunk + lane * kSeqPerLane;
        double sum = 0.0, mx = 0.0;
        int bad = 0;
#pragma unroll
        for (int t = 0; t < kSeqPerLane; ++t) {
            const int64_t j = j0 + t;
            if (j < n) {
                double v = b[j];
                if (upd) {
                    const double d = d2nd(x + j * l, cn, l);
                    if (d < v) {
                        v = d;
                        b[j] = v;
                    }
                }
                sum += v;
                mx = fmax(mx, v);
                bad |= !(v >= 0.0) || !isfinite(v);
            }
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            sum += __shfl_xor_sync(0xffffffffu, sum, d);
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
            bad |= __shfl_xor_sync(0xffffffffu, bad, d);
        }
        if (lane == 0) {
            w.A[c] = sum;
            w.vmax[c] = mx;
            if (bad) w.neg[r] = 4;
        }
    }
}

// per-round segment flags: restart still seeding and round i belongs to this call
// 1-D k-means++ round, one pass over the weights: one warp per chunk position, all restarts
// (x of the chunk is read once).  Each restart's weights take the distance to its newest
// centre (kmeans.py:137 np.minimum), the chunk's approximate sum / max are written for the
// prediction, and -- speculatively, on the grid the previous round predicted for the chunk
// (the weights only shrink, so most chunks keep their binade) -- the chunk's parity map.
// kmap records the grid each map was built on; k_seq_chunkmap_fix rebuilds the chunks whose
// new prediction differs, so no map is ever used on the wrong grid.
__global__ void __launch_bounds__(256, 4)
k_kpp_update_map(const double *__restrict__ x, int64_t n, int k, int i,
                 const int64_t *__restrict__ chosen, const int32_t *__restrict__ start,
                 const int32_t *__restrict__ on, const int32_t *__restrict__ round_on,
                 double *__restrict__ best, SeqWork w, int32_t *__restrict__ kmap, int64_t cps,
                 int R, double *__restrict__ a64) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nb = kpp_stride(n);
    // per-restart state once per block (no dependent global loads in the task loop)
    __shared__ int s_mode[kMaxKppR];  // 0 off, 1 on without a new centre, 2 update
    __shared__ double s_cn[kMaxKppR];
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
        const bool ro = round_on[r] != 0;
        const bool upd = ro && on[r] && i - 1 >= start[r];
        s_mode[r] = ro ? (upd ? 2 : 1) : 0;
        s_cn[r] = upd ? __ldg(x + chosen[(int64_t)r * k + i - 1]) : 0.0;
    }
    __syncthreads();
    // task t = (chunk position cc, restart r), r fastest: the R warps of one chunk position
    // read the same x lines (one HBM read, the rest from L1/L2)
    for (int64_t t = wid; t < cps * R; t += nw) {
        const int64_t cc = t / R;
        const int r = (int)(t - cc * R);
        const int mode = s_mode[r];
        if (!mode) continue;
        const int64_t j0 = cc * kSeqChunk + lane * kSeqPerLane;
        const int64_t c = (int64_t)r * cps + cc;
        const bool upd = mode == 2;
        const double cn = s_cn[r];
        double *b = best + (int64_t)r * nb;
        const int kp = w.kpred[c];
        double a[kSeqPerLane], xv[kSeqPerLane];
#pragma unroll
        for (int q = 0; q < kSeqPerLane; q += 2) {
            const double2 bb = *reinterpret_cast<const double2 *>(b + j0 + q);
            a[q] = bb.x;
            a[q + 1] = bb.y;
        }
        if (upd) {
            // (x holds n doubles: vector loads only for chunks wholly inside [0, n))
            if (j0 + kSeqPerLane <= n) {
#pragma unroll
                for (int q = 0; q < kSeqPerLane; q += 2) {
                    const double2 xx = __ldg(reinterpret_cast<const double2 *>(x + j0 + q));
                    xv[q] = xx.x;
                    xv[q + 1] = xx.y;
                }
            } else {
#pragma unroll
                for (int q = 0; q < kSeqPerLane; ++q) xv[q] = j0 + q < n ? __ldg(x + j0 + q) : 0.0;
            }
        }
        // chunk summaries in fp32: the sum only steers the prediction, and the max is
        // rounded UP, so it stays an upper bound (all the exact walk needs); a zero chunk
        // keeps a zero max.  Half the shuffle traffic of fp64 reductions.
        float sum = 0.f, mx = 0.f;
        bool bad = false;
        bool wr = false;
#pragma unroll
        for (int q = 0; q < kSeqPerLane; ++q) {
            if (upd && j0 + q < n) {
                const double d = d2ref(xv[q], cn);
                if (d < a[q]) {
                    a[q] = d;
                    wr = true;
                }
            }
            sum += __double2float_rn(a[q]);
            mx = fmaxf(mx, __double2float_ru(a[q]));
            bad |= !(a[q] >= 0.0) || !isfinite(a[q]);
        }
        if (wr) {
#pragma unroll
            for (int q = 0; q < kSeqPerLane; q += 2)
                *reinterpret_cast<double2 *>(b + j0 + q) = make_double2(a[q], a[q + 1]);
        }
        // a chunk none of whose weights changed keeps its map if it was built on kp already
        const bool changed = __any_sync(0xffffffffu, wr);
        const bool need_map = kp != kNoGrid && (changed || kmap[c] != kp);
        PMap lm = pmap_id();
        if (need_map) {
#pragma unroll
            for (int q = 0; q < kSeqPerLane; ++q) lm = pmap_then(lm, pmap_elem(to_units(a[q], kp)));
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            sum += __shfl_xor_sync(0xffffffffu, sum, d);
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        }
        const bool anybad = __any_sync(0xffffffffu, bad);
        if (need_map) lm = warp_scan_pmap(lm);
        if (a64) {  // fp64 chunk sum (13 roundings) for the certified fast draw (k_kpp_fast)
            double s64 = 0.0;
#pragma unroll
            for (int q = 0; q < kSeqPerLane; ++q) s64 = __dadd_rn(s64, a[q]);
#pragma unroll
            for (int d = 16; d; d >>= 1) s64 = __dadd_rn(s64, __shfl_xor_sync(0xffffffffu, s64, d));
            if (lane == 31) a64[c] = s64;
        }
        if (lane == 31) {
            w.A[c] = (double)sum;
            w.vmax[c] = (double)mx;
            if (anybad) w.neg[r] = 4;
            if (need_map) {
                w.q0[c] = lm.i0;
                w.q1[c] = lm.i1;
                kmap[c] = kp;
            } else if (changed) {
                kmap[c] = kNoMap;  // the old map no longer describes the chunk
            }
        }
    }
}

// Certified fast k-means++ draw (kmeans.py:116-118), one CTA per restart.  The reference picks
// idx = searchsorted(cum, u * cum[-1], 'right') on the SEQUENTIAL fp64 cumsum of the weights.
// Sums of nonnegative terms computed with m roundings in ANY order lie within m u / (1 - m u)
// of the real sum (u = 2^-53), so every sequential prefix cum[j] lies in [q (1 - eps),
// q (1 + eps)] for the tree-order prefix q of the same terms, eps >= (n + roundings of q) u (the
// host passes 1.0625 (n + 128 + tiles) u).  With T the tree total, the target u * cum[-1]
// (one more rounding) lies in [tl, th] = [u T (1 - eps - 2u), u T (1 + eps + 2u)] (directed
// roundings).  The draw is j exactly when cum[j-1] <= target < cum[j]; it is CERTIFIED when
// q[j-1] (1 + eps) <= tl and q[j] (1 - eps) > th (cum is nondecreasing, so j-1 covers all
// earlier indices).  Then chosen is written and the restart's round flag cleared, so the exact
// pipeline below (prediction, chunk maps, compose, search) skips it; otherwise nothing is
// written and the exact pipeline decides (probability ~2 eps T / weight per draw).  A zero tree
// total means every weight is zero exactly: the degenerate branch (kmeans.py:128-134), reported
// as k_kpp_search2 does.
__global__ void __launch_bounds__(256) k_kpp_fast(const double *__restrict__ best,
                                                  const double *__restrict__ a64, int64_t n,
                                                  int64_t nb, int64_t cps, int k, int i,
                                                  const double *__restrict__ u,
                                                  int64_t *__restrict__ chosen, int32_t *__restrict__ on,
                                                  int32_t *__restrict__ round_on,
                                                  int32_t *__restrict__ degen, double eps,
                                                  unsigned long long *__restrict__ stats) {
    using Reduce = cub::BlockReduce<double, 256>;
    using Scan = cub::BlockScan<double, 256>;
    __shared__ union {
        typename Reduce::TempStorage tr;
        typename Scan::TempStorage ts;
    } tmp;
    __shared__ double s_T, s_start;
    __shared__ long long s_chunk;
    const int r = blockIdx.x, tid = threadIdx.x;
    if (!round_on[r]) return;
    const double *A = a64 + (int64_t)r * cps;
    double part = 0.0;
    for (int64_t c = tid; c < cps; c += 256) part = __dadd_rn(part, A[c]);
    const double tot = Reduce(tmp.tr).Sum(part);
    if (tid == 0) {
        s_T = tot;
        s_chunk = -1;
    }
    __syncthreads();
    const double T = s_T;
    if (T == 0.0) {  // all weights are +0.0: degenerate round
        if (tid == 0) {
            degen[r] = i;
            on[r] = 0;
            round_on[r] = 0;
        }
        return;
    }
    if (!(T > 1e-280) || !(T < 1e280)) return;  // (NaN, overflow, near-subnormal: exact path)
    const double ur = u[(int64_t)r * (k - 1) + (i - 1)];
    const double dn = 1.0 - eps - 2.3e-16, up = 1.0 + eps + 2.3e-16;
    const double tl = __dmul_rd(__dmul_rd(ur, T), dn), th = __dmul_ru(__dmul_ru(ur, T), up);
    const double e_up = 1.0 + eps, e_dn = 1.0 - eps;
    // the chunk whose [start, end) certainly holds the target
    double carry = 0.0;
    for (int64_t c0 = 0; c0 < cps; c0 += 256) {
        const int64_t c = c0 + tid;
        const double v = c < cps ? A[c] : 0.0;
        double excl, agg;
        __syncthreads();
        Scan(tmp.ts).ExclusiveSum(v, excl, agg);
        const double st = __dadd_rn(carry, excl);
        const double end = __dadd_rn(carry, __dadd_rn(excl, v));
        carry = __dadd_rn(carry, agg);
        if (c < cps && __dmul_ru(st, e_up) <= tl && __dmul_rd(end, e_dn) > th) {
            s_chunk = (long long)c;
            s_start = st;
        }
    }
    __syncthreads();
    const long long cs = s_chunk;
    if (cs < 0) return;
    if (tid >= 32) return;
    // inside the chunk: lane-local sequential prefixes on top of a warp scan of the lane sums
    const int lane = tid;
    const double *wv = best + (int64_t)r * nb + cs * kSeqChunk + lane * kSeqPerLane;
    double a[kSeqPerLane], loc = 0.0;
#pragma unroll
    for (int q = 0; q < kSeqPerLane; ++q) {
        a[q] = wv[q];
        loc = __dadd_rn(loc, a[q]);
    }
    double inc = loc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc = __dadd_rn(inc, o);
    }
    double q = __dadd_rn(s_start, __shfl_up_sync(0xffffffffu, inc, 1));  // prefix before this lane
    if (lane == 0) q = s_start;
    int hit = -1;
    bool okp = false;
#pragma unroll
    for (int t = 0; t < kSeqPerLane; ++t) {
        const double qn = __dadd_rn(q, a[t]);
        if (hit < 0 && __dmul_rd(qn, e_dn) > th) {
            hit = t;
            okp = __dmul_ru(q, e_up) <= tl;
        }
        q = qn;
    }
    // the first lane that crosses decides (prefixes are nondecreasing)
    const unsigned mh = __ballot_sync(0xffffffffu, hit >= 0);
    if (!mh) return;
    const int wl = __ffs(mh) - 1;
    const int whit = __shfl_sync(0xffffffffu, hit, wl);
    const bool wok = __shfl_sync(0xffffffffu, okp, wl);
    const int64_t idx = cs * kSeqChunk + wl * kSeqPerLane + whit;
    if (lane == 0 && wok && idx < n) {
        chosen[(int64_t)r * k + i] = idx;
        round_on[r] = 0;
        if (stats) atomicAdd(stats, 1ull);
    }
}

// one warp per chunk: rebuild the parity map of every chunk whose predicted grid differs from
// the one its map was built on (k_kpp_update_map's speculation missed)
__global__ void k_seq_chunkmap_fix(SegView v, SeqWork w, int32_t *__restrict__ kmap,
                                   const int64_t *__restrict__ pn,
                                   unsigned long long *__restrict__ stats) {
    const int64_t nchunks = *pn;
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // 32 chunks per warp step: each lane checks one, then the warp rebuilds the misses
    for (int64_t c0 = wid * 32; c0 < nchunks; c0 += nw * 32) {
        const int64_t cl = c0 + lane;
        int kpl = kNoGrid;
        bool miss = false;
        if (cl < nchunks) {
            kpl = w.kpred[cl];
            miss = kpl != kNoGrid && kpl != kmap[cl];
        }
        unsigned mm = __ballot_sync(0xffffffffu, miss);
        while (mm) {
            const int b = __ffs(mm) - 1;
            mm &= mm - 1;
            const int64_t c = c0 + b;
            const int kp = __shfl_sync(0xffffffffu, kpl, b);
            const int s = seg_of_chunk(v, c);
            if (!seg_on(v, s)) continue;
            double a[kSeqPerLane];
            int64_t first;
            const int m = load_chunk(v, s, c, a, first);
            PMap lm = pmap_id();
#pragma unroll
            for (int t = 0; t < kSeqPerLane; ++t)
                if (lane * kSeqPerLane + t < m) lm = pmap_then(lm, pmap_elem(to_units(a[t], kp)));
            const PMap tot = warp_scan_pmap(lm);
            if (lane == 31) {
                w.q0[c] = tot.i0;
                w.q1[c] = tot.i1;
                kmap[c] = kp;
                if (stats) atomicAdd(stats, 1ull);
            }
        }
    }
}

// k-means++ draw (kmeans.py:116-118: searchsorted(cumsum(w), u * cumsum(w)[-1], 'right'),
// clipped) from the super-chunk starts of compose mode 2: binary search for the super, its
// chunk starts from the chunk maps (whole supers) or cstart (chunk-walked supers), then the
// chunk element by element.  Segments are super-aligned (kpp_stride).
__global__ void k_kpp_search2(SegView v, SeqWork w, int64_t n, int k, int i,
                              const double *__restrict__ u, int64_t *__restrict__ chosen,
                              int32_t *__restrict__ on, int32_t *__restrict__ degen) {
    const int lane = threadIdx.x & 31;
    const int r = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (r >= v.S || !seg_on(v, r)) return;
    const double tot = w.total[r];
    if (!(tot > 0.0)) {
        if (lane == 0) {
            degen[r] = i;
            on[r] = 0;
        }
        return;
    }
    const double target = __dmul_rn(u[(int64_t)r * (k - 1) + (i - 1)], tot);
    const int64_t c0 = v.cofs[r], c1 = v.cofs[r + 1];
    const int64_t G0 = c0 / kSuper, G1 = c1 / kSuper;
    // first super whose end exceeds target (ends are nondecreasing: the weights are >= 0)
    int64_t lo = G0, hi = G1;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const double end = mid + 1 < G1 ? w.sstart[mid + 1] : tot;
        if (end > target) hi = mid;
        else lo = mid + 1;
    }
    __shared__ double sbuf[8][kSeqChunk];  // launched with 256 threads
    int64_t idx = n - 1;
    if (lo < G1) {
        const int64_t G = lo;
        const double sst = w.sstart[G];
        const double send = G + 1 < G1 ? w.sstart[G + 1] : tot;
        const int64_t cb = G * kSuper;
        double cst;  // exact start of this lane's chunk cb + lane
        if (w.sflag[G]) {
            const Grid g = grid_of(sst);
            const int64_t S0 = (int64_t)to_units(sst, g.k);
            const PMap m{w.q0[cb + lane], w.q1[cb + lane]};
            cst = from_units(pmap_apply(warp_exclusive(warp_scan_pmap(m)), S0), g.k);
        } else {
            cst = w.cstart[cb + lane];
        }
        const double nxt = __shfl_down_sync(0xffffffffu, cst, 1);  // (every lane shuffles)
        const double cend = lane + 1 < kSuper ? nxt : send;
        const unsigned hit_m = __ballot_sync(0xffffffffu, cend > target);
        const int cl = hit_m ? __ffs(hit_m) - 1 : kSuper - 1;
        double run = __shfl_sync(0xffffffffu, cst, cl);
        double a[kSeqPerLane];
        int64_t first;
        const int m = load_chunk(v, r, cb + cl, a, first);
        const int hit = warp_step_seq(a, m, run, target, true, sbuf[(threadIdx.x >> 5) & 7]);
        if (hit >= 0) idx = first - v.seg_off[r] + hit;
        if (idx >= n) idx = n - 1;  // (padding never exceeds the target; clip like :118)
    }
    if (lane == 0) chosen[(int64_t)r * k + i] = idx;
}

__global__ void k_kpp_round_on(int R, int i, const int32_t *__restrict__ start,
                               const int32_t *__restrict__ on, int32_t *__restrict__ round_on,
                               int32_t *__restrict__ neg) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    round_on[r] = on[r] && i >= start[r];
    neg[r] = 0;
}

// Round i pick, one warp per restart: target = u * cumsum[-1] (exact), then
// searchsorted(cumsum, target, 'right') clipped to n-1 (kmeans.py:116-118).  A zero total
// (every weight 0) is the degenerate branch (kmeans.py:128-134): reported to the host.
__global__ void k_kpp_search(SegView v, SeqWork w, int64_t n, int k, int i,
                             const double *__restrict__ u, int64_t *__restrict__ chosen,
                             int32_t *__restrict__ on, int32_t *__restrict__ degen) {
    const int lane = threadIdx.x & 31;
    const int r = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (r >= v.S || !seg_on(v, r)) return;
    const double tot = w.total[r];
    if (!(tot > 0.0)) {
        if (lane == 0) {
            degen[r] = i;
            on[r] = 0;
        }
        return;
    }
    const double target = __dmul_rn(u[(int64_t)r * (k - 1) + (i - 1)], tot);
    const int64_t c0 = v.cofs[r], c1 = v.cofs[r + 1];
    // first chunk whose end exceeds target: last chunk with cstart <= target ... then check
    int64_t lo = c0, hi = c1;  // find first chunk c with end(c) > target; end(c) = cstart[c+1]
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const double end = mid + 1 < c1 ? w.cstart[mid + 1] : tot;
        if (end > target) hi = mid;
        else lo = mid + 1;
    }
    __shared__ double sbuf[8][kSeqChunk];  // launched with 256 threads
    int64_t idx = n - 1;
    if (lo < c1) {
        double run = w.cstart[lo];
        double a[kSeqPerLane];
        int64_t first;
        const int m = load_chunk(v, r, lo, a, first);
        const int hit = warp_step_seq(a, m, run, target, true, sbuf[(threadIdx.x >> 5) & 7]);
        if (hit >= 0) idx = first - v.seg_off[r] + hit;
    }
    if (lane == 0) chosen[(int64_t)r * k + i] = idx;
}

// ---------------------------------------------------------------------------
// Lloyd

// assignment: labels, counts, changed vs previous labels
__global__ void k_assign(const double *__restrict__ x, int64_t n, int l, int k,
                         const double *__restrict__ cen, const int32_t *__restrict__ active,
                         const int32_t *__restrict__ prev, int32_t *__restrict__ lab,
                         int32_t *__restrict__ cnt, int32_t *__restrict__ changed) {
    const int r = blockIdx.y;
    if (!active[r]) return;
    extern __shared__ unsigned char smem_raw[];
    double *c = reinterpret_cast<double *>(smem_raw);
    int32_t *hist = reinterpret_cast<int32_t *>(c + (size_t)k * l);
    for (int i = threadIdx.x; i < k * l; i += blockDim.x) c[i] = cen[(int64_t)r * k * l + i];
    for (int i = threadIdx.x; i < k; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    int ch = 0;
    const int32_t *pv = prev + (int64_t)r * n;
    int32_t *lb = lab + (int64_t)r * n;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double *xj = x + j * l;
        int bi = 0;
        double bd = d2nd(xj, c, l);
        for (int q = 1; q < k; ++q) {
            const double d = d2nd(xj, c + (size_t)q * l, l);
            if (d < bd) {
                bd = d;
                bi = q;
            }
        }
        lb[j] = bi;
        ch += (pv[j] != bi);
        atomicAdd(&hist[bi], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += blockDim.x)
        if (hist[i]) atomicAdd(&cnt[(int64_t)r * k + i], hist[i]);
    // warp-aggregate the changed count
    for (int o = 16; o; o >>= 1) ch += __shfl_xor_sync(0xffffffffu, ch, o);
    if ((threadIdx.x & 31) == 0 && ch) atomicAdd(&changed[r], ch);
}

// l == 1: the point is loaded once and the k centers come from shared memory; each point's
// work is k (sub, mul, compare) -- the generic kernel re-read x from global per center.  Two
// points per thread keep two independent compare chains in flight.
__global__ void __launch_bounds__(256) k_assign1(const double *__restrict__ x, int64_t n, int k,
                                                 const double *__restrict__ cen,
                                                 const int32_t *__restrict__ active,
                                                 const int32_t *__restrict__ prev,
                                                 int32_t *__restrict__ lab, int32_t *__restrict__ cnt,
                                                 int32_t *__restrict__ changed) {
    const int r = blockIdx.y;
    if (!active[r]) return;
    extern __shared__ unsigned char smem_raw[];
    double *c = reinterpret_cast<double *>(smem_raw);
    int32_t *hist = reinterpret_cast<int32_t *>(c + k);
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        c[i] = cen[(int64_t)r * k + i];
        hist[i] = 0;
    }
    __syncthreads();
    int ch = 0;
    const int32_t *pv = prev + (int64_t)r * n;
    int32_t *lb = lab + (int64_t)r * n;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += 2 * stride) {
        const int64_t j2 = j + stride;
        const bool two = j2 < n;
        const double xa = __ldg(x + j), xb = two ? __ldg(x + j2) : 0.0;
        const int32_t pa = __ldcs(pv + j), pb = two ? __ldcs(pv + j2) : 0;
        int ba = 0, bb = 0;
        double da = d2ref(xa, c[0]), db = d2ref(xb, c[0]);
        for (int q = 1; q < k; ++q) {
            const double cq = c[q];
            const double ea = d2ref(xa, cq), eb = d2ref(xb, cq);
            if (ea < da) {
                da = ea;
                ba = q;
            }
            if (eb < db) {
                db = eb;
                bb = q;
            }
        }
        __stcs(lb + j, ba);
        ch += (pa != ba);
        atomicAdd(&hist[ba], 1);
        if (two) {
            __stcs(lb + j2, bb);
            ch += (pb != bb);
            atomicAdd(&hist[bb], 1);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += blockDim.x)
        if (hist[i]) atomicAdd(&cnt[(int64_t)r * k + i], hist[i]);
    for (int o = 16; o; o >>= 1) ch += __shfl_xor_sync(0xffffffffu, ch, o);
    if ((threadIdx.x & 31) == 0 && ch) atomicAdd(&changed[r], ch);
}

// _repair_empty for all restarts with one cooperative grid (used when n is large): the
// per-empty-cluster argmax over the n own-distances is a grid-wide reduction instead of one
// CTA's scan, so a repair costs ~n/(SMs x bandwidth) instead of n/(one SM).  Same semantics
// as k_repair: clusters empty after assignment, in increasing order, each takes the first
// point of maximal own distance, whose own distance then becomes 0; counts and the
// changed-label count are recomputed for the repaired restarts.
constexpr int kRepairTPB = 512;
constexpr int64_t kCoopRepairMinN = 200000;  // below this one CTA per restart is cheaper
constexpr int kRepairMaxK = 16384;           // shared-memory histogram bins

__global__ void __launch_bounds__(kRepairTPB) k_repair_coop(
    const double *__restrict__ x, int64_t n, int l, int k, const double *__restrict__ cen,
    const int32_t *__restrict__ active, const int32_t *__restrict__ prev, int32_t *__restrict__ lab,
    int32_t *__restrict__ cnt, int32_t *__restrict__ changed, double *__restrict__ own_all,
    int32_t *__restrict__ elist, int32_t *__restrict__ mlist, double *__restrict__ pval,
    int64_t *__restrict__ pidx, int R) {
    cg::grid_group grid = cg::this_grid();
    const int G = gridDim.x, b = blockIdx.x;
    __shared__ int base;
    __shared__ double sv[kRepairTPB / 32];
    __shared__ int64_t si[kRepairTPB / 32];
    // phase 0: ordered list of the empty clusters of every active restart
    for (int r = b; r < R; r += G) {
        if (threadIdx.x == 0) base = 0;
        __syncthreads();
        if (active[r]) {
            for (int c0 = 0; c0 < k; c0 += blockDim.x) {
                const int c = c0 + threadIdx.x;
                const bool e = c < k && cnt[(int64_t)r * k + c] == 0;
                // block-ordered compaction: warp ballots, then warps in order
                const unsigned bal = __ballot_sync(0xffffffffu, e);
                __shared__ int wcnt[kRepairTPB / 32];
                if ((threadIdx.x & 31) == 0) wcnt[threadIdx.x >> 5] = __popc(bal);
                __syncthreads();
                int off = base;
                for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) off += wcnt[w];
                if (e) elist[(int64_t)r * k + off + __popc(bal & ((1u << (threadIdx.x & 31)) - 1))] = c;
                __syncthreads();
                if (threadIdx.x == 0)
                    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) base += wcnt[w];
                __syncthreads();
            }
        }
        if (threadIdx.x == 0) mlist[r] = active[r] ? base : 0;
        __syncthreads();
    }
    grid.sync();
    int mm = 0;
    for (int r = 0; r < R; ++r) mm = max(mm, mlist[r]);
    if (mm == 0) return;  // uniform across the grid
    // phase 1: own distances of the restarts that repair
    const int64_t tid = (int64_t)b * blockDim.x + threadIdx.x, nth = (int64_t)G * blockDim.x;
    for (int64_t t = tid; t < (int64_t)R * n; t += nth) {
        const int r = (int)(t / n);
        if (mlist[r] == 0) continue;
        const int64_t j = t - (int64_t)r * n;
        own_all[t] = d2nd(x + j * l, cen + ((int64_t)r * k + lab[t]) * l, l);
    }
    grid.sync();
    for (int i = 0; i < mm; ++i) {
        // phase A: per-block partial argmax (value desc, index asc) for every repairing restart
        for (int r = 0; r < R; ++r) {
            if (i >= mlist[r]) continue;
            const double *own = own_all + (int64_t)r * n;
            double bv = -1.0;
            int64_t bj = n;
            for (int64_t j = tid; j < n; j += nth) {
                const double v = own[j];
                if (v > bv) {
                    bv = v;
                    bj = j;
                }
            }
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int64_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
                if (ov > bv || (ov == bv && oj < bj)) {
                    bv = ov;
                    bj = oj;
                }
            }
            if ((threadIdx.x & 31) == 0) {
                sv[threadIdx.x >> 5] = bv;
                si[threadIdx.x >> 5] = bj;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                    if (sv[w] > sv[0] || (sv[w] == sv[0] && si[w] < si[0])) {
                        sv[0] = sv[w];
                        si[0] = si[w];
                    }
                pval[(int64_t)r * G + b] = sv[0];
                pidx[(int64_t)r * G + b] = si[0];
            }
            __syncthreads();
        }
        grid.sync();
        // phase B: one thread per repairing restart combines the partials and moves the point
        if (b == 0)
            for (int r = threadIdx.x; r < R; r += blockDim.x) {
                if (i >= mlist[r]) continue;
                double bv = -1.0;
                int64_t bj = n;
                for (int q = 0; q < G; ++q) {
                    const double v = pval[(int64_t)r * G + q];
                    const int64_t j = pidx[(int64_t)r * G + q];
                    if (v > bv || (v == bv && j < bj)) {
                        bv = v;
                        bj = j;
                    }
                }
                lab[(int64_t)r * n + bj] = elist[(int64_t)r * k + i];
                own_all[(int64_t)r * n + bj] = 0.0;
            }
        grid.sync();
    }
    // phase C: recount the repaired restarts
    for (int64_t t = tid; t < (int64_t)R * k; t += nth)
        if (mlist[t / k]) cnt[t] = 0;
    if (b == 0)
        for (int r = threadIdx.x; r < R; r += blockDim.x)
            if (mlist[r]) changed[r] = 0;
    grid.sync();
    // block-local histograms in shared memory (k bins), one global add per bin per block
    extern __shared__ int32_t hist[];
    for (int r = 0; r < R; ++r) {
        if (mlist[r] == 0) continue;
        for (int c = threadIdx.x; c < k; c += blockDim.x) hist[c] = 0;
        __syncthreads();
        int ch = 0;
        for (int64_t j = tid; j < n; j += nth) {
            const int32_t lb = lab[(int64_t)r * n + j];
            atomicAdd(&hist[lb], 1);
            ch += lb != prev[(int64_t)r * n + j];
        }
        for (int o = 16; o; o >>= 1) ch += __shfl_xor_sync(0xffffffffu, ch, o);
        if ((threadIdx.x & 31) == 0 && ch) atomicAdd(&changed[r], ch);
        __syncthreads();
        for (int c = threadIdx.x; c < k; c += blockDim.x)
            if (hist[c]) atomicAdd(&cnt[(int64_t)r * k + c], hist[c]);
        __syncthreads();
    }
}

// ---- assignment through sorted centers (k >= kSortedMinK) ------------------------------
// argmin_c d2ref(x, c) is found without evaluating all k centers.  With u = 2^-53 and
// D(c) = (x - c)^2 exact, d2ref's five roundings give |d2ref - D| <= 3.01 u (|x| + |c|)^2,
// and Dapprox(c) = fl(fl(x - c)^2) is within 3.01 u D of D and monotone in |x - c| on each
// side of x.  So every center with Dapprox(c) > Dapprox(c*) + 20 u (|x| + cmax)^2 (c* the
// nearest neighbour of x among the sorted centers) has d2ref(x, c) > d2ref(x, c*) and cannot
// be the argmin; the remaining window is contiguous in sorted order and evaluated exactly,
// ties going to the lowest original index -- the brute-force result, bit for bit.
constexpr int kSortedMinK = 16;
constexpr int kSortedMaxK = 4096;

// one CTA per active restart: bitonic sort of (value, original index), and max |c|
__global__ void __launch_bounds__(1024) k_sort_centers(int k, const double *__restrict__ cen,
                                                       const int32_t *__restrict__ active,
                                                       double *__restrict__ scen,
                                                       int32_t *__restrict__ sidx,
                                                       double *__restrict__ cmax) {
    const int r = blockIdx.x;
    if (!active[r]) return;
    extern __shared__ unsigned char sort_raw[];
    __shared__ double red[32];
    int P = 1;
    while (P < k) P <<= 1;
    double *v = reinterpret_cast<double *>(sort_raw);
    int32_t *ix = reinterpret_cast<int32_t *>(v + P);
    double mx = 0.0;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const double c = i < k ? cen[(int64_t)r * k + i] : INFINITY;
        v[i] = c;
        ix[i] = i < k ? i : INT32_MAX;
        if (i < k) mx = fmax(mx, fabs(c));
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const bool gt = v[i] > v[j] || (v[i] == v[j] && ix[i] > ix[j]);
                    if (gt == up) {
                        const double tv = v[i];
                        v[i] = v[j];
                        v[j] = tv;
                        const int32_t ti = ix[i];
                        ix[i] = ix[j];
                        ix[j] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        scen[(int64_t)r * k + i] = v[i];
        sidx[(int64_t)r * k + i] = ix[i];
    }
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int w = 0; w < (int)((blockDim.x + 31) >> 5); ++w) m = fmax(m, red[w]);
        cmax[r] = m;
    }
}

__global__ void k_assign_sorted(const double *__restrict__ x, int64_t n, int k,
                                const double *__restrict__ scen, const int32_t *__restrict__ sidx,
                                const double *__restrict__ cmax_r,
                                const int32_t *__restrict__ active,
                                const int32_t *__restrict__ prev, int32_t *__restrict__ lab,
                                int32_t *__restrict__ cnt, int32_t *__restrict__ changed) {
    const int r = blockIdx.y;
    if (!active[r]) return;
    extern __shared__ unsigned char smem_raw[];
    double *c = reinterpret_cast<double *>(smem_raw);
    int32_t *ci = reinterpret_cast<int32_t *>(c + k);
    int32_t *hist = ci + k;
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        c[i] = scen[(int64_t)r * k + i];
        ci[i] = sidx[(int64_t)r * k + i];
        hist[i] = 0;
    }
    const double cmax = cmax_r[r];
    __syncthreads();
    int ch = 0;
    const int32_t *pv = prev + (int64_t)r * n;
    int32_t *lb = lab + (int64_t)r * n;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double xj = x[j];
        // p = first sorted center >= xj
        int lo = 0, hi = k;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (c[mid] < xj) lo = mid + 1;
            else hi = mid;
        }
        const int p = lo;
        auto dap = [&](double cv) {
            const double t = __dsub_rn(xj, cv);
            return __dmul_rn(t, t);
        };
        double dstar = INFINITY;
        if (p > 0) dstar = dap(c[p - 1]);
        if (p < k) dstar = fmin(dstar, dap(c[p]));
        const double m = __dadd_rn(fabs(xj), cmax);
        const double thr = __dadd_rn(dstar, __dmul_rn(__dmul_rn(m, m), 20.0 * 1.1102230246251565e-16));
        int bi = INT32_MAX;
        double bd = INFINITY;
        auto take = [&](int q) {
            const double d = d2ref(xj, c[q]);
            const int id = ci[q];
            if (d < bd || (d == bd && id < bi)) {
                bd = d;
                bi = id;
            }
        };
        for (int q = p - 1; q >= 0 && dap(c[q]) <= thr; --q) take(q);
        for (int q = p; q < k && dap(c[q]) <= thr; ++q) take(q);
        lb[j] = bi;
        ch += (pv[j] != bi);
        atomicAdd(&hist[bi], 1);
    }
    __syncthreads();
    // hist is indexed by original center index
    for (int i = threadIdx.x; i < k; i += blockDim.x)
        if (hist[i]) atomicAdd(&cnt[(int64_t)r * k + i], hist[i]);
    for (int o = 16; o; o >>= 1) ch += __shfl_xor_sync(0xffffffffu, ch, o);
    if ((threadIdx.x & 31) == 0 && ch) atomicAdd(&changed[r], ch);
}

// _repair_empty (kmeans.py:151-164), one CTA per restart; returns at once when no
// cluster is empty (the common case).  Clusters empty after assignment are repaired in
// increasing order: the first point of maximal own distance moves in, its own distance
// becomes 0.  Then counts and the changed-label count of the restart are recomputed.
__global__ void __launch_bounds__(1024) k_repair(const double *__restrict__ x, int64_t n, int l,
                                                 int k,
                                                 const double *__restrict__ cen,
                                                 const int32_t *__restrict__ active,
                                                 const int32_t *__restrict__ prev,
                                                 int32_t *__restrict__ lab, int32_t *__restrict__ cnt,
                                                 int32_t *__restrict__ changed,
                                                 double *__restrict__ own_all) {
    const int r = blockIdx.x;
    if (!active[r]) return;
    extern __shared__ unsigned char smem_raw[];
    unsigned char *was_empty = smem_raw;  // k flags
    __shared__ int has;
    __shared__ double sv[32];
    __shared__ int64_t si[32];
    if (threadIdx.x == 0) has = 0;
    __syncthreads();
    int32_t *ct = cnt + (int64_t)r * k;
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        was_empty[c] = ct[c] == 0;
        if (was_empty[c]) has = 1;
    }
    __syncthreads();
    if (!has) return;
    int32_t *lb = lab + (int64_t)r * n;
    const double *cc = cen + (int64_t)r * k * l;
    double *own = own_all + (int64_t)r * n;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x)
        own[j] = d2nd(x + j * l, cc + (int64_t)lb[j] * l, l);
    __syncthreads();
    for (int e = 0; e < k; ++e) {
        if (!was_empty[e]) continue;
        double bv = -1.0;
        int64_t bj = n;
        for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
            const double v = own[j];
            if (v > bv) {
                bv = v;
                bj = j;
            }
        }
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int64_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (ov > bv || (ov == bv && oj < bj)) {
                bv = ov;
                bj = oj;
            }
        }
        if ((threadIdx.x & 31) == 0) {
            sv[threadIdx.x >> 5] = bv;
            si[threadIdx.x >> 5] = bj;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                if (sv[w] > sv[0] || (sv[w] == sv[0] && si[w] < si[0])) {
                    sv[0] = sv[w];
                    si[0] = si[w];
                }
            const int64_t far = si[0];
            lb[far] = e;
            own[far] = 0.0;
        }
        __syncthreads();
    }
    for (int c = threadIdx.x; c < k; c += blockDim.x) ct[c] = 0;
    if (threadIdx.x == 0) changed[r] = 0;
    __syncthreads();
    const int32_t *pv = prev + (int64_t)r * n;
    int ch = 0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
        atomicAdd(&ct[lb[j]], 1);
        ch += lb[j] != pv[j];
    }
    for (int o = 16; o; o >>= 1) ch += __shfl_xor_sync(0xffffffffu, ch, o);
    if ((threadIdx.x & 31) == 0 && ch) atomicAdd(&changed[r], ch);
}

// sort keys for the still-active restarts only: slot s = s-th active restart (act[s]),
// key = s*k + label, value = the point (a stable sort then keeps point-index order inside
// every (restart, cluster) segment -- the np.add.at order)
__global__ void k_make_keys(int64_t n, int k, const int32_t *__restrict__ lab,
                            const int32_t *__restrict__ act, int nact, int32_t *__restrict__ keys,
                            double *__restrict__ vals, const double *__restrict__ x) {
    const int64_t tot = (int64_t)nact * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / n, j = t - s * n;
        keys[t] = (int32_t)(s * k + lab[(int64_t)act[s] * n + j]);
        vals[t] = x[j];
    }
}

// ---- stable counting sort of the points by (slot, label) for small key counts ----------
// Replaces key construction + radix sort when nseg <= kCsMaxKeys: a tile histogram pass, an
// exclusive scan of the (key, tile) counts, and a scatter that ranks equal keys in point
// order inside the tile (warp match + per-warp running counters), so the output is exactly
// the stable sort's (np.add.at order preserved).
constexpr int kCsTile = 4096, kCsWarps = 8, kCsMaxKeys = 1024;

// Slot of element t of a tile [t0, t0 + kCsTile): the tile's slots are s0, s0 + 1, ... with
// boundaries edge, edge + n, ...; walking them replaces a 64-bit division per element (a tile
// spans one or two slots whenever n >= kCsTile).
struct CsSlot {
    int64_t s0, edge;
    __device__ CsSlot(int64_t t0, int64_t n) : s0(t0 / n), edge((t0 / n + 1) * n) {}
    __device__ __forceinline__ int64_t slot(int64_t t, int64_t n) const {
        int64_t s = s0, e = edge;
        while (t >= e) {
            ++s;
            e += n;
        }
        return s;
    }
};

__device__ __forceinline__ int cs_key(const CsSlot &sl, int64_t t, int64_t n, int k,
                                      const int32_t *lab, const int32_t *act, int64_t *jout = nullptr) {
    const int64_t s = sl.slot(t, n), j = t - s * n;
    if (jout) *jout = j;
    return (int)(s * k + lab[(int64_t)act[s] * n + j]);
}

template <int TILE = kCsTile>
__global__ void __launch_bounds__(32 * kCsWarps) k_cs_hist(int64_t m, int64_t n, int k,
                                                           const int32_t *__restrict__ lab,
                                                           const int32_t *__restrict__ act,
                                                           int nseg, int ntiles,
                                                           int32_t *__restrict__ bh) {
    extern __shared__ int32_t cs_h[];
    for (int q = threadIdx.x; q < nseg; q += blockDim.x) cs_h[q] = 0;
    __syncthreads();
    const int64_t t0 = (int64_t)blockIdx.x * TILE;
    const CsSlot sl(t0, n);
    for (int64_t t = t0 + threadIdx.x; t < min(m, t0 + TILE); t += blockDim.x)
        atomicAdd(&cs_h[cs_key(sl, t, n, k, lab, act)], 1);
    __syncthreads();
    for (int q = threadIdx.x; q < nseg; q += blockDim.x)
        bh[(int64_t)q * ntiles + blockIdx.x] = cs_h[q];
}

template <int TILE = kCsTile>
__global__ void __launch_bounds__(32 * kCsWarps) k_cs_scatter(
    int64_t m, int64_t n, int k, const int32_t *__restrict__ lab, const int32_t *__restrict__ act,
    int nseg, int ntiles, const int32_t *__restrict__ off, const double *__restrict__ x,
    double *__restrict__ out) {
    extern __shared__ int32_t cs_s[];  // [kCsWarps][nseg] counts, then running positions
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t *run = cs_s + w * nseg;
    for (int q = threadIdx.x; q < kCsWarps * nseg; q += blockDim.x) cs_s[q] = 0;
    __syncthreads();
    const int64_t t0 = (int64_t)blockIdx.x * TILE;
    constexpr int SUB = TILE / kCsWarps;
    const int64_t s0 = t0 + (int64_t)w * SUB, s1 = min(m, s0 + SUB);
    const CsSlot sl(t0, n);
    for (int64_t t = s0 + lane; t < s1; t += 32) atomicAdd(&run[cs_key(sl, t, n, k, lab, act)], 1);
    __syncthreads();
    // exclusive prefix over warps per key, plus the tile's global offset
    for (int q = threadIdx.x; q < nseg; q += blockDim.x) {
        int acc = off[(int64_t)q * ntiles + blockIdx.x];
        for (int ww = 0; ww < kCsWarps; ++ww) {
            const int c = cs_s[ww * nseg + q];
            cs_s[ww * nseg + q] = acc;
            acc += c;
        }
    }
    __syncthreads();
    for (int64_t b = s0; b < s1; b += 32) {
        const int64_t t = b + lane;
        const bool ok = t < s1;
        int64_t j = 0;
        const int key = ok ? cs_key(sl, t, n, k, lab, act, &j) : -1 - lane;
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        const int rank = __popc(peers & ((1u << lane) - 1));
        if (ok) out[run[key] + rank] = x[j];
        __syncwarp();
        if (ok && rank == 0) run[key] += __popc(peers);  // leader: lowest lane of the group
        __syncwarp();
    }
}

// l > 1: the sort carries the point index; each coordinate is gathered in sorted order
__global__ void k_make_keys_idx(int64_t n, int k, const int32_t *__restrict__ lab,
                                const int32_t *__restrict__ act, int nact,
                                int32_t *__restrict__ keys, int32_t *__restrict__ idx) {
    const int64_t tot = (int64_t)nact * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / n, j = t - s * n;
        keys[t] = (int32_t)(s * k + lab[(int64_t)act[s] * n + j]);
        idx[t] = (int32_t)j;
    }
}

__global__ void k_gather_coord(const double *__restrict__ x, const int32_t *__restrict__ idx,
                               int64_t m, int l, int q, double *__restrict__ vals) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
         t += (int64_t)gridDim.x * blockDim.x)
        vals[t] = x[(int64_t)idx[t] * l + q];
}

// Layout of the (slot, cluster) segments of the sorted points, straight from the cluster
// counts (k_assign / k_repair leave them consistent with the labels): seg = exclusive scan
// of the counts in (active slot, label) order -- the order of the sort keys -- and cofs the
// same over ceil(count / kSeqChunk) chunks.  One CTA, 1024 segments per round.
__global__ void __launch_bounds__(1024) k_seg_layout(int nseg, int k,
                                                     const int32_t *__restrict__ cnt,
                                                     const int32_t *__restrict__ act,
                                                     int64_t *__restrict__ seg,
                                                     int64_t *__restrict__ cofs,
                                                     int64_t *__restrict__ total) {
    __shared__ int64_t pl[1024], pc[1024];
    int64_t carry_l = 0, carry_c = 0;
    for (int base = 0; base < nseg; base += 1024) {
        const int i = base + threadIdx.x;
        const int64_t len = i < nseg ? cnt[(int64_t)act[i / k] * k + i % k] : 0;
        const int64_t ch = (len + kSeqChunk - 1) / kSeqChunk;
        pl[threadIdx.x] = len;
        pc[threadIdx.x] = ch;
        __syncthreads();
        for (int d = 1; d < 1024; d <<= 1) {
            const int64_t ol = threadIdx.x >= d ? pl[threadIdx.x - d] : 0;
            const int64_t oc = threadIdx.x >= d ? pc[threadIdx.x - d] : 0;
            __syncthreads();
            pl[threadIdx.x] += ol;
            pc[threadIdx.x] += oc;
            __syncthreads();
        }
        if (i < nseg) {
            seg[i] = carry_l + pl[threadIdx.x] - len;
            cofs[i] = carry_c + pc[threadIdx.x] - ch;
        }
        carry_l += pl[1023];
        carry_c += pc[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        seg[nseg] = carry_l;
        cofs[nseg] = carry_c;
        *total = carry_c;
    }
}

// means = ordered sum / count (cluster_means, kmeans.py:86-93); empty clusters keep 0
__global__ void k_seg_means(int nseg, int k, int l, int q, const int64_t *__restrict__ seg,
                            const double *__restrict__ total, const int32_t *__restrict__ act,
                            double *__restrict__ cen) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nseg) return;
    const int64_t c = seg[t + 1] - seg[t];
    cen[((int64_t)act[t / k] * k + t % k) * l + q] = c > 0 ? __ddiv_rn(total[t], (double)c) : 0.0;
}

// kmeans_cost in numpy einsum("ij,ij->") order (sc_oracle.c orc_einsum_sumsq): one warp
// per (restart, 8192-element buffer).  The warp stages the squared deviations
// fl(fl(x - c_label)^2) 256 at a time (coalesced, double-buffered in its shared-memory slot)
// while lanes 0 and 1 run the two SSE lane chains (8 elements per step in the order 6|7,
// 4|5, 2|3, 0|1, tail with zero fill) over the previous 256 at the FP64 add latency.  Many
// small warps instead of one 64 KB CTA per buffer keep every chain of the batch in flight.
constexpr int kCostWarps = 8;
constexpr int kCostChunk = 256;

// (points of dimension l: the buffers run over the n*l coordinates in C order, as numpy's
// nditer does for the (n, l) operands)
__global__ void __launch_bounds__(32 * kCostWarps) k_cost_buf(
    const double *__restrict__ x, int64_t n, int l, int k, const int32_t *__restrict__ lab,
    const double *__restrict__ cen, const int32_t *__restrict__ active, int64_t nbuf,
    double *__restrict__ part) {
    __shared__ double sq[kCostWarps][2][kCostChunk];
    const int r = blockIdx.y;
    if (!active[r]) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t bufi = (int64_t)blockIdx.x * kCostWarps + wib;
    if (bufi >= nbuf) return;
    const int64_t base = bufi * kEinsumBuf, nl = n * l;
    const int m = (int)min((int64_t)kEinsumBuf, nl - base);
    const int32_t *lr = lab + (int64_t)r * n;
    const double *c = cen + (int64_t)r * k * l;
    const double *xb0 = x + base;
    // raw loads of chunk q+2 are issued before the chains of chunk q and the dependent
    // center lookup of chunk q+1 runs after them, so no lane waits on HBM in between
    constexpr int PL = kCostChunk / 32;
    double xa[PL], xb[PL], v[PL];
    int32_t la[PL], lbv[PL];
    auto raw = [&](int q, double (&xv)[PL], int32_t (&lv)[PL]) {
#pragma unroll
        for (int t = 0; t < PL; ++t) {
            const int j = q * kCostChunk + t * 32 + lane;
            const int64_t e = base + j;
            xv[t] = j < m ? __ldg(xb0 + j) : 0.0;
            lv[t] = j >= m ? -1 : (l == 1 ? __ldcs(lr + e) : lr[e / l] * l + (int)(e % l));
        }
    };
    auto finish = [&](const double (&xv)[PL], const int32_t (&lv)[PL]) {
#pragma unroll
        for (int t = 0; t < PL; ++t) {
            v[t] = 0.0;
            if (lv[t] >= 0) {
                const double d = __dsub_rn(xv[t], c[lv[t]]);
                v[t] = __dmul_rn(d, d);
            }
        }
    };
    const int nq = (m + kCostChunk - 1) / kCostChunk;
    raw(0, xa, la);
    if (nq > 1) raw(1, xb, lbv);
    finish(xa, la);
    double acc = 0.0;
    for (int q = 0; q < nq; ++q) {
        double *cur = sq[wib][q & 1];
#pragma unroll
        for (int t = 0; t < PL; ++t) cur[t * 32 + lane] = v[t];
        __syncwarp();
        if (q + 2 < nq) raw(q + 2, xa, la);  // chunk q's raw registers are free again
        if (lane < 2) {
            const int mm = min(kCostChunk, m - q * kCostChunk);
            if (mm == kCostChunk) {
                // full chunk: 32 steps, the next step's four operands are read from shared
                // memory while the current four are added (the chain is the only latency)
                double p6 = cur[6 + lane], p4 = cur[4 + lane], p2 = cur[2 + lane], p0 = cur[lane];
#pragma unroll 4
                for (int i = 8; i <= kCostChunk; i += 8) {
                    double n6 = 0.0, n4 = 0.0, n2 = 0.0, n0 = 0.0;
                    if (i < kCostChunk) {
                        n6 = cur[i + 6 + lane];
                        n4 = cur[i + 4 + lane];
                        n2 = cur[i + 2 + lane];
                        n0 = cur[i + lane];
                    }
                    acc = __dadd_rn(p6, acc);
                    acc = __dadd_rn(p4, acc);
                    acc = __dadd_rn(p2, acc);
                    acc = __dadd_rn(p0, acc);
                    p6 = n6;
                    p4 = n4;
                    p2 = n2;
                    p0 = n0;
                }
            } else {
                int i = 0;
                for (; mm - i >= 8; i += 8) {
                    acc = __dadd_rn(cur[i + 6 + lane], acc);
                    acc = __dadd_rn(cur[i + 4 + lane], acc);
                    acc = __dadd_rn(cur[i + 2 + lane], acc);
                    acc = __dadd_rn(cur[i + lane], acc);
                }
                for (; i < mm; i += 2) acc = __dadd_rn(i + lane < mm ? cur[i + lane] : 0.0, acc);
            }
        }
        if (q + 1 < nq) finish(xb, lbv);
#pragma unroll
        for (int t = 0; t < PL; ++t) {  // rotate: chunk q+2 becomes "next"
            const double tx = xa[t];
            xa[t] = xb[t];
            xb[t] = tx;
            const int32_t tl = la[t];
            la[t] = lbv[t];
            lbv[t] = tl;
        }
        __syncwarp();
    }
    if (lane < 2) part[((int64_t)r * nbuf + bufi) * 2 + lane] = acc;
}

// buffer totals (l0 + l1) added into the running output in buffer order
// (the partials are staged in shared memory by the whole CTA first, so the sequential chain
// runs at the add latency rather than one global-load latency per buffer)
constexpr int kCombineStage = 2048;  // buffers per staging round (2 partials each)

__global__ void k_cost_combine(int64_t nbuf, const double *__restrict__ part,
                               const int32_t *__restrict__ active, double *__restrict__ cost) {
    __shared__ double sp[2 * kCombineStage];
    const int r = blockIdx.x;
    if (!active[r]) return;
    double out = 0.0;
    const double *p = part + (int64_t)r * nbuf * 2;
    for (int64_t b0 = 0; b0 < nbuf; b0 += kCombineStage) {
        const int nb = (int)(nbuf - b0 < kCombineStage ? nbuf - b0 : kCombineStage);
        __syncthreads();
        for (int t = threadIdx.x; t < 2 * nb; t += blockDim.x) sp[t] = p[2 * b0 + t];
        __syncthreads();
        if (threadIdx.x == 0)
            for (int b = 0; b < nb; ++b) out = __dadd_rn(__dadd_rn(sp[2 * b], sp[2 * b + 1]), out);
    }
    if (threadIdx.x == 0) cost[r] = out;
}

__global__ void k_gather_centers(const double *__restrict__ x, const int64_t *__restrict__ chosen,
                                 int rk, int l, double *__restrict__ cen) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < rk * l) cen[t] = x[chosen[t / l] * l + t % l];
}

template <typename T>
static int32_t grow(T **p, size_t count, cudaStream_t s) {
    // stream-ordered allocations from the device's default pool (kept warm, see km_init):
    // repeated clusterings reuse the pool instead of paying cudaMalloc/cudaFree each time
    if (*p) cudaFreeAsync(*p, s);
    *p = nullptr;
    cudaError_t e = cudaMallocAsync((void **)p, std::max<size_t>(count, 1) * sizeof(T), s);
    if (e != cudaSuccess)
        return fail(e == cudaErrorMemoryAllocation ? SC_E_OOM : SC_E_CUDA, "cudaMalloc: %s",
                    cudaGetErrorString(e));
    return SC_OK;
}

static int32_t ensure(sc_kmeans *km, int R, int k) {
    if (R <= km->cap_r && k <= km->cap_k) return SC_OK;
    R = std::max(R, km->cap_r);
    k = std::max(k, km->cap_k);
    const int64_t n = km->n;
    const int64_t nbuf = (n * km->l + kEinsumBuf - 1) / kEinsumBuf;
    // chunks: kpp uses R * ceil(n/C); Lloyd's R*k segments need at most R*n/C + R*k
    // k-means++ lays restart r's D^2 weights out at best + r * nb, nb = n rounded up to a
    // super-chunk, so every super-chunk lies inside one restart (zero padding)
    const int64_t nb = kpp_stride(n);
    const int64_t nch = (int64_t)R * (nb / kSeqChunk) + (int64_t)R * k + 1;
    const int64_t S = (int64_t)R * k + 1;
    int32_t st;
    if ((st = grow(&km->d_best, (size_t)R * nb, km->stream))) return st;
    if ((st = grow(&km->d_lab[0], (size_t)R * n, km->stream))) return st;
    if ((st = grow(&km->d_lab[1], (size_t)R * n, km->stream))) return st;
    if ((st = grow(&km->d_keys, (size_t)R * n, km->stream))) return st;
    if ((st = grow(&km->d_keys_alt, (size_t)R * n, km->stream))) return st;
    if ((st = grow(&km->d_vals, (size_t)R * n, km->stream))) return st;
    if ((st = grow(&km->d_vals_alt, (size_t)R * n, km->stream))) return st;
    if ((st = grow(&km->d_chosen, (size_t)R * k, km->stream))) return st;
    if ((st = grow(&km->d_u, (size_t)R * k, km->stream))) return st;
    if ((st = grow(&km->d_start, (size_t)R, km->stream))) return st;
    if ((st = grow(&km->d_degen, (size_t)R, km->stream))) return st;
    if ((st = grow(&km->d_cen, (size_t)2 * R * k * km->l, km->stream))) return st;
    if (km->l > 1) {
        if ((st = grow(&km->d_idx, (size_t)R * n, km->stream))) return st;
        if ((st = grow(&km->d_idx_alt, (size_t)R * n, km->stream))) return st;
    }
    if ((st = grow(&km->d_scen, (size_t)R * k, km->stream))) return st;
    if ((st = grow(&km->d_sidx, (size_t)R * k, km->stream))) return st;
    if ((st = grow(&km->d_cmax, (size_t)R, km->stream))) return st;
    if ((st = grow(&km->d_elist, (size_t)R * k, km->stream))) return st;
    if ((st = grow(&km->d_mlist, (size_t)R, km->stream))) return st;
    if (!km->coop_grid) {
        int per = 0;
        cudaFuncSetAttribute(k_repair_coop, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kRepairMaxK * 4);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_repair_coop, kRepairTPB,
                                                      kRepairMaxK * 4);
        km->coop_grid = std::max(1, per) * km->sm_count;
    }
    if ((st = grow(&km->d_pval, (size_t)R * km->coop_grid, km->stream))) return st;
    if ((st = grow(&km->d_pidx, (size_t)R * km->coop_grid, km->stream))) return st;
    if ((st = grow(&km->d_cnt, (size_t)R * k, km->stream))) return st;
    if ((st = grow(&km->d_seg, (size_t)S, km->stream))) return st;
    if ((st = grow(&km->d_part, (size_t)R * nbuf * 2, km->stream))) return st;
    if ((st = grow(&km->d_cost, (size_t)R, km->stream))) return st;
    if ((st = grow(&km->d_changed, (size_t)2 * R, km->stream))) return st;
    if ((st = grow(&km->d_active, (size_t)2 * R, km->stream))) return st;
    if (R > km->cap_host_r) {
        // page-locked result/flag slots: each context owns one block drawn from a
        // process-wide pool (cudaMallocHost per clustering would cost milliseconds); a block
        // goes back to the pool only when its context grows or is destroyed, so no other
        // context ever holds a pointer into it
        const size_t need = (size_t)R * (16 + 8 + 16);
        unsigned char *blk = pinned_take(need);
        if (!blk) return fail(SC_E_OOM, "pinned host buffers");
        if (km->h_block) pinned_give(km->h_block, km->h_block_bytes);
        km->h_block = blk;
        km->h_block_bytes = need;
        km->h_cost = reinterpret_cast<double *>(blk);
        km->h_changed = reinterpret_cast<int32_t *>(blk + (size_t)R * 16);
        km->h_act = reinterpret_cast<int32_t *>(blk + (size_t)R * 24);
        km->cap_host_r = R;
    }
    if ((st = grow(&km->d_empty, (size_t)R, km->stream))) return st;
    if ((st = grow(&km->d_A, (size_t)nch, km->stream))) return st;
    if ((st = grow(&km->d_a64, (size_t)nch, km->stream))) return st;
    if ((st = grow(&km->d_vmax, (size_t)nch, km->stream))) return st;
    if ((st = grow(&km->d_cstart, (size_t)nch, km->stream))) return st;
    if ((st = grow(&km->d_kpred, (size_t)nch, km->stream))) return st;
    if ((st = grow(&km->d_q0, (size_t)nch, km->stream))) return st;
    if ((st = grow(&km->d_q1, (size_t)nch, km->stream))) return st;
    if ((st = grow(&km->d_sq0, (size_t)nch / kSuper + 1, km->stream))) return st;
    if ((st = grow(&km->d_sq1, (size_t)nch / kSuper + 1, km->stream))) return st;
    if ((st = grow(&km->d_svmax, (size_t)nch / kSuper + 1, km->stream))) return st;
    if ((st = grow(&km->d_skp, (size_t)nch / kSuper + 1, km->stream))) return st;
    if ((st = grow(&km->d_kmap, (size_t)nch, km->stream))) return st;
    if ((st = grow(&km->d_sstart, (size_t)nch / kSuper + 1, km->stream))) return st;
    if ((st = grow(&km->d_sflag, (size_t)nch / kSuper + 1, km->stream))) return st;
    if ((st = grow(&km->d_total, (size_t)S, km->stream))) return st;
    if ((st = grow(&km->d_neg, (size_t)S, km->stream))) return st;
    if ((st = grow(&km->d_cofs, (size_t)S + 1, km->stream))) return st;
    if ((st = grow(&km->d_nchunks, 1, km->stream))) return st;
    if ((st = grow(&km->d_round_on, (size_t)R, km->stream))) return st;
    if ((st = grow(&km->d_on, (size_t)R, km->stream))) return st;
    if ((st = grow(&km->d_segkpp, (size_t)R + 1, km->stream))) return st;
    size_t need = 0, need2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, km->d_keys, km->d_keys_alt, km->d_vals,
                                    km->d_vals_alt, (int64_t)R * n, 0, 31, km->stream);
    cub::DeviceRadixSort::SortPairs(nullptr, need2, km->d_keys, km->d_keys_alt, km->d_idx,
                                    km->d_idx_alt, (int64_t)R * n, 0, 31, km->stream);
    need = std::max(need, need2);
    size_t need3 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need3, km->d_keys, km->d_keys_alt, (int64_t)R * n,
                                  km->stream);
    need = std::max(need, need3);
    if ((st = grow((unsigned char **)&km->d_cub, need, km->stream))) return st;
    km->cub_bytes = need;
    km->cap_r = R;
    km->cap_k = k;
    km->cap_chunks = nch;
    return SC_OK;
}

static SeqWork seq_work(sc_kmeans *km) {
    SeqWork w;
    w.A = km->d_A;
    w.vmax = km->d_vmax;
    w.kpred = km->d_kpred;
    w.q0 = km->d_q0;
    w.q1 = km->d_q1;
    w.cstart = km->d_cstart;
    w.neg = km->d_neg;
    w.total = km->d_total;
    w.sq0 = km->d_sq0;
    w.sq1 = km->d_sq1;
    w.svmax = km->d_svmax;
    w.skp = km->d_skp;
    w.sstart = km->d_sstart;
    w.sflag = km->d_sflag;
    return w;
}

static int grid_1d(const sc_kmeans *km, int64_t work, int tpb) {
    const int64_t want = (work + tpb - 1) / tpb;
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)km->sm_count * 8));
}

static int32_t km_init(int device, int64_t n, int l, sc_kmeans **out) {
    sc_kmeans *km = new sc_kmeans();
    km->device = device;
    km->n = n;
    km->l = l;
    cudaDeviceGetAttribute(&km->sm_count, cudaDevAttrMultiProcessorCount, device);
    // keep freed workspace memory in the device pool across contexts (repeated clusterings)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaError_t e = cudaStreamCreateWithFlags(&km->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&km->stream2, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&km->ev_main, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&km->ev_cost, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMallocAsync((void **)&km->d_x, (size_t)n * l * 8, km->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(km->stream);
    if (e != cudaSuccess) {
        sc_kmeans_destroy(km);
        return fail(SC_E_CUDA, "k-means context: %s", cudaGetErrorString(e));
    }
    *out = km;
    return SC_OK;
}

}  // namespace sc

using namespace sc;

extern "C" {

int32_t sc_kmeans_create_nd(const double *points_host, int64_t n, int32_t l, int32_t device,
                            sc_kmeans **out) {
    SC_REQUIRE(out && points_host, SC_E_INVALID, "null argument");
    SC_REQUIRE(n >= 1, SC_E_INVALID, "need n >= 1 points");
    SC_REQUIRE(l >= 1 && l <= 64, SC_E_INVALID, "point dimension %d outside [1, 64]", l);
    SC_REQUIRE(n < (int64_t(1) << 31), SC_E_INVALID, "n too large");
    for (int64_t i = 0; i < n * l; ++i)
        SC_REQUIRE(std::isfinite(points_host[i]), SC_E_INVALID, "points contain NaN or Inf");
    SC_CUDA(cudaSetDevice(device));
    int32_t st = km_init(device, n, l, out);
    if (st) return st;
    SC_CUDA(cudaMemcpy((*out)->d_x, points_host, (size_t)n * l * 8, cudaMemcpyHostToDevice));
    return SC_OK;
}

int32_t sc_kmeans_create(const double *points_host, int64_t n, int32_t device,
                         sc_kmeans **out) {
    return sc_kmeans_create_nd(points_host, n, 1, device, out);
}

int32_t sc_kmeans_create_from_graph(sc_graph *g, sc_kmeans **out) {
    SC_REQUIRE(g && out, SC_E_INVALID, "null argument");
    const double *f = graph_f_device(g);
    SC_REQUIRE(f, SC_E_STATE, "graph has no embedding yet: call sc_power_iterate first");
    SC_CUDA(cudaSetDevice(graph_device(g)));
    int32_t st = km_init(graph_device(g), graph_n(g), 1, out);
    if (st) return st;
    SC_CUDA(cudaMemcpy((*out)->d_x, f, (size_t)graph_n(g) * 8, cudaMemcpyDeviceToDevice));
    return SC_OK;
}

int32_t sc_kmeans_set_flags(sc_kmeans *km, uint32_t flags) {
    SC_REQUIRE(km != nullptr, SC_E_INVALID, "null k-means context");
    SC_REQUIRE((flags & ~SC_KM_NO_COST_ASSERT) == 0, SC_E_INVALID, "unknown k-means flags 0x%x",
               flags);
    km->assert_cost = !(flags & SC_KM_NO_COST_ASSERT);
    return SC_OK;
}

void sc_kmeans_destroy(sc_kmeans *km) {
    if (!km) return;
    cudaSetDevice(km->device);
    if (km->stream) cudaStreamSynchronize(km->stream);
    void *ptrs[] = {km->d_x, km->d_best, km->d_lab[0], km->d_lab[1], km->d_keys, km->d_keys_alt,
                    km->d_vals, km->d_vals_alt, km->d_cub, km->d_chosen, km->d_u,
                    km->d_start, km->d_degen, km->d_cen, km->d_scen, km->d_sidx, km->d_cmax,
                    km->d_cnt, km->d_seg, km->d_part,
                    km->d_cost, km->d_changed, km->d_active, km->d_empty, km->d_A, km->d_a64,
                    km->d_vmax, km->d_cstart, km->d_total, km->d_kpred, km->d_neg,
                    km->d_round_on, km->d_on, km->d_q0, km->d_q1, km->d_cofs, km->d_nchunks,
                    km->d_sq0, km->d_sq1, km->d_svmax, km->d_skp, km->d_idx, km->d_idx_alt,
                    km->d_kmap, km->d_sstart, km->d_sflag,
                    km->d_elist, km->d_mlist, km->d_pval, km->d_pidx,
                    km->d_segkpp};
    if (km->stream2) cudaStreamSynchronize(km->stream2);
    for (void *p : ptrs)
        if (p) cudaFreeAsync(p, km->stream);
    if (km->stream) {
        cudaStreamSynchronize(km->stream);
        cudaStreamDestroy(km->stream);
    }
    if (km->stream2) cudaStreamDestroy(km->stream2);
    if (km->ev_main) cudaEventDestroy(km->ev_main);
    if (km->ev_cost) cudaEventDestroy(km->ev_cost);
    if (km->h_block) pinned_give(km->h_block, km->h_block_bytes);
    fused_lloyd_free(km->fused);
    delete km;
}

int32_t sc_kmeans_pp(sc_kmeans *km, int32_t k, int32_t R, const int32_t *start_round,
                     const double *uniforms, int64_t *chosen, int32_t *degenerate_out) {
    SC_REQUIRE(km && start_round && chosen && degenerate_out, SC_E_INVALID, "null argument");
    SC_REQUIRE(k >= 1 && k <= km->n, SC_E_INVALID, "need 1 <= k <= n, got k=%d, n=%lld", k,
               (long long)km->n);
    SC_REQUIRE(R >= 1, SC_E_INVALID, "restarts must be >= 1");
    SC_REQUIRE(k == 1 || uniforms, SC_E_INVALID, "uniforms required for k > 1");
    for (int r = 0; r < R; ++r) {
        SC_REQUIRE(start_round[r] >= 1 && start_round[r] <= k, SC_E_INVALID,
                   "start_round[%d]=%d out of [1, k]", r, start_round[r]);
        for (int i = 0; i < start_round[r]; ++i)
            SC_REQUIRE(chosen[(int64_t)r * k + i] >= 0 && chosen[(int64_t)r * k + i] < km->n,
                       SC_E_RANGE, "chosen index out of range");
    }
    SC_CUDA(cudaSetDevice(km->device));
    int32_t st = ensure(km, R, k);
    if (st) return st;
    cudaStream_t s = km->stream;
    const int64_t n = km->n;
    SC_CUDA(cudaMemcpyAsync(km->d_chosen, chosen, (size_t)R * k * 8, cudaMemcpyHostToDevice, s));
    if (k > 1)
        SC_CUDA(cudaMemcpyAsync(km->d_u, uniforms, (size_t)R * (k - 1) * 8,
                                cudaMemcpyHostToDevice, s));
    SC_CUDA(cudaMemcpyAsync(km->d_start, start_round, (size_t)R * 4, cudaMemcpyHostToDevice, s));
    SC_CUDA(cudaMemsetAsync(km->d_degen, 0xff, (size_t)R * 4, s));
    int smin = k;
    std::vector<int32_t> on(R);
    for (int r = 0; r < R; ++r) {
        smin = std::min(smin, start_round[r]);
        on[r] = start_round[r] < k;
    }
    SC_CUDA(cudaMemcpyAsync(km->d_on, on.data(), (size_t)R * 4, cudaMemcpyHostToDevice, s));
    if (k > 1 && small_kmeans_eligible(km->l, k, n)) {
        // every round of every restart in one launch (one CTA per restart)
        if ((st = small_kpp(km->device, s, km->d_x, n, k, R, km->d_start, km->d_u, km->d_chosen,
                            km->d_degen)))
            return st;
        SC_CUDA(cudaMemcpyAsync(chosen, km->d_chosen, (size_t)R * k * 8, cudaMemcpyDeviceToHost, s));
        SC_CUDA(cudaMemcpyAsync(degenerate_out, km->d_degen, (size_t)R * 4, cudaMemcpyDeviceToHost, s));
        SC_CUDA(cudaStreamSynchronize(s));
        return SC_OK;
    }
    // segments r over the D^2 weights best[r * nb + (0..nb)] (zero past n; nb a whole
    // number of super-chunks, so supers never straddle restarts)
    const int64_t nb = kpp_stride(n);
    const int64_t cps = nb / kSeqChunk;
    std::vector<int64_t> segoff(R + 1), cofs(R + 1);
    for (int r = 0; r <= R; ++r) {
        segoff[r] = (int64_t)r * nb;
        cofs[r] = (int64_t)r * cps;
    }
    const int64_t nch = (int64_t)R * cps;
    SC_CUDA(cudaMemcpyAsync(km->d_segkpp, segoff.data(), (size_t)(R + 1) * 8, cudaMemcpyHostToDevice, s));
    SC_CUDA(cudaMemcpyAsync(km->d_cofs, cofs.data(), (size_t)(R + 1) * 8, cudaMemcpyHostToDevice, s));
    SC_CUDA(cudaMemcpyAsync(km->d_nchunks, &nch, 8, cudaMemcpyHostToDevice, s));
    SegView v;
    v.vals = km->d_best;
    v.seg_off = km->d_segkpp;
    v.cofs = km->d_cofs;
    v.S = R;
    v.on = km->d_round_on;
    v.on_div = 1;
    const SeqWork w = seq_work(km);
    const dim3 g2(grid_1d(km, n, 256) / std::max(1, std::min(R, 8)) + 1, R);
    const int gw = grid_1d(km, nch * 32, 256);
    const int gs = (R * 32 + 255) / 256;
    k_kpp_init<<<g2, 256, 0, s>>>(km->d_x, n, km->l, k, km->d_chosen, km->d_start, km->d_on,
                                  km->d_best, km->d_kpred, cps);
    SC_CUDA(cudaGetLastError());
    // no chunk map of this call yet (0x7f7f7f7f is no grid exponent and not kNoGrid)
    SC_CUDA(cudaMemsetAsync(km->d_kmap, 0x7f, (size_t)nch * 4, s));
    const bool fused1d = km->l == 1 && R <= kMaxKppR && getenv("SC_KPP_CLASSIC") == nullptr;
    // SC_KPP_STATS: count the chunk maps the fix-up pass had to rebuild (diagnostics)
    unsigned long long *d_stats = nullptr;
    if (getenv("SC_KPP_STATS")) {
        SC_CUDA(cudaMallocAsync((void **)&d_stats, 16, s));
        SC_CUDA(cudaMemsetAsync(d_stats, 0, 16, s));
    }
    const int gu = grid_1d(km, cps * R * 32, 256);
    // certified fast draw (k_kpp_fast): n up to 2^24 (beyond, the sequential sum's own rounding
    // bound n * 2^-53 approaches the weights' share of the total and certification fails)
    const bool fast = fused1d && n <= (int64_t(1) << 24) && getenv("SC_KPP_NOFAST") == nullptr;
    // (SC_KPP_EPS_SCALE widens the certification margin: tests force the mixed case where some
    // restarts of a round are certified and others take the exact pipeline)
    const char *eps_scale = getenv("SC_KPP_EPS_SCALE");
    const double fast_eps = std::min(0.25, (eps_scale ? atof(eps_scale) : 1.0) * 1.0625 *
                                               (double)(n + 128 + (cps + 255) / 256) *
                                               1.1102230246251565e-16);
    for (int i = smin; i < k; ++i) {
        k_kpp_round_on<<<(R + 127) / 128, 128, 0, s>>>(R, i, km->d_start, km->d_on,
                                                       km->d_round_on, km->d_neg);
        if (fused1d) {
            // one pass: weights, chunk summaries and (speculative) chunk maps; x read once
            k_kpp_update_map<<<gu, 256, 0, s>>>(km->d_x, n, k, i, km->d_chosen, km->d_start,
                                                km->d_on, km->d_round_on, km->d_best, w,
                                                km->d_kmap, cps, R, fast ? km->d_a64 : nullptr);
            if (fast)
                k_kpp_fast<<<R, 256, 0, s>>>(km->d_best, km->d_a64, n, nb, cps, k, i, km->d_u,
                                             km->d_chosen, km->d_on, km->d_round_on, km->d_degen,
                                             fast_eps, d_stats ? d_stats + 1 : nullptr);
            k_seq_predict<32><<<R, 32 * 32, 0, s>>>(v, w);
            k_seq_chunkmap_fix<<<grid_1d(km, nch, 256), 256, 0, s>>>(v, w, km->d_kmap,
                                                                    km->d_nchunks, d_stats);
            k_seq_superize<<<gw, 256, 0, s>>>(v, w, km->d_nchunks);
            k_seq_compose<<<(R + kComposeWarps - 1) / kComposeWarps, 32 * kComposeWarps,
                            kComposeSmem, s>>>(v, w, 2);
            k_kpp_search2<<<gs, 256, 0, s>>>(v, w, n, k, i, km->d_u, km->d_chosen, km->d_on,
                                             km->d_degen);
        } else {
            k_kpp_update_sum<<<gw, 256, 0, s>>>(km->d_x, n, km->l, k, i, km->d_chosen,
                                                km->d_start, km->d_on, km->d_round_on,
                                                km->d_best, w, cps, R);
            k_seq_predict<><<<R, 32 * kPredictWarps, 0, s>>>(v, w);
            k_seq_chunkmap<<<gw, 256, 0, s>>>(v, w, km->d_nchunks);
            k_seq_superize<<<gw, 256, 0, s>>>(v, w, km->d_nchunks);
            k_seq_compose<<<(R + kComposeWarps - 1) / kComposeWarps, 32 * kComposeWarps,
                            kComposeSmem, s>>>(v, w, 1);
            k_kpp_search<<<gs, 256, 0, s>>>(v, w, n, k, i, km->d_u, km->d_chosen, km->d_on,
                                             km->d_degen);
        }
    }
    SC_CUDA(cudaGetLastError());
    SC_CUDA(cudaMemcpyAsync(chosen, km->d_chosen, (size_t)R * k * 8, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaMemcpyAsync(degenerate_out, km->d_degen, (size_t)R * 4, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaStreamSynchronize(s));
    if (d_stats) {
        unsigned long long hh[2] = {0, 0};
        cudaMemcpy(hh, d_stats, 16, cudaMemcpyDeviceToHost);
        cudaFree(d_stats);
        const unsigned long long h = hh[0];
        fprintf(stderr, "[kpp] rounds %d..%d, R=%d, chunks %lld: chunk maps rebuilt %llu (%.2f per round per restart); "
                "draws certified by the fast path %llu\n",
                smin, k - 1, R, (long long)cps, h, (double)h / std::max(1, k - smin) / R, hh[1]);
    }
    return SC_OK;
}

int32_t sc_kmeans_lloyd(sc_kmeans *km, int32_t k, int32_t R, const int64_t *chosen,
                        int32_t max_iters, double tol, int64_t *labels_out, double *costs_out,
                        int32_t *iters_out, int32_t *best_restart_out, double *ms_out) {
    SC_REQUIRE(km && chosen && labels_out, SC_E_INVALID, "null argument");
    SC_REQUIRE(k >= 1 && k <= km->n, SC_E_INVALID, "need 1 <= k <= n, got k=%d", k);
    SC_REQUIRE(R >= 1, SC_E_INVALID, "restarts must be >= 1, got %d", R);
    SC_REQUIRE(max_iters >= 1, SC_E_INVALID, "max_iters must be >= 1");
    SC_REQUIRE((int64_t)R * k < ((int64_t)1 << 30), SC_E_INVALID, "restarts * k too large");
    for (int64_t i = 0; i < (int64_t)R * k; ++i)
        SC_REQUIRE(chosen[i] >= 0 && chosen[i] < km->n, SC_E_RANGE, "chosen index out of range");
    SC_CUDA(cudaSetDevice(km->device));
    int32_t st = ensure(km, R, k);
    if (st) return st;
    auto t0 = std::chrono::steady_clock::now();
    cudaStream_t s = km->stream;
    const int64_t n = km->n;
    const int l = km->l;
    const int64_t nbuf = (n * l + kEinsumBuf - 1) / kEinsumBuf;
    const int rk = R * k;
    SC_CUDA(cudaMemcpyAsync(km->d_chosen, chosen, (size_t)rk * 8, cudaMemcpyHostToDevice, s));
    if (small_kmeans_eligible(l, k, n)) {
        st = small_lloyd(s, km->d_x, n, k, R, km->d_chosen, max_iters, tol, km->assert_cost,
                         km->d_lab[0], km->d_cost, km->d_active, km->d_empty, labels_out,
                         costs_out, iters_out, best_restart_out);
        if (ms_out)
            *ms_out = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                          .count();
        return st;
    }
    if (fused_lloyd_eligible(l, k, R, n)) {
        // every iteration of every restart in one persistent kernel (sc_kmeans_fused.cu);
        // 1 = not applicable (points of both signs): the general path below
        st = fused_lloyd(&km->fused, km->device, km->sm_count, s, km->d_x, n, k, R, km->d_chosen,
                         max_iters, tol, km->assert_cost, labels_out, costs_out, iters_out,
                         best_restart_out);
        if (st != 1) {
            if (ms_out)
                *ms_out = std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now() - t0).count();
            return st;
        }
        st = SC_OK;
    }
    k_gather_centers<<<(rk * l + 255) / 256, 256, 0, s>>>(km->d_x, km->d_chosen, rk, l, km->d_cen);
    // labels start at zero (kmeans.py:195)
    SC_CUDA(cudaMemsetAsync(km->d_lab[0], 0, (size_t)R * n * 4, s));
    std::vector<int32_t> active(R, 1), changed(R), iters(R, 0), final_buf(R, 0);
    std::vector<double> prev(R, INFINITY), cost(R, INFINITY);
    int cur = 0;  // d_lab[cur] = labels of the previous iteration
    int end_bit = 1;
    while ((1ll << end_bit) < (long long)rk) ++end_bit;
    const size_t smem_assign = (size_t)k * (8 * l + 4);
    SC_REQUIRE(smem_assign <= 200 * 1024, SC_E_INVALID, "k=%d too large for the assign kernel", k);
    if (smem_assign > 48 * 1024) {
        SC_CUDA(cudaFuncSetAttribute(k_assign, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_assign));
        SC_CUDA(cudaFuncSetAttribute(k_assign1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_assign));
    }
    const char *cst = getenv("SC_CS_TILE");  // counting-sort tile (A/B: 4096, 8192, 16384)
    const int cs_tile = cst ? atoi(cst) : kCsTile;
    const char *smk = getenv("SC_KMEANS_SORTED_MIN_K");
    const int sorted_min_k = smk ? atoi(smk) : kSortedMinK;
    const bool sorted_assign = l == 1 && k >= sorted_min_k && k <= kSortedMaxK &&
                               getenv("SC_KMEANS_BRUTE_ASSIGN") == nullptr;
    const size_t smem_sorted = (size_t)k * 16;
    size_t smem_sort = 12;
    while (smem_sort < (size_t)k * 12) smem_sort <<= 1;  // next power of two of k, x 12 B
    if (sorted_assign && smem_sorted > 48 * 1024)
        SC_CUDA(cudaFuncSetAttribute(k_assign_sorted, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_sorted));
    if (sorted_assign)  // (plus 256 B of static shared memory)
        SC_CUDA(cudaFuncSetAttribute(k_sort_centers, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_sort));
    if (k > 48 * 1024)
        SC_CUDA(cudaFuncSetAttribute(k_repair, cudaFuncAttributeMaxDynamicSharedMemorySize, k));
    const dim3 ga(grid_1d(km, n, 256) / std::max(1, std::min(R, 8)) + 1, R);
    const dim3 gc((unsigned)((nbuf + kCostWarps - 1) / kCostWarps), R);
    SegView vm;
    vm.vals = km->d_vals_alt;
    vm.seg_off = km->d_seg;
    vm.cofs = km->d_cofs;
    vm.S = rk;
    vm.on = nullptr;  // segments are built for active restarts only
    vm.on_div = 1;
    const SeqWork wm = seq_work(km);
    const bool prof = getenv("SC_KMEANS_PROFILE") != nullptr;
    cudaEvent_t pe[5];
    double pacc[4] = {0, 0, 0, 0};
    if (prof)
        for (auto &ev : pe) cudaEventCreate(&ev);
    // Iteration it: "main" (assign, repair, sort, ordered sums, means) on stream s, then the
    // einsum cost on stream s2.  While the host waits for cost(it) to decide which restarts
    // stop, main(it+1) already runs speculatively for every restart still active at it (a
    // restart that stops at it simply ignores its iteration it+1), so the cost chain and
    // the host round trip overlap the next iteration.  Double-buffered per parity of it:
    // centers (assign reads cen[it&1], means write cen[(it+1)&1]), active flags, changed
    // counts, host result slots.
    cudaStream_t s2 = km->stream2;
    auto cen_buf = [&](int i) { return km->d_cen + (size_t)(i & 1) * rk * l; };
    auto act_buf = [&](int i) { return km->d_active + (i & 1) * R; };
    auto chg_buf = [&](int i) { return km->d_changed + (i & 1) * R; };
    const bool tl = getenv("SC_KMEANS_TIMELINE") != nullptr;
    std::vector<cudaEvent_t> tl_ev;
    std::vector<double> tl_host;
    cudaEvent_t tl0 = nullptr;
    auto host_ms = [&]() {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
            .count();
    };
    auto tl_mark = [&](cudaStream_t st_) {
        if (!tl) return;
        cudaEvent_t e_;
        cudaEventCreate(&e_);
        cudaEventRecord(e_, st_);
        tl_ev.push_back(e_);
        tl_host.push_back(host_ms());
    };
    if (tl) {
        cudaEventCreate(&tl0);
        cudaEventRecord(tl0, s);
    }
    auto launch_main = [&](int it, const std::vector<int32_t> &actv, int cur_lab) -> int32_t {
        tl_mark(s);
        // pinned staging (a pageable copy would make the host wait for the stream)
        int32_t *hflags = km->h_act + (size_t)(it & 1) * 2 * R, *hlist = hflags + R;
        int nact = 0;
        for (int r = 0; r < R; ++r) {
            hflags[r] = actv[r];
            if (actv[r]) hlist[nact++] = r;
        }
        const int nxt = cur_lab ^ 1;
        const int nseg = nact * k;
        int end_bit = 1;
        while ((1ll << end_bit) < (long long)nseg) ++end_bit;
        int32_t *d_act = act_buf(it), *d_chg = chg_buf(it);
        double *cen_in = cen_buf(it), *cen_out = cen_buf(it + 1);
        SC_CUDA(cudaMemcpyAsync(d_act, hflags, (size_t)R * 4, cudaMemcpyHostToDevice, s));
        SC_CUDA(cudaMemcpyAsync(km->d_empty, hlist, (size_t)nact * 4, cudaMemcpyHostToDevice, s));
        SC_CUDA(cudaMemsetAsync(km->d_cnt, 0, (size_t)rk * 4, s));
        SC_CUDA(cudaMemsetAsync(d_chg, 0, (size_t)R * 4, s));
        if (prof) cudaEventRecord(pe[0], s);
        if (sorted_assign) {
            k_sort_centers<<<R, 1024, smem_sort, s>>>(k, cen_in, d_act, km->d_scen, km->d_sidx,
                                                      km->d_cmax);
            k_assign_sorted<<<ga, 256, smem_sorted, s>>>(km->d_x, n, k, km->d_scen, km->d_sidx,
                                                         km->d_cmax, d_act, km->d_lab[cur_lab],
                                                         km->d_lab[nxt], km->d_cnt, d_chg);
        } else if (l == 1) {
            k_assign1<<<ga, 256, smem_assign, s>>>(km->d_x, n, k, cen_in, d_act, km->d_lab[cur_lab],
                                                    km->d_lab[nxt], km->d_cnt, d_chg);
        } else {
            k_assign<<<ga, 256, smem_assign, s>>>(km->d_x, n, l, k, cen_in, d_act,
                                                   km->d_lab[cur_lab], km->d_lab[nxt], km->d_cnt,
                                                   d_chg);
        }
        if (n >= kCoopRepairMinN && k <= kRepairMaxK && getenv("SC_KMEANS_CTA_REPAIR") == nullptr) {
            const double *a_x = km->d_x, *a_cen = cen_in;
            const int32_t *a_act = d_act, *a_prev = km->d_lab[cur_lab];
            int32_t *a_lab = km->d_lab[nxt], *a_cnt = km->d_cnt, *a_ch = d_chg;
            double *a_own = km->d_best, *a_pv = km->d_pval;
            int32_t *a_el = km->d_elist, *a_ml = km->d_mlist;
            int64_t *a_pi = km->d_pidx;
            int64_t a_n = n;
            int a_l = l, a_k = k, a_R = R;
            void *args[] = {&a_x, &a_n, &a_l, &a_k, &a_cen, &a_act, &a_prev, &a_lab, &a_cnt,
                            &a_ch, &a_own, &a_el, &a_ml, &a_pv, &a_pi, &a_R};
            SC_CUDA(cudaLaunchCooperativeKernel((const void *)k_repair_coop, km->coop_grid,
                                                kRepairTPB, args, (size_t)k * 4, s));
        } else {
            k_repair<<<R, 1024, (size_t)k, s>>>(km->d_x, n, l, k, cen_in, d_act,
                                                  km->d_lab[cur_lab], km->d_lab[nxt], km->d_cnt,
                                                  d_chg, km->d_best);
        }
        // np.add.at order: stable radix sort of the active restarts' points on
        // (slot, label) keeps point-index order inside every cluster; then exact ordered sums
        if (prof) cudaEventRecord(pe[1], s);
        const int64_t m = (int64_t)nact * n;
        size_t tb = km->cub_bytes;
        if (l == 1 && nseg <= kCsMaxKeys && getenv("SC_KMEANS_RADIX_SORT") == nullptr) {
            // tile of the counting sort: larger tiles shrink the (key, tile) count matrix and its
            // scan (nseg x m / tile ints), at ~4 elements per key per 4096-tile at k = 100
            const int tile = cs_tile;
            const int ntiles = (int)((m + tile - 1) / tile);
            int32_t *bh = km->d_keys, *boff = km->d_keys_alt;  // nseg * ntiles <= m ints each
            auto hist = [&](auto tl) {
                constexpr int TL = decltype(tl)::value;
                k_cs_hist<TL><<<ntiles, 32 * kCsWarps, (size_t)nseg * 4, s>>>(
                    m, n, k, km->d_lab[nxt], km->d_empty, nseg, ntiles, bh);
            };
            auto scatter = [&](auto tl) {
                constexpr int TL = decltype(tl)::value;
                k_cs_scatter<TL><<<ntiles, 32 * kCsWarps, (size_t)nseg * kCsWarps * 4, s>>>(
                    m, n, k, km->d_lab[nxt], km->d_empty, nseg, ntiles, boff, km->d_x,
                    km->d_vals_alt);
            };
            if (tile == 16384) hist(std::integral_constant<int, 16384>{});
            else if (tile == 8192) hist(std::integral_constant<int, 8192>{});
            else hist(std::integral_constant<int, 4096>{});
            size_t sb = km->cub_bytes;
            SC_CUDA(cub::DeviceScan::ExclusiveSum(km->d_cub, sb, bh, boff, (int64_t)nseg * ntiles,
                                                  s));
            if (tile == 16384) scatter(std::integral_constant<int, 16384>{});
            else if (tile == 8192) scatter(std::integral_constant<int, 8192>{});
            else scatter(std::integral_constant<int, 4096>{});
        } else if (l == 1) {
            k_make_keys<<<grid_1d(km, m, 256), 256, 0, s>>>(n, k, km->d_lab[nxt], km->d_empty,
                                                             nact, km->d_keys, km->d_vals, km->d_x);
            SC_CUDA(cub::DeviceRadixSort::SortPairs(km->d_cub, tb, km->d_keys, km->d_keys_alt,
                                                    km->d_vals, km->d_vals_alt, m, 0, end_bit, s));
        } else {
            k_make_keys_idx<<<grid_1d(km, m, 256), 256, 0, s>>>(n, k, km->d_lab[nxt], km->d_empty,
                                                                 nact, km->d_keys, km->d_idx);
            SC_CUDA(cub::DeviceRadixSort::SortPairs(km->d_cub, tb, km->d_keys, km->d_keys_alt,
                                                    km->d_idx, km->d_idx_alt, m, 0, end_bit, s));
        }
        k_seg_layout<<<1, 1024, 0, s>>>(nseg, k, km->d_cnt, km->d_empty, km->d_seg, km->d_cofs,
                                        km->d_nchunks);
        if (prof) cudaEventRecord(pe[2], s);
        vm.S = nseg;
        const int gwm = grid_1d(km, (m / kSeqChunk + nseg) * 32, 256);
        for (int q = 0; q < l; ++q) {  // np.add.at over each coordinate column
            if (l > 1)
                k_gather_coord<<<grid_1d(km, m, 256), 256, 0, s>>>(km->d_x, km->d_idx_alt, m, l, q,
                                                                    km->d_vals_alt);
            SC_CUDA(cudaMemsetAsync(km->d_neg, 0, (size_t)nseg * 4, s));
            k_seq_summarize<<<gwm, 256, 0, s>>>(vm, wm, km->d_nchunks);
            k_seq_flip<<<gwm, 256, 0, s>>>(vm, wm, km->d_nchunks);
            k_seq_predict<><<<nseg, 32 * kPredictWarps, 0, s>>>(vm, wm);
            k_seq_chunkmap<<<gwm, 256, 0, s>>>(vm, wm, km->d_nchunks);
            k_seq_superize<<<gwm, 256, 0, s>>>(vm, wm, km->d_nchunks);
            k_seq_compose<<<(nseg + kComposeWarps - 1) / kComposeWarps, 32 * kComposeWarps,
                            kComposeSmem, s>>>(vm, wm, 0);
            k_seg_means<<<(nseg + 127) / 128, 128, 0, s>>>(nseg, k, l, q, km->d_seg, km->d_total,
                                                           km->d_empty, cen_out);
        }
        if (prof) cudaEventRecord(pe[3], s);
        tl_mark(s);
        SC_CUDA(cudaGetLastError());
        return SC_OK;
    };
    // cost of iteration it (labels d_lab[lab_buf], centers cen[(it+1)&1]) on s2 after main(it)
    auto launch_cost = [&](int it, int lab_buf) -> int32_t {
        SC_CUDA(cudaEventRecord(km->ev_main, s));
        SC_CUDA(cudaStreamWaitEvent(s2, km->ev_main, 0));
        k_cost_buf<<<gc, 32 * kCostWarps, 0, s2>>>(km->d_x, n, l, k, km->d_lab[lab_buf],
                                                    cen_buf(it + 1), act_buf(it), nbuf, km->d_part);
        k_cost_combine<<<R, 256, 0, s2>>>(nbuf, km->d_part, act_buf(it), km->d_cost);
        SC_CUDA(cudaGetLastError());
        if (prof) cudaEventRecord(pe[4], s2);
        SC_CUDA(cudaMemcpyAsync(km->h_cost + (it & 1) * R, km->d_cost, (size_t)R * 8,
                                cudaMemcpyDeviceToHost, s2));
        SC_CUDA(cudaMemcpyAsync(km->h_changed + (it & 1) * R, chg_buf(it), (size_t)R * 4,
                                cudaMemcpyDeviceToHost, s2));
        SC_CUDA(cudaEventRecord(km->ev_cost, s2));
        tl_mark(s2);
        return SC_OK;
    };
    const bool speculate = getenv("SC_KMEANS_NO_SPECULATION") == nullptr;
    const bool trace = getenv("SC_KMEANS_TRACE") != nullptr;
    double wait_ms = 0.0;
    if ((st = launch_main(0, active, cur))) return st;
    for (int it = 0; it < max_iters; ++it) {
        const int nxt = cur ^ 1;
        if ((st = launch_cost(it, nxt))) return st;
        const bool spec = speculate && it + 1 < max_iters;
        if (spec && (st = launch_main(it + 1, active, nxt))) return st;
        auto w0 = std::chrono::steady_clock::now();
        SC_CUDA(cudaEventSynchronize(km->ev_cost));
        wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
        if (prof)
            for (int q = 0; q < 4; ++q) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, pe[q], pe[q + 1]);
                pacc[q] += ms;
            }
        const double *hc = km->h_cost + (it & 1) * R;
        const int32_t *hch = km->h_changed + (it & 1) * R;
        int nact = 0;
        for (int r = 0; r < R; ++r) {
            if (!active[r]) continue;
            // kmeans.py:202-210, in the same double arithmetic
            const bool fin = std::isfinite(prev[r]);
            const bool unchanged = hch[r] == 0 && fin;
            const double c = hc[r];
            // kmeans.py:206: assert cost <= prev_cost * (1 + 1e-12) + 1e-12
            if (km->assert_cost && !(c <= prev[r] * (1.0 + 1e-12) + 1e-12)) {
                cudaStreamSynchronize(s);
                return fail(SC_E_INTERNAL, "k-means cost increased (restart %d, iteration %d: "
                            "%.17g > %.17g)", r, iters[r], c, prev[r]);
            }
            const bool small_gain = fin && (prev[r] - c <= tol * std::max(prev[r], 1e-300));
            if (r == 0 && trace)
                fprintf(stderr, "exact  r0 it %d cost %.17g changed %d\n", iters[r], c, hch[r]);
            prev[r] = c;
            iters[r] += 1;
            final_buf[r] = nxt;
            if (unchanged || small_gain) active[r] = 0;
            nact += active[r];
        }
        cur = nxt;
        if (!nact) break;
        if (!speculate && it + 1 < max_iters && (st = launch_main(it + 1, active, cur))) return st;
    }
    if (prof) fprintf(stderr, "[sc_kmeans_lloyd] host waited %.3f ms for the iteration results\n", wait_ms);
    if (tl) {
        cudaDeviceSynchronize();
        // records come in the order main-start, main-end, cost-end per launch; print device
        // time (ms since the first record) and the host time each was enqueued
        for (size_t q = 0; q < tl_ev.size() && q < 60; ++q) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, tl0, tl_ev[q]);
            fprintf(stderr, "[timeline] %2zu dev %8.3f ms  host-enqueue %8.3f ms\n", q, ms,
                    tl_host[q]);
        }
        for (auto e_ : tl_ev) cudaEventDestroy(e_);
        cudaEventDestroy(tl0);
    }
    SC_CUDA(cudaStreamSynchronize(s));  // a speculative iteration may still be running
    if (prof) {
        fprintf(stderr, "[sc_kmeans_lloyd] assign+repair %.3f ms, sort %.3f ms, ordered sums %.3f ms, cost %.3f ms\n",
                pacc[0], pacc[1], pacc[2], pacc[3]);
        for (auto &ev : pe) cudaEventDestroy(ev);
    }
    int best = -1;
    double best_cost = INFINITY;
    for (int r = 0; r < R; ++r)
        if (prev[r] < best_cost) {
            best_cost = prev[r];
            best = r;
        }
    SC_REQUIRE(best >= 0, SC_E_INTERNAL, "no restart produced a finite cost");
    std::vector<int32_t> lab32((size_t)n);
    SC_CUDA(cudaMemcpyAsync(lab32.data(), km->d_lab[final_buf[best]] + (size_t)best * n,
                            (size_t)n * 4, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaStreamSynchronize(s));
    sc::widen_labels(lab32.data(), labels_out, n);
    if (costs_out)
        for (int r = 0; r < R; ++r) costs_out[r] = prev[r];
    if (iters_out)
        for (int r = 0; r < R; ++r) iters_out[r] = iters[r];
    if (best_restart_out) *best_restart_out = best;
    if (ms_out)
        *ms_out = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                      .count();
    return SC_OK;
}

}  // extern "C"

namespace sc {
// ---------------------------------------------------------------------------------------
// Fast 1-D Lloyd on sorted values (BASELINE north star, step 3: "CUB radix sort, prefix sums
// and a Lloyd split on the sorted values").  In one dimension every cluster is an interval
// of the sorted points, so an iteration is k binary searches for the boundaries plus prefix-
// sum lookups for the means and the cost: O(k log n) instead of O(n).  One CTA runs all the
// iterations of one restart.  Seeding (k-means++), the argmin tie rule, the empty-cluster
// repair (the far end of an interval) and the stop rules follow the reference; the sums come
// from prefix sums instead of np.add.at / einsum, so this mode is not bit-exact: labels can
// differ from the replica only where a distance or a stopping decision sits within rounding.
constexpr int kFastMaxK = 2048;

__device__ __forceinline__ bool upper_wins(double x, double cl, int il, double cu, int iu) {
    const double dl = d2ref(x, cl), du = d2ref(x, cu);
    return du < dl || (du == dl && iu < il);
}

__global__ void __launch_bounds__(256) k_lloyd_sorted(
    const double *__restrict__ xs, const int32_t *__restrict__ ix, const double *__restrict__ P,
    const double *__restrict__ Q, int64_t n, int k, const double *__restrict__ cen0,
    int max_iters, double tol, int64_t *__restrict__ out_lo, int64_t *__restrict__ out_hi,
    double *__restrict__ out_cost, int32_t *__restrict__ out_iters, int trace) {
    extern __shared__ unsigned char fs_raw[];
    const int r = blockIdx.x;
    int Pk = 1;
    while (Pk < k) Pk <<= 1;
    double *cv = reinterpret_cast<double *>(fs_raw);  // centers by id
    double *sv = cv + k;                              // sorted center values (Pk)
    int32_t *si = reinterpret_cast<int32_t *>(sv + Pk);  // their ids (Pk)
    int64_t *lo = reinterpret_cast<int64_t *>(si + Pk + (Pk & 1));
    int64_t *hi = lo + k, *plo = hi + k, *phi = plo + k;
    __shared__ double red[8];
    __shared__ int flag;
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        cv[i] = cen0[(int64_t)r * k + i];
        plo[i] = -1;
        phi[i] = -1;
    }
    double prev_cost = INFINITY;
    int it = 0;
    for (; it < max_iters; ++it) {
        __syncthreads();
        // (a) centers sorted by (value, id)
        for (int i = threadIdx.x; i < Pk; i += blockDim.x) {
            sv[i] = i < k ? cv[i] : INFINITY;
            si[i] = i < k ? i : INT32_MAX;
        }
        __syncthreads();
        for (int size = 2; size <= Pk; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int i = threadIdx.x; i < Pk; i += blockDim.x) {
                    const int j = i ^ stride;
                    if (j > i) {
                        const bool up = (i & size) == 0;
                        const bool gt = sv[i] > sv[j] || (sv[i] == sv[j] && si[i] > si[j]);
                        if (gt == up) {
                            const double tv = sv[i];
                            sv[i] = sv[j];
                            sv[j] = tv;
                            const int32_t ti = si[i];
                            si[i] = si[j];
                            si[j] = ti;
                        }
                    }
                }
                __syncthreads();
            }
        // (b) intervals: the first of equal-valued centers (lowest id) owns their points;
        // between consecutive distinct centers the boundary is the first point the upper one
        // wins (argmin, ties to the lower id)
        for (int j = threadIdx.x; j < k; j += blockDim.x) {
            lo[si[j]] = 0;
            hi[si[j]] = 0;
        }
        __syncthreads();
        for (int j = threadIdx.x; j < k; j += blockDim.x) {
            if (j > 0 && sv[j] == sv[j - 1]) continue;  // duplicate value: empty
            // previous distinct owner
            int jp = j - 1;
            while (jp > 0 && sv[jp] == sv[jp - 1]) --jp;
            int jn = j + 1;
            while (jn < k && sv[jn] == sv[j]) ++jn;
            int64_t a = 0, b = n;
            if (j > 0) {  // first point that j wins against its lower neighbour
                int64_t l0 = 0, h0 = n;
                while (l0 < h0) {
                    const int64_t m = (l0 + h0) >> 1;
                    if (upper_wins(xs[m], sv[jp], si[jp], sv[j], si[j])) h0 = m;
                    else l0 = m + 1;
                }
                a = l0;
            }
            if (jn < k) {  // first point the next distinct center wins against j
                int64_t l0 = 0, h0 = n;
                while (l0 < h0) {
                    const int64_t m = (l0 + h0) >> 1;
                    if (upper_wins(xs[m], sv[j], si[j], sv[jn], si[jn])) h0 = m;
                    else l0 = m + 1;
                }
                b = l0;
            }
            lo[si[j]] = a;
            hi[si[j]] = b < a ? a : b;
        }
        __syncthreads();
        // (c) empty clusters in increasing id take the far end of the interval with the
        // largest own distance (first point index on ties); a moved point keeps distance 0
        if (threadIdx.x == 0) {
            for (int e = 0; e < k; ++e) {
                if (hi[e] > lo[e]) continue;
                double bv = -1.0;
                int32_t bidx = INT32_MAX;
                int bj = -1;
                int64_t bp = -1;
                for (int j = 0; j < k; ++j) {
                    if (hi[j] - lo[j] < 2) continue;  // singletons (incl. moved points): 0
                    const int64_t cand[2] = {lo[j], hi[j] - 1};
                    for (int q = 0; q < 2; ++q) {
                        const double d = d2ref(xs[cand[q]], cv[j]);
                        const int32_t id = ix[cand[q]];
                        if (d > bv || (d == bv && id < bidx)) {
                            bv = d;
                            bidx = id;
                            bj = j;
                            bp = cand[q];
                        }
                    }
                }
                if (bj < 0) break;  // nothing left to move
                if (bp == lo[bj]) ++lo[bj];
                else --hi[bj];
                lo[e] = bp;
                hi[e] = bp + 1;
            }
        }
        __syncthreads();
        // (d) means, cost and change
        double cst = 0.0;
        int ch = 0;
        const double x0 = xs[n / 2];  // P, Q hold prefix sums of x - x0 and (x - x0)^2
        for (int j = threadIdx.x; j < k; j += blockDim.x) {
            const int64_t a = lo[j], b = hi[j];
            const double cnt = (double)(b - a);
            const double S = P[b] - P[a], S2 = Q[b] - Q[a];
            const double m = cnt > 0 ? S / cnt : 0.0;  // centred mean
            const double mu = cnt > 0 ? x0 + m : 0.0;
            cst += fmax(0.0, S2 - 2.0 * m * S + cnt * m * m);
            ch |= (a != plo[j]) || (b != phi[j]);
            plo[j] = a;
            phi[j] = b;
            cv[j] = mu;
        }
        for (int o = 16; o; o >>= 1) {
            cst += __shfl_xor_sync(0xffffffffu, cst, o);
            ch |= __shfl_xor_sync(0xffffffffu, ch, o);
        }
        if (threadIdx.x == 0) flag = 0;
        __syncthreads();
        if ((threadIdx.x & 31) == 0) {
            red[threadIdx.x >> 5] = cst;
            if (ch) atomicOr(&flag, 1);
        }
        __syncthreads();
        double cost = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) cost += red[w];
        const bool fin = isfinite(prev_cost);
        const bool unchanged = fin && flag == 0;
        if (trace && r == 0 && threadIdx.x == 0)
            printf("sorted r0 it %d cost %.17g changed %d\n", it, cost, flag);
        const bool small_gain = fin && (prev_cost - cost <= tol * fmax(prev_cost, 1e-300));
        prev_cost = cost;
        if (unchanged || small_gain) {
            ++it;
            break;
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        out_lo[(int64_t)r * k + j] = plo[j];
        out_hi[(int64_t)r * k + j] = phi[j];
    }
    if (threadIdx.x == 0) {
        out_cost[r] = prev_cost;
        out_iters[r] = it;
    }
}

__global__ void k_sorted_labels(const int32_t *__restrict__ ix, const int64_t *__restrict__ lo,
                                const int64_t *__restrict__ hi, int k,
                                int32_t *__restrict__ lab) {
    const int j = blockIdx.x;
    if (j >= k) return;
    for (int64_t p = lo[j] + threadIdx.x; p < hi[j]; p += blockDim.x) lab[ix[p]] = j;
}

__global__ void k_iota(int32_t *__restrict__ a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (int32_t)i;
}

// y = x - x0 and y^2 (x0 = the median sorted value, read on the device): prefix sums of
// centred values keep the cost Q - 2 mu S + n mu^2 from cancelling away (embeddings are
// typically a narrow band far from zero, e.g. f ~ 0.4999 +- 1e-6 at config 2)
__global__ void k_center_square(const double *__restrict__ xs, int64_t n, double *__restrict__ y,
                                double *__restrict__ y2) {
    const double x0 = xs[n / 2];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = xs[i] - x0;
        y[i] = v;
        y2[i] = v * v;
    }
}
}  // namespace sc

extern "C" int32_t sc_kmeans_lloyd_sorted(sc_kmeans *km, int32_t k, int32_t R,
                                          const int64_t *chosen, int32_t max_iters, double tol,
                                          int64_t *labels_out, double *costs_out,
                                          int32_t *iters_out, int32_t *best_restart_out) {
    using namespace sc;
    SC_REQUIRE(km && chosen && labels_out, SC_E_INVALID, "null argument");
    SC_REQUIRE(km->l == 1, SC_E_INVALID, "the sorted Lloyd handles 1-D points only");
    SC_REQUIRE(k >= 1 && k <= km->n && k <= kFastMaxK, SC_E_INVALID,
               "need 1 <= k <= min(n, %d), got k=%d", kFastMaxK, k);
    SC_REQUIRE(R >= 1 && max_iters >= 1, SC_E_INVALID, "bad restarts / max_iters");
    for (int64_t i = 0; i < (int64_t)R * k; ++i)
        SC_REQUIRE(chosen[i] >= 0 && chosen[i] < km->n, SC_E_RANGE, "chosen index out of range");
    SC_CUDA(cudaSetDevice(km->device));
    int32_t st = ensure(km, R, k);
    if (st) return st;
    cudaStream_t s = km->stream;
    const int64_t n = km->n;
    // sorted points, their indices and prefix sums (kept in the Lloyd workspaces)
    double *fb = nullptr;  // sorted x, P, Q, squares
    void *tmp = nullptr;
    size_t tb = 0, sb = 0;
    SC_CUDA(cudaMallocAsync((void **)&fb, (size_t)(4 * n + 2) * 8, s));
    double *ys = nullptr;  // centred sorted values
    SC_CUDA(cudaMallocAsync((void **)&ys, (size_t)n * 8, s));
    double *xs = fb, *P = fb + n, *Q = P + n + 1, *sq = Q + n + 1;
    int32_t *ixs = km->d_keys_alt, *iota = km->d_keys;
    k_iota<<<grid_1d(km, n, 256), 256, 0, s>>>(iota, n);
    SC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, km->d_x, xs, iota, ixs, n, 0, 64, s));
    SC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, sb, xs, P + 1, n, s));
    SC_CUDA(cudaMallocAsync(&tmp, std::max(tb, sb) + 16, s));
    SC_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, km->d_x, xs, iota, ixs, n, 0, 64, s));
    SC_CUDA(cudaMemsetAsync(P, 0, 8, s));
    SC_CUDA(cudaMemsetAsync(Q, 0, 8, s));
    k_center_square<<<grid_1d(km, n, 256), 256, 0, s>>>(xs, n, ys, sq);
    SC_CUDA(cub::DeviceScan::InclusiveSum(tmp, sb, ys, P + 1, n, s));
    SC_CUDA(cub::DeviceScan::InclusiveSum(tmp, sb, sq, Q + 1, n, s));
    const int rk = R * k;
    SC_CUDA(cudaMemcpyAsync(km->d_chosen, chosen, (size_t)rk * 8, cudaMemcpyHostToDevice, s));
    k_gather_centers<<<(rk + 255) / 256, 256, 0, s>>>(km->d_x, km->d_chosen, rk, 1, km->d_cen);
    int Pk = 1;
    while (Pk < k) Pk <<= 1;
    const size_t smem = (size_t)k * 8 + (size_t)Pk * 12 + 8 + (size_t)k * 32;
    SC_CUDA(cudaFuncSetAttribute(k_lloyd_sorted, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    int64_t *dlo = nullptr, *dhi = nullptr;
    int64_t *buf = nullptr;
    SC_CUDA(cudaMallocAsync((void **)&buf, (size_t)rk * 16, s));
    dlo = buf;
    dhi = buf + rk;
    k_lloyd_sorted<<<R, 256, smem, s>>>(xs, ixs, P, Q, n, k, km->d_cen, max_iters, tol, dlo, dhi,
                                        km->d_cost, km->d_changed,
                                        getenv("SC_KMEANS_TRACE") != nullptr);
    std::vector<double> cost((size_t)R);
    std::vector<int32_t> iters((size_t)R);
    SC_CUDA(cudaMemcpyAsync(cost.data(), km->d_cost, (size_t)R * 8, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaMemcpyAsync(iters.data(), km->d_changed, (size_t)R * 4, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaStreamSynchronize(s));
    int best = -1;
    double bc = INFINITY;
    for (int r = 0; r < R; ++r)
        if (cost[(size_t)r] < bc) {
            bc = cost[(size_t)r];
            best = r;
        }
    if (best < 0) {
        cudaFreeAsync(buf, s);
        cudaFreeAsync(fb, s);
        cudaFreeAsync(tmp, s);
        cudaFreeAsync(ys, s);
        return fail(SC_E_INTERNAL, "no restart produced a finite cost");
    }
    k_sorted_labels<<<k, 256, 0, s>>>(ixs, dlo + (int64_t)best * k, dhi + (int64_t)best * k, k,
                                      km->d_lab[1]);
    std::vector<int32_t> lab32((size_t)n);
    SC_CUDA(cudaMemcpyAsync(lab32.data(), km->d_lab[1], (size_t)n * 4, cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(buf, s);
    cudaFreeAsync(fb, s);
    cudaFreeAsync(tmp, s);
    cudaFreeAsync(ys, s);
    SC_CUDA(cudaStreamSynchronize(s));
    sc::widen_labels(lab32.data(), labels_out, n);
    if (costs_out)
        for (int r = 0; r < R; ++r) costs_out[r] = cost[(size_t)r];
    if (iters_out)
        for (int r = 0; r < R; ++r) iters_out[r] = iters[(size_t)r];
    if (best_restart_out) *best_restart_out = best;
    return SC_OK;
}

namespace sc {
// exact sequential sums of the nseg segments of device array d_vals (host segment offsets):
// the seqsum pipeline of the k-means replica run once, synchronously, on the current device
static int32_t seqsum_device(const double *d_vals, int32_t nseg, const int64_t *seg_off,
                             double *totals, double *chunk_starts) {
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    std::vector<int64_t> cofs(nseg + 1, 0);
    for (int s = 0; s < nseg; ++s)
        cofs[s + 1] = cofs[s] + (seg_off[s + 1] - seg_off[s] + kSeqChunk - 1) / kSeqChunk;
    const int64_t nch = cofs[nseg];
    double *d_A = nullptr, *d_vmax = nullptr, *d_cs = nullptr, *d_tot = nullptr;
    int64_t *d_seg = nullptr, *d_cofs = nullptr, *d_q0 = nullptr, *d_q1 = nullptr, *d_nch = nullptr;
    int32_t *d_kp = nullptr, *d_neg = nullptr, *d_skp = nullptr;
    int64_t *d_sq0 = nullptr, *d_sq1 = nullptr;
    double *d_svm = nullptr;
    auto al = [](void **p, size_t b) { return cudaMalloc(p, b ? b : 16); };
    const size_t nsup = (size_t)nch / kSuper + 1;
    cudaError_t e = al((void **)&d_A, nch * 8);
    if (!e) e = al((void **)&d_vmax, nch * 8);
    if (!e) e = al((void **)&d_cs, nch * 8);
    if (!e) e = al((void **)&d_tot, nseg * 8);
    if (!e) e = al((void **)&d_seg, (nseg + 1) * 8);
    if (!e) e = al((void **)&d_cofs, (nseg + 1) * 8);
    if (!e) e = al((void **)&d_q0, nch * 8);
    if (!e) e = al((void **)&d_q1, nch * 8);
    if (!e) e = al((void **)&d_nch, 8);
    if (!e) e = al((void **)&d_kp, nch * 4);
    if (!e) e = al((void **)&d_neg, nseg * 4);
    if (!e) e = al((void **)&d_skp, nsup * 4);
    if (!e) e = al((void **)&d_sq0, nsup * 8);
    if (!e) e = al((void **)&d_sq1, nsup * 8);
    if (!e) e = al((void **)&d_svm, nsup * 8);
    if (!e) e = cudaMemcpy(d_seg, seg_off, (nseg + 1) * 8, cudaMemcpyHostToDevice);
    if (!e) e = cudaMemcpy(d_cofs, cofs.data(), (nseg + 1) * 8, cudaMemcpyHostToDevice);
    if (!e) e = cudaMemcpy(d_nch, &nch, 8, cudaMemcpyHostToDevice);
    if (!e) e = cudaMemset(d_neg, 0, nseg * 4);
    if (!e) {
        SegView v{d_vals, d_seg, d_cofs, nseg, nullptr, 1};
        SeqWork w{d_A, d_vmax, d_kp, d_q0, d_q1, d_cs, d_neg, d_tot, d_sq0, d_sq1, d_svm, d_skp};
        const int gw = (int)std::min<int64_t>((nch * 32 + 255) / 256 + 1, (int64_t)sms * 8);
        const int gs = (nseg * 32 + 255) / 256;
        k_seq_summarize<<<gw, 256>>>(v, w, d_nch);
        k_seq_flip<<<gw, 256>>>(v, w, d_nch);
        k_seq_predict<><<<nseg, 32 * kPredictWarps>>>(v, w);
        k_seq_chunkmap<<<gw, 256>>>(v, w, d_nch);
        k_seq_superize<<<gw, 256>>>(v, w, d_nch);
        k_seq_compose<<<(nseg + kComposeWarps - 1) / kComposeWarps, 32 * kComposeWarps, kComposeSmem>>>(
            v, w, chunk_starts != nullptr);
        e = cudaDeviceSynchronize();
    }
    if (!e) e = cudaMemcpy(totals, d_tot, nseg * 8, cudaMemcpyDeviceToHost);
    if (!e && chunk_starts) e = cudaMemcpy(chunk_starts, d_cs, nch * 8, cudaMemcpyDeviceToHost);
    void *ps[] = {d_A, d_vmax, d_cs, d_tot, d_seg, d_cofs, d_q0, d_q1, d_nch, d_kp, d_neg,
                  d_skp, d_sq0, d_sq1, d_svm};
    for (void *p : ps) cudaFree(p);
    SC_CUDA(e);
    return SC_OK;
}

// histograms; out-of-range keys are not counted (the totals then disagree with m / n and
// the caller reports the input error)
__global__ void k_key_hist(const int32_t *__restrict__ keys, int64_t m, int32_t nkeys,
                           int64_t *__restrict__ cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t q = keys[i];
        if (q >= 0 && q < nkeys) atomicAdd(reinterpret_cast<unsigned long long *>(cnt + q), 1ull);
    }
}

__global__ void k_pair_hist(const int64_t *__restrict__ a, const int64_t *__restrict__ b, int64_t n,
                            int64_t ka, int64_t kb, int64_t *__restrict__ cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = a[i], y = b[i];
        if (x >= 0 && x < ka && y >= 0 && y < kb)
            atomicAdd(reinterpret_cast<unsigned long long *>(cnt + x * kb + y), 1ull);
    }
}
}  // namespace sc

extern "C" int32_t sc_seqsum(const double *vals, int32_t nseg, const int64_t *seg_off,
                             int32_t device, double *totals, double *chunk_starts) {
    using namespace sc;
    SC_REQUIRE(vals && seg_off && totals && nseg >= 1, SC_E_INVALID, "null argument");
    for (int s = 0; s < nseg; ++s)
        SC_REQUIRE(seg_off[s + 1] >= seg_off[s], SC_E_RANGE, "segment offsets decrease");
    SC_CUDA(cudaSetDevice(device));
    const int64_t n = seg_off[nseg];
    double *d_vals = nullptr;
    SC_CUDA(cudaMalloc((void **)&d_vals, n ? n * 8 : 16));
    cudaError_t e = cudaMemcpy(d_vals, vals, n * 8, cudaMemcpyHostToDevice);
    if (e) {
        cudaFree(d_vals);
        SC_CUDA(e);
    }
    const int32_t st = seqsum_device(d_vals, nseg, seg_off, totals, chunk_starts);
    cudaFree(d_vals);
    return st;
}

namespace sc {
// np.add.at over device arrays (dk, dv are consumed as sort input)
static int32_t keyed_sums_device(int32_t *dk, double *dv, int64_t m, int32_t nkeys,
                                 double *sums_out, int64_t *counts_out) {
    int32_t *dk2 = nullptr;
    double *dv2 = nullptr;
    int64_t *dc = nullptr;
    void *tmp = nullptr;
    size_t tb = 0;
    int end_bit = 1;
    while ((1ll << end_bit) < (long long)nkeys) ++end_bit;
    std::vector<int64_t> cnt((size_t)nkeys), seg((size_t)nkeys + 1, 0);
    cudaError_t e = cudaMalloc((void **)&dk2, m ? m * 4 : 16);
    if (!e) e = cudaMalloc((void **)&dv2, m ? m * 8 : 16);
    if (!e) e = cudaMalloc((void **)&dc, (size_t)nkeys * 8);
    if (!e) e = cudaMemset(dc, 0, (size_t)nkeys * 8);
    if (!e && m) {
        k_key_hist<<<1184, 256>>>(dk, m, nkeys, dc);
        e = cudaGetLastError();
    }
    if (!e) e = cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dk2, dv, dv2, (int)m, 0, end_bit);
    if (!e) e = cudaMalloc(&tmp, tb ? tb : 16);
    if (!e) e = cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dk2, dv, dv2, (int)m, 0, end_bit);
    if (!e) e = cudaMemcpy(cnt.data(), dc, (size_t)nkeys * 8, cudaMemcpyDeviceToHost);
    int32_t st = SC_OK;
    if (!e) {
        for (int32_t q = 0; q < nkeys; ++q) seg[(size_t)q + 1] = seg[(size_t)q] + cnt[(size_t)q];
        if (seg[(size_t)nkeys] != m) {
            st = fail(SC_E_RANGE, "keys must lie in [0, %d)", nkeys);
        } else {
            st = seqsum_device(dv2, nkeys, seg.data(), sums_out, nullptr);
            if (counts_out) std::memcpy(counts_out, cnt.data(), (size_t)nkeys * 8);
        }
    }
    for (void *p : {(void *)dk2, (void *)dv2, (void *)dc, tmp}) cudaFree(p);
    SC_CUDA(e);
    return st;
}

// crossing entries of the CSR (label[row] != label[col]) in CSR order: key = label[row],
// val = weight (1.0 if w is null); non-crossing entries get key -1
__global__ void k_cut_keys(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                           const double *__restrict__ w, const int64_t *__restrict__ lab, int64_t n,
                           int32_t *__restrict__ keys, double *__restrict__ vals) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lr = lab[r];
        for (int64_t j = rp[r]; j < rp[r + 1]; ++j) {
            const bool cross = lab[col[j]] != lr;
            keys[j] = cross ? (int32_t)lr : -1;
            vals[j] = w ? w[j] : 1.0;
        }
    }
}

struct NonNeg {
    __device__ bool operator()(const int32_t &k) const { return k >= 0; }
};

__global__ void k_flags_from_keys(const int32_t *__restrict__ keys, int64_t m,
                                  int32_t *__restrict__ flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        flags[i] = keys[i] >= 0;
}
}  // namespace sc

// np.add.at(out, keys, vals) for out = zeros(nkeys): stable sort by key on the device, then
// every key's values summed left to right in input order (the exact np.add.at rounding).
extern "C" int32_t sc_keyed_sums(const int32_t *keys, const double *vals, int64_t m,
                                 int32_t nkeys, int32_t device, double *sums_out,
                                 int64_t *counts_out) {
    using namespace sc;
    SC_REQUIRE(keys && vals && sums_out && nkeys >= 1 && m >= 0 && m < (int64_t(1) << 31),
               SC_E_INVALID, "bad argument");
    SC_CUDA(cudaSetDevice(device));
    int32_t *dk = nullptr;
    double *dv = nullptr;
    cudaError_t e = cudaMalloc((void **)&dk, m ? m * 4 : 16);
    if (!e) e = cudaMalloc((void **)&dv, m ? m * 8 : 16);
    if (!e && m) e = cudaMemcpy(dk, keys, m * 4, cudaMemcpyHostToDevice);
    if (!e && m) e = cudaMemcpy(dv, vals, m * 8, cudaMemcpyHostToDevice);
    int32_t st = SC_OK;
    if (!e) st = keyed_sums_device(dk, dv, m, nkeys, sums_out, counts_out);
    cudaFree(dk);
    cudaFree(dv);
    SC_CUDA(e);
    return st;
}

// cut weight of every part: np.add.at(cut, labels[src[crossing]], w[crossing]) with the
// crossing entries in CSR order (partition_conductances, metrics.py:143-146)
extern "C" int32_t sc_cut_sums(const int64_t *row_ptr, const int32_t *col, const double *w,
                               const int64_t *labels, int64_t n, int64_t nnz, int32_t k,
                               int32_t device, double *cut_out) {
    using namespace sc;
    SC_REQUIRE(row_ptr && (col || nnz == 0) && labels && cut_out && n >= 1 && k >= 1 &&
                   nnz < (int64_t(1) << 31),
               SC_E_INVALID, "bad argument");
    for (int64_t i = 0; i < n; ++i)
        SC_REQUIRE(labels[i] >= 0 && labels[i] < k, SC_E_RANGE, "label %lld of vertex %lld "
                   "outside [0, %d)", (long long)labels[i], (long long)i, k);
    SC_CUDA(cudaSetDevice(device));
    int64_t *drp = nullptr, *dlab = nullptr;
    int32_t *dcol = nullptr, *dkeys = nullptr, *dk = nullptr, *dnsel = nullptr;
    double *dw = nullptr, *dvals = nullptr, *dv = nullptr;
    void *tmp = nullptr;
    size_t tb = 0;
    cudaError_t e = cudaMalloc((void **)&drp, (n + 1) * 8);
    if (!e) e = cudaMalloc((void **)&dlab, n * 8);
    if (!e) e = cudaMalloc((void **)&dcol, nnz ? nnz * 4 : 16);
    if (!e && w) e = cudaMalloc((void **)&dw, nnz ? nnz * 8 : 16);
    if (!e) e = cudaMalloc((void **)&dkeys, nnz ? nnz * 4 : 16);
    if (!e) e = cudaMalloc((void **)&dvals, nnz ? nnz * 8 : 16);
    if (!e) e = cudaMalloc((void **)&dk, nnz ? nnz * 4 : 16);
    if (!e) e = cudaMalloc((void **)&dv, nnz ? nnz * 8 : 16);
    if (!e) e = cudaMalloc((void **)&dnsel, 16);
    if (!e) e = cudaMemcpy(drp, row_ptr, (n + 1) * 8, cudaMemcpyHostToDevice);
    if (!e) e = cudaMemcpy(dlab, labels, n * 8, cudaMemcpyHostToDevice);
    if (!e && nnz) e = cudaMemcpy(dcol, col, nnz * 4, cudaMemcpyHostToDevice);
    if (!e && w && nnz) e = cudaMemcpy(dw, w, nnz * 8, cudaMemcpyHostToDevice);
    if (!e) {
        k_cut_keys<<<1184, 256>>>(drp, dcol, dw, dlab, n, dkeys, dvals);
        e = cudaGetLastError();
    }
    // order-preserving compaction of the crossing entries (keys >= 0), values alongside
    if (!e) e = cub::DeviceSelect::If(nullptr, tb, dkeys, dk, dnsel, (int)nnz, NonNeg());
    size_t tb2 = 0;
    if (!e) e = cub::DeviceSelect::Flagged(nullptr, tb2, dvals, dkeys, dv, dnsel, (int)nnz);
    if (!e) e = cudaMalloc(&tmp, std::max(std::max(tb, tb2), (size_t)16));
    int32_t nsel = 0;
    // values first (flags = keys >= 0 computed from a copy of keys as 0/1), then keys
    if (!e) {
        k_flags_from_keys<<<1184, 256>>>(dkeys, nnz, dk);
        e = cudaGetLastError();
    }
    if (!e) e = cub::DeviceSelect::Flagged(tmp, tb2, dvals, dk, dv, dnsel, (int)nnz);
    if (!e) e = cub::DeviceSelect::If(tmp, tb, dkeys, dk, dnsel, (int)nnz, NonNeg());
    if (!e) e = cudaMemcpy(&nsel, dnsel, 4, cudaMemcpyDeviceToHost);
    int32_t st = SC_OK;
    if (!e) st = keyed_sums_device(dk, dv, nsel, k, cut_out, nullptr);
    for (void *p : {(void *)drp, (void *)dlab, (void *)dcol, (void *)dw, (void *)dkeys,
                    (void *)dvals, (void *)dk, (void *)dv, (void *)dnsel, tmp})
        cudaFree(p);
    SC_CUDA(e);
    return st;
}

// contingency counts[a][b] of two labelings (exact integer counts)
extern "C" int32_t sc_contingency(const int64_t *la, const int64_t *lb, int64_t n, int32_t ka,
                                  int32_t kb, int32_t device, int64_t *counts_out) {
    using namespace sc;
    SC_REQUIRE(la && lb && counts_out && n >= 0 && ka >= 1 && kb >= 1, SC_E_INVALID,
               "bad argument");
    SC_CUDA(cudaSetDevice(device));
    int64_t *da = nullptr, *db = nullptr, *dc = nullptr;
    const size_t cells = (size_t)ka * kb;
    cudaError_t e = cudaMalloc((void **)&da, n ? n * 8 : 16);
    if (!e) e = cudaMalloc((void **)&db, n ? n * 8 : 16);
    if (!e) e = cudaMalloc((void **)&dc, cells * 8);
    if (!e && n) e = cudaMemcpy(da, la, n * 8, cudaMemcpyHostToDevice);
    if (!e && n) e = cudaMemcpy(db, lb, n * 8, cudaMemcpyHostToDevice);
    if (!e) e = cudaMemset(dc, 0, cells * 8);
    if (!e && n) {
        k_pair_hist<<<1184, 256>>>(da, db, n, ka, kb, dc);
        e = cudaGetLastError();
    }
    if (!e) e = cudaMemcpy(counts_out, dc, cells * 8, cudaMemcpyDeviceToHost);
    cudaFree(da);
    cudaFree(db);
    cudaFree(dc);
    SC_CUDA(e);
    int64_t tot = 0;
    for (size_t c = 0; c < cells; ++c) tot += counts_out[c];
    SC_REQUIRE(tot == n, SC_E_RANGE, "labels must lie in [0, %d) x [0, %d)", ka, kb);
    return SC_OK;
}