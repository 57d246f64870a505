// sc_graph.cu -- graph handle, Irwin-Hall start vector (K1) and the fused lazy-random-walk
// SpMV (K2 + K3) for sm_100a.
//
// Reference semantics (paths under /root/reference/pkg/src/specluster):
//   power_method           spectral.py:87-102   x <- M x, t times, no normalisation
//   rw operator            SURVEY.md CS2        M x = 0.5*x + 0.5*(A @ (x/d))
//   SignlessLaplacianOp    spectral.py:52-57    M x = 0.5*x + 0.5*(s*(A @ (s*x)))
//   scipy csr_matvec       (sparsetools)        per row: sum = 0; sum += A_ij * v_j in
//                                               stored column order, no FMA
//
// Layout: the CSR is re-laid out once, on the device, as SELL-32-sigma.
//   * rows are renumbered: inside every window of kSigma consecutive rows, rows are
//     stably sorted by decreasing length; rows longer than kSellMax ("wide" rows) go to
//     the end.  Column indices are renamed with the same permutation.  Renaming changes
//     WHERE z values live, never the ORDER of the products inside a row, so every row sum
//     stays bit-identical to scipy's.
//   * 32 consecutive renumbered rows form a slice stored column-major (entry t of the
//     slice's row `lane` at slice_base + 32 t + lane), padded to the slice's longest row.
//     One warp owns a slice, one lane owns a row: entry loads are perfectly coalesced
//     128-byte lines, each lane adds its own products strictly left to right, and there
//     is no shared memory and no barrier on the hot path -- the kernel runs at the
//     random-gather limit of the L1/L2 request path.
//   * wide rows: one warp per row; 32 entries per step are gathered in parallel and the
//     warp folds them in order with shuffles (every lane holds the same running sum).
// The epilogue fuses the lazy blend 0.5 x + sign*0.5 s and the degree scaling of the next
// iterate: it writes x_{t+1} and z_{t+1} = x_{t+1} / d, the vector the next step gathers,
// and after the last step the embedding f = D^-1 x_T itself.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda/atomic>
#include <thread>
#include <vector>

#include "sc_common.cuh"

namespace sc {
#include "sc_hostcopy.cuh"
}  // namespace sc

namespace sc {

thread_local std::string g_last_error;

void set_error(const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

int32_t fail(int32_t code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

constexpr int kSlice = 32;         // rows per slice (one per lane)
constexpr int kSigma = 4096;       // sorting window (rows)
#ifndef SC_SELL_MAX
#define SC_SELL_MAX 256
#endif
constexpr int kSellMax = SC_SELL_MAX;  // longer rows are laid out first, globally length-sorted
static_assert(kSellMax < 512, "the renumbering key packs kSellMax - length into 9 bits");
constexpr int kExtreme = kSellMax;  // longer rows ("wide") get one warp each
constexpr int64_t kWideKeyMax = int64_t(1) << 24;  // wide rows are ordered by min(length, this)
constexpr uint32_t kPad = 0xffffffffu;  // padding entry of a slice
constexpr int kStepTPB = 256;      // 8 warps per CTA
#ifndef SC_UNROLL
#define SC_UNROLL 8
#endif
constexpr int kUnroll = SC_UNROLL;  // slice steps in flight per lane

struct StepArgs {
    const int64_t *slice_ptr;  // nslices + 1 (entries, multiples of 32)
    const uint32_t *col;       // SELL column-major entries (renamed columns / kPad)
    const double *val;         // SELL weights or null (unit)
    const int64_t *wide_ptr;   // nwide + 1 into wcol / wval
    const uint32_t *wcol;
    const double *wval;
    const double *scale;       // deg (rw) or deg^-1/2 (sym), renumbered order
    const double *x_in;
    const double *z_in;        // gathered vector, indexed by renamed column
    double *x_out;
    double *z_out;             // written at col_offset + row
    int64_t n_sell, n_wide, nslices;
    int64_t slice_lo, slice_hi; // slices of this launch (a row range of the shard)
    int64_t wide_lo, wide_hi;   // wide rows of this launch
    int64_t col_offset;
    int wide_blocks;           // CTAs of the wide-row kernel
    double hs;                 // +0.5 or -0.5
    // fused exchange (multi-GPU, peer memory over NVLink): every z value written is also
    // stored at the same offset of each peer's z allocation (peer_base[q] + peer_off + i)
    double *const *peer_base;
    int64_t peer_off;
    int npeer;
    const float *val32;   // fp32 weights (SC_CREATE_FP32_VALUES), SELL / wide layouts
    const float *wval32;
    int zhint;            // 1: z space larger than the L2 -> 64-byte L2 fetch hint on the gathers
};

// The z gather of the SELL kernels (read-only path).  An L2 miss of a plain load fetches a whole
// 128-byte line from DRAM (measured at config 5: 118 B of DRAM reads per random cross-block
// gather, 32.5 GB per step against 8.9 GB without those edges); the L2::64B prefetch-size hint
// halves that (21.7 GB per step, 7.50 -> 7.10 ms).  L2::128B equals the default, L2::256B and
// L1::no_allocate are worse (35.1 / 35.7 GB); there is no 32-byte hint and
// cudaLimitMaxL2FetchGranularity changes nothing.  When z fits the L2 the hint only costs
// (config 2 panels 127.3 -> 131.0 us, C3/C4 +0.5 %), so it is used when the z space is larger
// than the L2 (StepArgs::zhint, set by launch_step).
__device__ __forceinline__ double ldz64(const double *p) {
    double v;
    asm("ld.global.nc.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
// run-time selected form (wide-row kernel: registers to spare); the slice kernel takes the hint
// as a template parameter -- either form of a run-time choice spills its 48-register weighted
// variant (260 -> 279 us at C3)
__device__ __forceinline__ double ldz(const double *p, int hint64) {
    double v;
    asm("{\n .reg .pred h;\n setp.ne.s32 h, %2, 0;\n"
        " @h ld.global.nc.L2::64B.f64 %0, [%1];\n"
        " @!h ld.global.nc.f64 %0, [%1];\n}\n"
        : "=d"(v)
        : "l"(p), "r"(hint64));
    return v;
}

template <bool SYM>
__device__ __forceinline__ void row_epilogue(const StepArgs &a, int64_t r, double s, double xr,
                                             double sc) {
    if (SYM) s = __dmul_rn(sc, s);
    const double y = __dadd_rn(__dmul_rn(0.5, xr), __dmul_rn(a.hs, s));
    __stcs(a.x_out + r, y);
    const double zv = SYM ? __dmul_rn(sc, y) : __ddiv_rn(y, sc);
    a.z_out[a.col_offset + r] = zv;
    for (int q = 0; q < a.npeer; ++q) a.peer_base[q][a.peer_off + a.col_offset + r] = zv;
}

// make this thread's peer stores visible system-wide before the barrier kernel's flag
__device__ __forceinline__ void peer_fence(const StepArgs &a) {
    if (a.npeer) __threadfence_system();
}

// Wide rows (> kExtreme entries): one warp per row.  The in-order fold of a row is a chain
// of dependent adds, so the row's time is bounded below by (entries x add latency); every
// memory latency is kept off that chain: the warp gathers 128 products per step into its
// double-buffered shared-memory slot while lane 0 adds the previous 128 strictly in order
// (the scipy order), and the column indices are fetched one step earlier still, so a
// gather never waits for its index load.
constexpr int kWideBatch = 128;
// Grid cap of the wide-row kernel (x SM count).  The kernel needs 114 registers per thread, so
// two resident CTAs leave the concurrent slice kernel no room on an SM and the two ran back to
// back (C3: 207 us slices + 74 us wide rows = 272 us per step).  One CTA per SM keeps 36 K
// registers for the slices: 272 -> 261 us.  Graphs whose wide rows hold a quarter of the entries
// or more keep two.
constexpr int kWideCtasPerSM = 1;
constexpr int kWidePL = kWideBatch / 32;

// s + v[0] + v[1] + ... + v[m-1], left to right (v 16-byte aligned): shared-memory loads of
// the next 8 values are issued before the adds of the current 8
__device__ __forceinline__ double wide_fold(double s, const double *v, int m) {
    const double2 *v2 = reinterpret_cast<const double2 *>(v);
    const int mf = m & ~7;
    double2 cur[4], nxt[4];
    if (mf) {
#pragma unroll
        for (int u = 0; u < 4; ++u) cur[u] = v2[u];
    }
    for (int t = 0; t < mf; t += 8) {
        const bool more = t + 8 < mf;
        if (more) {
#pragma unroll
            for (int u = 0; u < 4; ++u) nxt[u] = v2[(t + 8) / 2 + u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            s = __dadd_rn(s, cur[u].x);
            s = __dadd_rn(s, cur[u].y);
        }
        if (more) {
#pragma unroll
            for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
        }
    }
    for (int t = mf; t < m; ++t) s = __dadd_rn(s, v[t]);
    return s;
}

#ifndef SC_WIDE_MINB
#define SC_WIDE_MINB 2  // 114 registers; 3 (80) and 4 (64) spill into the in-order fold: 278 / 333 us at C3
#endif
template <bool UNIT, bool SYM, bool F32 = false>
__global__ void __launch_bounds__(kStepTPB, SC_WIDE_MINB) k_rw_wide(StepArgs a) {
    __shared__ __align__(16) double wbuf[kStepTPB / 32][2][kWideBatch];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    // rows are dealt round-robin over the grid's warps (they come in decreasing length, so the
    // longest in-order folds start first); the grid is capped at a few CTAs per SM so the
    // concurrent slice kernel keeps most of every SM (launch_step)
    for (int64_t w = a.wide_lo + (int64_t)blockIdx.x * (kStepTPB / 32) + warp; w < a.wide_hi;
         w += (int64_t)gridDim.x * (kStepTPB / 32)) {
    const int64_t r = a.n_sell + w;
    const double xr = __ldcs(a.x_in + r), sc = __ldcs(a.scale + r);
    const int64_t lo = a.wide_ptr[w], hi = a.wide_ptr[w + 1];
    double *buf0 = wbuf[warp][0], *buf1 = wbuf[warp][1];
    auto load_cols = [&](int64_t base, uint32_t (&c)[kWidePL]) {
#pragma unroll
        for (int q = 0; q < kWidePL; ++q) {
            const int64_t j = base + 32 * q + lane;
            c[q] = j < hi ? __ldcs(a.wcol + j) : 0u;
        }
    };
    // loads only: the products are formed after the fold, so the fold never waits on them
    auto issue = [&](int64_t base, const uint32_t (&c)[kWidePL], double (&zr)[kWidePL],
                     double (&wr)[kWidePL]) {
#pragma unroll
        for (int q = 0; q < kWidePL; ++q) {
            const int64_t j = base + 32 * q + lane;
            zr[q] = 0.0;
            wr[q] = 1.0;
            if (j < hi) {
                zr[q] = ldz(a.z_in + c[q], a.zhint);
                if (!UNIT) wr[q] = F32 ? (double)__ldcs(a.wval32 + j) : __ldcs(a.wval + j);
            }
        }
    };
    auto store = [&](double *buf, const double (&zr)[kWidePL], const double (&wr)[kWidePL]) {
#pragma unroll
        for (int q = 0; q < kWidePL; ++q) buf[32 * q + lane] = UNIT ? zr[q] : __dmul_rn(wr[q], zr[q]);
    };
    uint32_t cn[kWidePL];
    double zr[kWidePL], wr[kWidePL];
    load_cols(lo, cn);
    issue(lo, cn, zr, wr);
    if (lo + kWideBatch < hi) load_cols(lo + kWideBatch, cn);  // indices of step 1
    store(buf0, zr, wr);
    double s = 0.0;
    for (int64_t base = lo; base < hi; base += kWideBatch) {
        __syncwarp();
        const bool more = base + kWideBatch < hi;
        uint32_t cnn[kWidePL];
        if (more) {
            issue(base + kWideBatch, cn, zr, wr);  // in flight during the fold below
            if (base + 2 * kWideBatch < hi) load_cols(base + 2 * kWideBatch, cnn);
        }
        if (lane == 0) {
            const int m = (int)(hi - base < kWideBatch ? hi - base : kWideBatch);
            s = wide_fold(s, buf0, m);
        }
        __syncwarp();
        if (more) {
            store(buf1, zr, wr);
#pragma unroll
            for (int q = 0; q < kWidePL; ++q) cn[q] = cnn[q];
        }
        double *tb = buf0;
        buf0 = buf1;
        buf1 = tb;
    }
    if (lane == 0) row_epilogue<SYM>(a, r, s, xr, sc);
    __syncwarp();
    }
    peer_fence(a);
}

#ifndef SC_MINB_U
#define SC_MINB_U 1
#endif
#ifndef SC_MINB_W
#define SC_MINB_W 5  // weighted: 5 CTAs of 256 (C4 539 -> 497 us, C3 275 -> 270; 6 spills and thrashes C4)
#endif
template <bool UNIT, bool SYM, bool F32 = false, bool BIGZ = false>
__global__ void __launch_bounds__(kStepTPB, (UNIT || F32 || BIGZ) ? SC_MINB_U : SC_MINB_W) k_rw_step(StepArgs a) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    // ---- SELL slices: one warp per slice, one lane per row
    const int64_t sl = a.slice_lo + (int64_t)blockIdx.x * (kStepTPB / 32) + warp;
    if (sl >= a.slice_hi) return;
    const int64_t r = sl * kSlice + lane;
    const bool live = r < a.n_sell;
    double xr = 0.0, sc = 1.0;
    if (live) {
        xr = __ldcs(a.x_in + r);
        sc = __ldcs(a.scale + r);
    }
    const int64_t base = a.slice_ptr[sl];
    const int width = (int)((a.slice_ptr[sl + 1] - base) >> 5);
    const uint32_t *cp = a.col + base + lane;
    const double *vp = (UNIT || F32) ? nullptr : a.val + base + lane;
    const float *vp32 = F32 ? a.val32 + base + lane : nullptr;
    // Software pipeline: batch i+1's column indices are loaded while batch i's z values
    // (and weights, which do not depend on the indices) are fetched and added, so a slice
    // pays about one memory latency per batch; the last batch is predicated, not peeled.
    auto load_cols = [&](int t0, uint32_t (&cc)[kUnroll]) {
#pragma unroll
        for (int q = 0; q < kUnroll; ++q) {
            const int t = t0 + q;
            cc[q] = t < width ? __ldcs(cp + (int64_t)t * kSlice) : kPad;
        }
    };
    uint32_t c[kUnroll];
    load_cols(0, c);
    double s = 0.0;
    for (int t = 0; t < width; t += kUnroll) {
        uint32_t cn[kUnroll];
        const bool more = t + kUnroll < width;
        if (more) load_cols(t + kUnroll, cn);
        double p[kUnroll];
#pragma unroll
        for (int q = 0; q < kUnroll; ++q) {
            p[q] = 0.0;
            if (c[q] != kPad) {
                const double zv = BIGZ ? ldz64(a.z_in + c[q]) : __ldg(a.z_in + c[q]);
                const double wv = UNIT ? 1.0
                                  : F32 ? (double)__ldcs(vp32 + (int64_t)(t + q) * kSlice)
                                        : __ldcs(vp + (int64_t)(t + q) * kSlice);
                p[q] = UNIT ? zv : __dmul_rn(wv, zv);
            }
        }
#pragma unroll
        for (int q = 0; q < kUnroll; ++q)
            if (c[q] != kPad) s = __dadd_rn(s, p[q]);
        if (more) {
#pragma unroll
            for (int q = 0; q < kUnroll; ++q) c[q] = cn[q];
        }
    }
    if (live) row_epilogue<SYM>(a, r, s, xr, sc);
    peer_fence(a);
}

// ---- block power method: L columns at once (pm_log_k, spectral.py:52-57 on an (n, L)
// block).  scipy's csr_matvecs adds, per row and per stored entry, a_ij * x_jk to every
// column k in turn, so each column sees exactly the single-vector summation order; here a
// lane owns a row and keeps L accumulators, and the gathered vector z = d^-1/2 x is stored
// row-major [n][L] so one gather brings a row's L values (one or a few sectors) instead of
// L scattered ones.
struct BlkArgs {
    const int64_t *slice_ptr;
    const uint32_t *col;
    const double *val;
    const int64_t *wide_ptr;
    const uint32_t *wcol;
    const double *wval;
    const double *isd;  // d^-1/2, renumbered
    const double *x_in, *z_in;
    double *x_out, *z_out;
    int64_t n_sell, nslices, n_wide;
};

// 256-bit read-only load (sm_100: LDG.E.ENL2.256), p 32-byte aligned
__device__ __forceinline__ void ld_nc_v4(const double *p, double &a, double &b, double &c,
                                         double &d) {
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
                 : "l"(p));
}

template <int L>
__device__ __forceinline__ void blk_epilogue(const BlkArgs &a, int64_t r, const double (&acc)[L],
                                             const double (&xr)[L], double sc) {
#pragma unroll
    for (int q = 0; q < L; ++q) {
        const double y = __dadd_rn(__dmul_rn(0.5, xr[q]), __dmul_rn(0.5, __dmul_rn(sc, acc[q])));
        a.x_out[r * L + q] = y;
        a.z_out[r * L + q] = __dmul_rn(sc, y);
    }
}

template <int L, bool UNIT>
__global__ void __launch_bounds__(kStepTPB) k_blk_step(BlkArgs a) {
    constexpr int U = L <= 4 ? 4 : 2;  // entries in flight per lane
    const int lane = threadIdx.x & 31;
    const int64_t sl = (int64_t)blockIdx.x * (kStepTPB / 32) + (threadIdx.x >> 5);
    if (sl >= a.nslices) return;
    const int64_t r = sl * kSlice + lane;
    const bool live = r < a.n_sell;
    double xr[L], acc[L];
    double sc = 1.0;
#pragma unroll
    for (int q = 0; q < L; ++q) {
        acc[q] = 0.0;
        xr[q] = live ? a.x_in[r * L + q] : 0.0;
    }
    if (live) sc = a.isd[r];
    const int64_t base = a.slice_ptr[sl];
    const int width = (int)((a.slice_ptr[sl + 1] - base) >> 5);
    const uint32_t *cp = a.col + base + lane;
    const double *vp = UNIT ? nullptr : a.val + base + lane;
    for (int t = 0; t < width; t += U) {
        uint32_t c[U];
        double v[U][L], w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            c[u] = t + u < width ? __ldcs(cp + (int64_t)(t + u) * kSlice) : kPad;
            w[u] = (!UNIT && c[u] != kPad) ? __ldcs(vp + (int64_t)(t + u) * kSlice) : 1.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < L; q += 4) {  // one 32-byte load per 4 columns (L % 4 == 0)
                if (c[u] != kPad) ld_nc_v4(a.z_in + (int64_t)c[u] * L + q, v[u][q], v[u][q + 1],
                                            v[u][q + 2], v[u][q + 3]);
                else v[u][q] = v[u][q + 1] = v[u][q + 2] = v[u][q + 3] = 0.0;
            }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (c[u] != kPad)
#pragma unroll
                for (int q = 0; q < L; ++q)
                    acc[q] = __dadd_rn(acc[q], UNIT ? v[u][q] : __dmul_rn(w[u], v[u][q]));
    }
    if (live) blk_epilogue<L>(a, r, acc, xr, sc);
}

// wide rows: one warp per row; 32 entries per batch are gathered (lane = entry) into the
// warp's shared-memory slot, lanes 0..L-1 then fold them in order for their column while the
// next batch's gathers are in flight
template <int L, bool UNIT>
__global__ void __launch_bounds__(kStepTPB) k_blk_wide(BlkArgs a) {
    __shared__ double wb[kStepTPB / 32][32][L];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t w = (int64_t)blockIdx.x * (kStepTPB / 32) + warp;
    if (w >= a.n_wide) return;
    const int64_t r = a.n_sell + w;
    const int64_t lo = a.wide_ptr[w], hi = a.wide_ptr[w + 1];
    double v[L];
    auto gather = [&](int64_t j) {
#pragma unroll
        for (int q = 0; q < L; ++q) v[q] = 0.0;
        if (j < hi) {
            const int64_t c = __ldcs(a.wcol + j);
            const double wt = UNIT ? 1.0 : __ldcs(a.wval + j);
#pragma unroll
            for (int q = 0; q < L; q += 4) {
                double z0, z1, z2, z3;
                ld_nc_v4(a.z_in + c * L + q, z0, z1, z2, z3);
                v[q] = UNIT ? z0 : __dmul_rn(wt, z0);
                v[q + 1] = UNIT ? z1 : __dmul_rn(wt, z1);
                v[q + 2] = UNIT ? z2 : __dmul_rn(wt, z2);
                v[q + 3] = UNIT ? z3 : __dmul_rn(wt, z3);
            }
        }
    };
    double acc = 0.0;
    gather(lo + lane);
    for (int64_t b = lo; b < hi; b += 32) {
        __syncwarp();
#pragma unroll
        for (int q = 0; q < L; ++q) wb[warp][lane][q] = v[q];
        __syncwarp();
        if (b + 32 < hi) gather(b + 32 + lane);
        if (lane < L) {
            const int m = (int)(hi - b < 32 ? hi - b : 32);
            for (int e = 0; e < m; ++e) acc = __dadd_rn(acc, wb[warp][e][lane]);
        }
    }
    // lane q holds column q's sum; lanes 0..L-1 finish their column
    if (lane < L) {
        const double sc = a.isd[r], xr = a.x_in[r * L + lane];
        const double y = __dadd_rn(__dmul_rn(0.5, xr), __dmul_rn(0.5, __dmul_rn(sc, acc)));
        a.x_out[r * L + lane] = y;
        a.z_out[r * L + lane] = __dmul_rn(sc, y);
    }
}

// out[i*lo + q] = in[idx[i]*li + q] for q < L (row permutation of an [n][L] block between
// row strides li and lo; columns L..lo-1 of out are zero-filled), and z = s * x rows
__global__ void k_gather_rows(const double *__restrict__ in, const int32_t *__restrict__ idx,
                              double *__restrict__ out, int64_t n, int L, int li, int lo) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * lo;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / lo, q = t - i * lo;
        out[t] = q < L ? in[(int64_t)idx[i] * li + q] : 0.0;
    }
}

__global__ void k_scale_rows(const double *__restrict__ x, const double *__restrict__ s,
                             double *__restrict__ z, int64_t n, int L) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * L;
         t += (int64_t)gridDim.x * blockDim.x)
        z[t] = __dmul_rn(s[t / L], x[t]);
}

// z[col_offset + i] = x[i] / d[i]   (rw)   or   x[i] * d[i]^-1/2   (sym)
__global__ void k_scale(const double *__restrict__ x, const double *__restrict__ scale,
                        double *__restrict__ z, int64_t n, int64_t off, int sym,
                        double *const *peer_base = nullptr, int64_t peer_off = 0, int npeer = 0) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = sym ? __dmul_rn(x[i], scale[i]) : __ddiv_rn(x[i], scale[i]);
        z[off + i] = v;
        for (int q = 0; q < npeer; ++q) peer_base[q][peer_off + off + i] = v;
    }
    if (npeer) __threadfence_system();
}

// Cross-GPU barrier of the fused exchange: this rank's epoch counter (flags[kEpochSlot]) is
// bumped, written into slot `rank` of every peer's flag array (release, system scope), and the
// kernel waits until every peer has written at least that epoch into our own array (acquire).
// Launched after each step, it is also what makes the peers' z stores of that step visible.
constexpr int kMaxWorld = 32;
constexpr int kEpochSlot = 63;

__global__ void k_peer_barrier(uint32_t *flags, uint32_t *const *peer_flags, int world, int rank) {
    __shared__ uint32_t e;
    if (threadIdx.x == 0) {
        e = flags[kEpochSlot] + 1;
        flags[kEpochSlot] = e;
    }
    __syncthreads();
    const int q = threadIdx.x;
    if (q < world && q != rank) {
        cuda::atomic_ref<uint32_t, cuda::thread_scope_system> out(peer_flags[q][rank]);
        out.store(e, cuda::memory_order_release);
        cuda::atomic_ref<uint32_t, cuda::thread_scope_system> in(flags[q]);
        while (in.load(cuda::memory_order_acquire) < e) __nanosleep(64);
    }
    __syncthreads();
}

// 1/sqrt(d), as numpy's 1.0 / np.sqrt(d) (spectral.py:49)
__global__ void k_inv_sqrt(const double *__restrict__ d, double *__restrict__ s, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        s[i] = __ddiv_rn(1.0, __dsqrt_rn(d[i]));
}

// K1: Irwin-Hall start vector, written in renumbered order.  Uniform j of global vertex u
// is word j%4 of Philox4x64-10(key, (j/4 + 1, u, 0, 0)); floor(deg) uniforms are summed
// left to right, a fractional degree adds frac * one more uniform (mean deg/2 always).
__global__ void k_irwin_hall(const double *__restrict__ deg, const int32_t *__restrict__ perm,
                             double *__restrict__ x0, int64_t n, int64_t global_row0, uint64_t k0,
                             uint64_t k1) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double d = deg[i];
        const double fl = floor(d);
        const int64_t m = (int64_t)fl;
        const double frac = __dsub_rn(d, fl);
        const int64_t need = m + (frac > 0.0 ? 1 : 0);
        const uint64_t u = (uint64_t)(global_row0 + perm[i]);
        double s = 0.0;
        for (int64_t blk = 0; 4 * blk < need; ++blk) {
            const u64x4 r = philox4x64_10(u64x4{(uint64_t)blk + 1u, u, 0, 0}, k0, k1);
            const uint64_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t j = 4 * blk + q;
                if (j < m) s = __dadd_rn(s, u53(w[q]));
                else if (j < need) s = __dadd_rn(s, __dmul_rn(frac, u53(w[q])));
            }
        }
        x0[i] = s;
    }
}

// out[i] = in[idx[i]]: original -> renumbered order with idx = perm, back with idx = iperm
__global__ void k_gather_perm(const double *__restrict__ in, const int32_t *__restrict__ idx,
                              double *__restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[idx[i]];
}

// ---- construction kernels (once per graph) ----------------------------------------------

// Row checks on the device: stats[2] = first row whose offsets decrease, stats[3] = first
// row with a non-positive / non-finite degree (n if none); for the renumbering:
// stats[0] = rows with <= kSellMax entries, stats[1] = their entries, stats[4] = max length
__global__ void k_validate_rows(const int64_t *__restrict__ rp, const double *__restrict__ deg,
                                int64_t n, int32_t *__restrict__ flag,
                                int64_t *__restrict__ stats) {
    __shared__ unsigned long long sc, ss, smx, sbad, sdeg;
    if (threadIdx.x == 0) {
        sc = ss = smx = 0;
        sbad = sdeg = (unsigned long long)n;
    }
    __syncthreads();
    unsigned long long c = 0, sm = 0, mx = 0, bad = n, bdeg = n;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t len = rp[r + 1] - rp[r];
        if (len < 0 && (unsigned long long)r < bad) bad = r;
        const double d = deg[r];
        if (!(d > 0.0 && d < 1e308) && (unsigned long long)r < bdeg) bdeg = r;
        if (len >= 0 && len <= kSellMax) {
            ++c;
            sm += len;
            if ((unsigned long long)len > mx) mx = len;
        }
    }
    atomicAdd(&sc, c);
    atomicAdd(&ss, sm);
    atomicMax(&smx, mx);
    atomicMin(&sbad, bad);
    atomicMin(&sdeg, bdeg);
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(reinterpret_cast<unsigned long long *>(stats + 0), sc);
        atomicAdd(reinterpret_cast<unsigned long long *>(stats + 1), ss);
        atomicMax(reinterpret_cast<unsigned long long *>(stats + 4), smx);
        // stats[2], [3] start at 0: store n - (first bad) so that 0 means "none"... use min
        // on a biased value instead: first = n - max(n - bad)
        atomicMax(reinterpret_cast<unsigned long long *>(stats + 5), (unsigned long long)n - sbad);
        atomicMax(reinterpret_cast<unsigned long long *>(stats + 6), (unsigned long long)n - sdeg);
    }
}

__global__ void k_finish_stats(int64_t *stats, int64_t n) {
    stats[2] = n - stats[5];
    stats[3] = n - stats[6];
}

// sort key of the SELL renumbering: (window, kSellMax - length); wide rows after every window,
// by decreasing length (sell_order's order exactly)
__global__ void k_sell_keys(const int64_t *__restrict__ rp, int64_t n, int64_t sigma, int64_t nwin,
                            uint32_t *__restrict__ keys, int32_t *__restrict__ iota) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t len = rp[r + 1] - rp[r];
        keys[r] = len <= kSellMax ? (uint32_t)((r / sigma) * 512 + (kSellMax - len))
                                  : (uint32_t)(nwin * 512 + (kWideKeyMax - (len < kWideKeyMax ? len : kWideKeyMax)));
        iota[r] = (int32_t)r;
    }
}

// ---- optional locality-preserving pre-order (SC_CREATE_REORDER_BFS) ----------------------
// Multi-source breadth-first search from every kBfsStride-th vertex: each vertex joins the
// region of the first seed to reach it; vertices are then ordered by (region, level), so a
// region -- a ball of ~kBfsStride vertices -- is contiguous in the new numbering and the rows
// of a slice gather from a small window of z.  Renumbering changes where z values live, never
// the order of a row's products, so results stay bit-identical.
constexpr int64_t kBfsStride = 4096;

__global__ void k_bfs_init(int64_t n, int32_t *__restrict__ region, int32_t *__restrict__ lev,
                           int32_t *__restrict__ cur) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const bool seed = v % kBfsStride == 0;
        region[v] = seed ? (int32_t)(v / kBfsStride) : -1;
        lev[v] = seed ? 0 : -1;
        if (seed) cur[v / kBfsStride] = (int32_t)v;
    }
}

// one warp per frontier vertex, lanes over its neighbours (coalesced column reads); claimed
// vertices are appended with one warp-aggregated atomic per batch
__global__ void k_bfs_expand(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                             int32_t *__restrict__ region, int32_t *__restrict__ lev,
                             const int32_t *__restrict__ cur, int32_t ncur, int32_t *__restrict__ nxt,
                             int32_t *__restrict__ nnxt, int32_t level) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < ncur;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t v = cur[i], rv = region[v];
        const int64_t lo = rp[v], hi = rp[v + 1];
        for (int64_t j0 = lo; j0 < hi; j0 += 32) {
            const int64_t j = j0 + lane;
            bool won = false;
            int32_t u = 0;
            if (j < hi) {
                u = col[j];
                won = region[u] == -1 && atomicCAS(&region[u], -1, rv) == -1;
            }
            const unsigned m = __ballot_sync(0xffffffffu, won);
            if (m) {
                int32_t base = 0;
                if (lane == 0) base = atomicAdd(nnxt, __popc(m));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (won) {
                    lev[u] = level + 1;
                    nxt[base + __popc(m & ((1u << lane) - 1))] = u;
                }
            }
        }
    }
}

// key (region, level); vertices no seed reached keep their original order after all regions
__global__ void k_bfs_keys(int64_t n, const int32_t *__restrict__ region,
                           const int32_t *__restrict__ lev, int64_t nseeds,
                           uint64_t *__restrict__ keys, int32_t *__restrict__ iota) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t rg = region[v] >= 0 ? region[v] : nseeds + v / kBfsStride;
        keys[v] = ((uint64_t)rg << 20) | (uint64_t)(lev[v] >= 0 ? min(lev[v], (1 << 20) - 1) : 0);
        iota[v] = (int32_t)v;
    }
}

// SELL keys over a pre-order: position p holds original row ord[p]
__global__ void k_sell_keys_ord(const int64_t *__restrict__ rp, const int32_t *__restrict__ ord,
                                int64_t n, int64_t sigma, int64_t nwin,
                                uint32_t *__restrict__ keys, int32_t *__restrict__ payload) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = ord[p];
        const int64_t len = rp[r + 1] - rp[r];
        keys[p] = len <= kSellMax ? (uint32_t)((p / sigma) * 512 + (kSellMax - len))
                                  : (uint32_t)(nwin * 512 + (kWideKeyMax - (len < kWideKeyMax ? len : kWideKeyMax)));
        payload[p] = r;
    }
}

// lengths of the wide rows (renumbered order), with a trailing 0 for the exclusive scan
__global__ void k_wide_lens(const int64_t *__restrict__ rp, const int32_t *__restrict__ wperm,
                            int64_t n_wide, int64_t *__restrict__ len) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w <= n_wide;
         w += (int64_t)gridDim.x * blockDim.x)
        len[w] = w < n_wide ? rp[wperm[w] + 1] - rp[wperm[w]] : 0;
}

// out[i] = slot_of[col[i]] (global vertex -> z slot of a multi-GPU plan); *bad = 1 on an
// out-of-range column
__global__ void k_rename_cols(const int32_t *__restrict__ col, int64_t m,
                              const int32_t *__restrict__ slot_of, int64_t n,
                              int32_t *__restrict__ out, int32_t *__restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = col[i];
        if ((uint32_t)c >= (uint64_t)n) {
            *bad = 1;
            out[i] = 0;
        } else {
            out[i] = __ldg(slot_of + c);
        }
    }
}

// flag[0] = 1 if any column index is outside [0, ncols)
__global__ void k_col_range(const int32_t *__restrict__ col, int64_t nnz, int64_t ncols,
                            int32_t *__restrict__ flag) {
    int bad = 0;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = __ldcs(col + j);
        bad |= (c < 0) | ((int64_t)c >= ncols);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) flag[0] = 1;
}

__global__ void k_inverse_perm(const int32_t *__restrict__ perm, int32_t *__restrict__ iperm,
                               int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        iperm[perm[i]] = (int32_t)i;
}

__global__ void k_slice_sizes(const int64_t *__restrict__ rp, const int32_t *__restrict__ perm,
                              int64_t n_sell, int64_t nslices, int64_t *__restrict__ sizes) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslices;
         s += (int64_t)gridDim.x * blockDim.x) {
        int64_t w = 0;
        for (int l = 0; l < kSlice; ++l) {
            const int64_t p = s * kSlice + l;
            if (p < n_sell) {
                const int32_t r = perm[p];
                w = max(w, rp[r + 1] - rp[r]);
            }
        }
        sizes[s] = w * kSlice;
    }
}

// one thread per lane of every slice: copy the renumbered row's entries column-major into
// its slice; lanes past n_sell in the last slice are all padding (the step kernel still
// loads their columns, so they must never hold stale indices)
__global__ void k_fill_sell(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                            const double *__restrict__ val, const int32_t *__restrict__ perm,
                            const int32_t *__restrict__ iperm, const int64_t *__restrict__ slice_ptr,
                            int64_t n_sell, int64_t nslices, int64_t col_offset, int64_t n,
                            int rename, uint32_t *__restrict__ scol, double *__restrict__ sval,
                            float *__restrict__ sval32) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nslices * kSlice;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = p / kSlice, lane = p % kSlice;
        const int64_t base = slice_ptr[s];
        const int64_t width = (slice_ptr[s + 1] - base) / kSlice;
        const int32_t r = p < n_sell ? perm[p] : 0;
        const int64_t lo = p < n_sell ? rp[r] : 0, len = p < n_sell ? rp[r + 1] - lo : 0;
        for (int64_t t = 0; t < width; ++t) {
            const int64_t dst = base + t * kSlice + lane;
            if (t < len) {
                int64_t c = col[lo + t];
                if (rename && c >= col_offset && c < col_offset + n)
                    c = col_offset + iperm[c - col_offset];
                scol[dst] = (uint32_t)c;
                if (sval) sval[dst] = val[lo + t];
                if (sval32) sval32[dst] = __double2float_rn(val[lo + t]);
            } else {
                scol[dst] = kPad;
                if (sval) sval[dst] = 0.0;
                if (sval32) sval32[dst] = 0.0f;
            }
        }
    }
}

__global__ void k_fill_wide(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                            const double *__restrict__ val, const int32_t *__restrict__ perm,
                            const int32_t *__restrict__ iperm, const int64_t *__restrict__ wide_ptr,
                            int64_t n_sell, int64_t n_wide, int64_t col_offset, int64_t n,
                            int rename, uint32_t *__restrict__ wcol, double *__restrict__ wval,
                            float *__restrict__ wval32) {
    const int64_t w = blockIdx.x;
    if (w >= n_wide) return;
    const int32_t r = perm[n_sell + w];
    const int64_t lo = rp[r], len = rp[r + 1] - lo, dst = wide_ptr[w];
    for (int64_t t = threadIdx.x; t < len; t += blockDim.x) {
        int64_t c = col[lo + t];
        if (rename && c >= col_offset && c < col_offset + n) c = col_offset + iperm[c - col_offset];
        wcol[dst + t] = (uint32_t)c;
        if (wval) wval[dst + t] = val[lo + t];
        if (wval32) wval32[dst + t] = __double2float_rn(val[lo + t]);
    }
}

}  // namespace sc

using namespace sc;

namespace sc {
struct PanGroup;
struct WinItem;
}

namespace sc {
struct Multi;  // sc_multi.cuh: one handle over several GPUs
}

struct sc_graph {
    int device = 0;
    int sm_count = 0;
    int64_t l2_bytes = 0;
    int64_t n = 0, nnz = 0, ncols = 0, col_offset = 0, global_row0 = 0;
    int64_t n_sell = 0, n_wide = 0, nslices = 0, sell_entries = 0, wide_entries = 0;
    bool unit = false;
    int32_t *d_perm = nullptr;    // renumbered row -> original local row
    int32_t *d_iperm = nullptr;   // original local row -> renumbered row
    int64_t *d_slice_ptr = nullptr;
    uint32_t *d_col = nullptr;    // SELL entries
    double *d_val = nullptr;
    int64_t *d_wide_ptr = nullptr;
    uint32_t *d_wcol = nullptr;
    double *d_wval = nullptr;
    double *d_deg = nullptr;      // renumbered
    double *d_isd = nullptr;
    double *d_x0 = nullptr;
    double *d_x[2] = {nullptr, nullptr};
    double *d_z[2] = {nullptr, nullptr};
    double *d_tmp = nullptr;      // n doubles: host <-> device reorder staging
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // wide-row kernel, forked from / joined into the step stream
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_fork = nullptr, ev_join = nullptr;
    bool have_x0 = false;
    int result = -1;  // buffer index holding z_T (= f) after the last power_iterate
    cudaGraphExec_t gexec = nullptr;
    int32_t g_T = -1;
    uint32_t g_flags = 0;
    double g_sign = 0.0;
    int64_t bytes = 0;
    bool l2_window = false;
    double *d_f_orig = nullptr;   // f in original vertex order (for the k-means context)
    bool f32 = false;             // weights stored as fp32 (SC_CREATE_FP32_VALUES)
    int64_t bfs_sigma = 0, bfs_nwin = 0;  // SELL window parameters for the BFS pre-order
    float *d_val32 = nullptr, *d_wval32 = nullptr;
    std::vector<std::pair<void *, size_t>> allocs;  // every dmalloc'd buffer (returned to the cache)
    // fused peer exchange (sc_shard_set_peers)
    uint32_t *d_flags = nullptr;        // 64 words: peer epochs [0, world), own epoch [63]
    double **d_peer_z = nullptr;        // npeer peer z-allocation bases
    uint32_t **d_peer_flags = nullptr;  // world peer flag arrays (own slot unused)
    int npeer = 0, world = 1, rank = 0;
    // column-panel layout (sc_panel.cuh; SC_CREATE_PANELS), used for whole-graph steps
    int pan_ctas = 0, pan_slot = 0, pan_groups = 0, pan_rpc = 0;
    int64_t pan_bytes = 0;
    int32_t *d_pan_blk = nullptr;
    sc::PanGroup *d_pan_grp = nullptr;
    uint8_t *d_pan_stream = nullptr;
    int64_t zstride = 0;  // d_z[1] - d_z[0] (ncols + a zero slot, rounded up to 32)
    // row-window layout (sc_window.cuh; SC_CREATE_WINDOWS), used for whole-handle steps
    int win_items = 0;
    int64_t win_far = 0, win_pairs = 0;
    double win_cover = 0.0;
    sc::WinItem *d_win_items = nullptr;
    int64_t *d_win_ptr = nullptr;
    uint32_t *d_win_idx = nullptr;
    double2 *d_win_val = nullptr;
    float2 *d_win_val32 = nullptr;
    uint32_t *d_win_far = nullptr;
    // peers synchronised by stream events (sc_multi.cuh) instead of sc_shard_barrier: the
    // panel kernel may then mirror z into peers too (it has no system fence of its own)
    bool peer_events = false;
    sc::Multi *multi = nullptr;  // multi-GPU handle: the shards live there, this one is a shell
};

namespace sc {  // sc_multi.cuh (included at the end of this file)
static void multi_free(sc_graph *mg);
static int32_t multi_sample(sc_graph *mg, uint64_t key0, uint64_t key1, double *x0_out);
static int32_t multi_set_x0(sc_graph *mg, const double *x0);
static int32_t multi_power(sc_graph *mg, int32_t T, double sign, uint32_t flags, double *xT_out,
                           double *f_out, sc_timing *t_out);
static int32_t multi_download_f(sc_graph *mg, double *f_out);
static const double *multi_f_device(sc_graph *mg);
static int32_t multi_info(const sc_graph *mg, sc_graph_info *o);
}  // namespace sc
// whole-handle entry points that a multi-GPU shell forwards; shard-level ones refuse it
#define SC_NOT_MULTI(g) \
    SC_REQUIRE(!(g)->multi, SC_E_STATE, "not available on a multi-GPU handle")

namespace sc {

// Device buffers of graph handles come from plain cudaMalloc (persistent buffers live as
// long as the handle; the stream-ordered pool is used for the construction staging only) and
// go back to a small process-wide cache on destroy, so a pipeline that builds a graph per
// call does not pay cudaMalloc/cudaFree (whose device-wide synchronisation and unmapping
// cost up to hundreds of ms for a multi-GB graph) every time.  A buffer is cached only after
// the handle's streams are synchronised.  SC_BUFFER_CACHE_MB caps it (default 16384, 0 = off).
namespace {
struct CachedBuf {
    int device;
    size_t bytes;
    void *p;
};
std::mutex g_cache_mu;
std::vector<CachedBuf> g_cache;
size_t g_cache_bytes = 0;

size_t cache_cap() {
    static size_t cap = [] {
        const char *e = getenv("SC_BUFFER_CACHE_MB");
        return (size_t)(e ? atoll(e) : 16384) << 20;
    }();
    return cap;
}

// returns a cached buffer of at least `bytes` and stores its real size in *got
void *cache_take(int device, size_t bytes, size_t *got) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    int best = -1;
    for (int i = 0; i < (int)g_cache.size(); ++i) {
        const CachedBuf &c = g_cache[i];
        if (c.device == device && c.bytes >= bytes && c.bytes <= bytes + bytes / 4 + (1u << 20) &&
            (best < 0 || c.bytes < g_cache[best].bytes))
            best = i;
    }
    if (best < 0) return nullptr;
    void *p = g_cache[best].p;
    *got = g_cache[best].bytes;
    g_cache_bytes -= g_cache[best].bytes;
    g_cache.erase(g_cache.begin() + best);
    return p;
}

// frees every cached buffer of `device` (all devices if < 0); returns bytes released
size_t cache_flush(int device) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    size_t freed = 0;
    for (size_t i = 0; i < g_cache.size();) {
        if (device < 0 || g_cache[i].device == device) {
            cudaSetDevice(g_cache[i].device);
            cudaFree(g_cache[i].p);
            freed += g_cache[i].bytes;
            g_cache_bytes -= g_cache[i].bytes;
            g_cache.erase(g_cache.begin() + i);
        } else {
            ++i;
        }
    }
    cudaSetDevice(cur);
    return freed;
}

void cache_give(int device, void *p, size_t bytes) {
    if (!p) return;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        if (bytes <= cache_cap()) {
            g_cache.push_back({device, bytes, p});
            g_cache_bytes += bytes;
            // evict oldest first
            while (g_cache_bytes > cache_cap() && !g_cache.empty()) {
                cudaFree(g_cache.front().p);
                g_cache_bytes -= g_cache.front().bytes;
                g_cache.erase(g_cache.begin());
            }
            return;
        }
    }
    cudaFree(p);
}
}  // namespace

static int32_t dmalloc(sc_graph *g, void **p, size_t bytes) {
    bytes = bytes ? bytes : 16;
    static const bool poison = getenv("SC_DEBUG_POISON") != nullptr;  // read-before-write hunt
    if (poison) {
        cudaError_t e = cudaMalloc(p, bytes);
        if (e != cudaSuccess) return fail(SC_E_OOM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
        cudaMemset(*p, 0x7f, bytes);  // out-of-range indices, huge doubles
        cudaDeviceSynchronize();
        g->allocs.push_back({*p, bytes});
        g->bytes += (int64_t)bytes;
        return SC_OK;
    }
    size_t got = 0;
    if ((*p = cache_take(g->device, bytes, &got))) {
        g->allocs.push_back({*p, got});  // the real size, so the cache files it correctly
        g->bytes += (int64_t)got;
        return SC_OK;
    }
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaErrorMemoryAllocation && cache_flush(g->device)) {
        cudaGetLastError();
        e = cudaMalloc(p, bytes);
    }
    if (e != cudaSuccess)
        return fail(e == cudaErrorMemoryAllocation ? SC_E_OOM : SC_E_CUDA,
                    "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
    g->allocs.push_back({*p, bytes});
    g->bytes += (int64_t)bytes;
    return SC_OK;
}

// Renumbering (host, O(n log n) only over long rows):
//   1. long rows (kSellMax < len <= kExtreme), globally stable-sorted by decreasing length --
//      they come first so their (longer-running) slices are scheduled first, and global
//      sorting packs rows of similar length into a slice (little padding);
//   2. every window of kSigma rows: rows of length <= kSellMax in decreasing length
//      (counting sort, stable) -- keeps the columns' locality;
//   3. extreme rows (len > kExtreme) by decreasing length (stable; lengths saturate at
//      kWideKeyMax): one warp per row, so the longest in-order folds start first instead of
//      forming the tail of the wide-row kernel.
// Returns the number of rows laid out as SELL slices (groups 1 + 2).
static int64_t sell_order(const int64_t *rp, int64_t n, std::vector<int32_t> &perm) {
    perm.resize((size_t)n);
    int64_t pos = 0;
    {
        std::vector<std::pair<int64_t, int32_t>> lng;
        for (int64_t r = 0; r < n; ++r) {
            const int64_t len = rp[r + 1] - rp[r];
            if (len > kSellMax && len <= kExtreme) lng.emplace_back(-len, (int32_t)r);
        }
        std::stable_sort(lng.begin(), lng.end(),
                         [](const std::pair<int64_t, int32_t> &a,
                            const std::pair<int64_t, int32_t> &b) { return a.first < b.first; });
        for (auto &pr : lng) perm[(size_t)pos++] = pr.second;
    }
    std::vector<int32_t> cnt(kSellMax + 2);
    // Sorting window: kSigma rows keeps neighbouring rows (and their columns' locality)
    // together; a heavy-tailed length distribution (max > 4x mean among SELL rows) is
    // sorted globally instead, which packs equal lengths into slices and schedules the
    // longest slices first.
    int64_t sigma = kSigma;
    {
        int64_t cnt_rows = 0, sum = 0, mx = 0;
        for (int64_t r = 0; r < n; ++r) {
            const int64_t len = rp[r + 1] - rp[r];
            if (len <= kSellMax) {
                ++cnt_rows;
                sum += len;
                mx = std::max(mx, len);
            }
        }
        if (cnt_rows && mx * cnt_rows > 4 * sum) sigma = n;
    }
    for (int64_t w0 = 0; w0 < n; w0 += sigma) {
        const int64_t w1 = std::min(n, w0 + sigma);
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t r = w0; r < w1; ++r) {
            const int64_t len = rp[r + 1] - rp[r];
            if (len <= kSellMax) cnt[kSellMax - len]++;
        }
        int32_t acc = 0;
        for (int b = 0; b <= kSellMax; ++b) {
            const int32_t c = cnt[b];
            cnt[b] = acc;
            acc += c;
        }
        for (int64_t r = w0; r < w1; ++r) {
            const int64_t len = rp[r + 1] - rp[r];
            if (len <= kSellMax) perm[(size_t)(pos + cnt[kSellMax - len]++)] = (int32_t)r;
        }
        pos += acc;
    }
    const int64_t n_sell = pos;
    std::vector<std::pair<int64_t, int32_t>> ext;
    for (int64_t r = 0; r < n; ++r) {
        const int64_t len = rp[r + 1] - rp[r];
        if (len > kExtreme) ext.emplace_back(-std::min<int64_t>(len, kWideKeyMax), (int32_t)r);
    }
    std::stable_sort(ext.begin(), ext.end(),
                     [](const std::pair<int64_t, int32_t> &a, const std::pair<int64_t, int32_t> &b) {
                         return a.first < b.first;
                     });
    for (auto &pr : ext) perm[(size_t)pos++] = pr.second;
    return n_sell;
}

static int grid_for(const sc_graph *g, int64_t n, int tpb) {
    int64_t want = (n + tpb - 1) / tpb;
    int64_t cap = (int64_t)std::max(g->sm_count, 1) * 8;
    return (int)std::max<int64_t>(1, std::min(want, cap));
}

// Builds the SELL sort keys over a BFS pre-order into keys / payload (see k_bfs_*); waits
// for the column upload (ev_join) first.
static cudaError_t reorder_bfs(sc_graph *g, cudaStream_t s, const int64_t *rp, const int32_t *col,
                               int64_t n, uint32_t *keys_out, int32_t *payload_out, bool prof) {
    const int64_t nseeds = (n + kBfsStride - 1) / kBfsStride;
    int32_t *region = nullptr, *lev = nullptr, *q0 = nullptr, *q1 = nullptr, *cnt = nullptr,
            *ord = nullptr, *iota = nullptr, *ordv = nullptr;
    uint64_t *k64 = nullptr, *k64b = nullptr;
    void *tmp = nullptr;
    cudaError_t e = cudaStreamWaitEvent(s, g->ev_join, 0);
    for (auto pp : {(void **)&region, (void **)&lev, (void **)&q0, (void **)&q1, (void **)&ord,
                    (void **)&iota, (void **)&ordv})
        if (!e) e = cudaMallocAsync(pp, (size_t)n * 4, s);
    if (!e) e = cudaMallocAsync((void **)&cnt, 16, s);
    if (!e) e = cudaMallocAsync((void **)&k64, (size_t)n * 8, s);
    if (!e) e = cudaMallocAsync((void **)&k64b, (size_t)n * 8, s);
    if (!e) {
        k_bfs_init<<<grid_for(g, n, 256), 256, 0, s>>>(n, region, lev, q0);
        e = cudaGetLastError();
    }
    int32_t ncur = (int32_t)nseeds, level = 0;
    while (!e && ncur > 0) {
        e = cudaMemsetAsync(cnt, 0, 4, s);
        if (!e) {
            k_bfs_expand<<<grid_for(g, (int64_t)ncur * 32, 256), 256, 0, s>>>(
                rp, col, region, lev, q0, ncur, q1, cnt, level);
            e = cudaGetLastError();
        }
        if (!e) e = cudaMemcpyAsync(&ncur, cnt, 4, cudaMemcpyDeviceToHost, s);
        if (!e) e = cudaStreamSynchronize(s);
        std::swap(q0, q1);
        ++level;
    }
    if (prof) fprintf(stderr, "[sc_graph_create] BFS: %lld seeds, %d levels\n",
                      (long long)nseeds, level);
    size_t tb = 0;
    int end_bit = 21;
    while ((int64_t(1) << (end_bit - 20)) <= 2 * nseeds + 1) ++end_bit;
    if (!e) {
        k_bfs_keys<<<grid_for(g, n, 256), 256, 0, s>>>(n, region, lev, nseeds, k64, iota);
        e = cudaGetLastError();
    }
    if (!e) e = cub::DeviceRadixSort::SortPairs(nullptr, tb, k64, k64b, iota, ord, n, 0, end_bit, s);
    if (!e) e = cudaMallocAsync(&tmp, tb + 16, s);
    if (!e) e = cub::DeviceRadixSort::SortPairs(tmp, tb, k64, k64b, iota, ord, n, 0, end_bit, s);
    if (!e) {
        // the SELL keys are then built over the BFS positions (the caller sorts them)
        k_sell_keys_ord<<<grid_for(g, n, 256), 256, 0, s>>>(rp, ord, n, g->bfs_sigma, g->bfs_nwin,
                                                            keys_out, payload_out);
        e = cudaGetLastError();
    }
    for (void *p_ : {(void *)region, (void *)lev, (void *)q0, (void *)q1, (void *)cnt, (void *)ord,
                     (void *)iota, (void *)ordv, (void *)k64, (void *)k64b, tmp})
        if (p_) cudaFreeAsync(p_, s);
    return e;
}

#include "sc_panel.cuh"  // (inside namespace sc)
#include "sc_window.cuh"

// col == nullptr with dcol != nullptr: the column array is already on `device` (borrowed,
// e.g. from sc_generate_sbm) and is neither copied nor freed.
static int32_t graph_init(const int64_t *row_ptr, const int32_t *col, const double *val,
                          const double *deg, int64_t n, int64_t nnz, int64_t ncols,
                          int64_t col_offset, int64_t global_row0, int rename, uint32_t cflags, int32_t device,
                          sc_graph **out, const int32_t *dcol = nullptr,
                          const double *dval = nullptr) {
    SC_REQUIRE(out, SC_E_INVALID, "out is null");
    *out = nullptr;
    const bool prof = getenv("SC_GRAPH_PROFILE") != nullptr;
    auto tp0 = std::chrono::steady_clock::now();
    auto lap = [&](const char *what) {
        if (!prof) return;
        auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "[sc_graph_create] %-22s %8.2f ms\n", what,
                std::chrono::duration<double, std::milli>(t - tp0).count());
        tp0 = t;
    };
    SC_REQUIRE(row_ptr && deg && (col || dcol || nnz == 0), SC_E_INVALID, "null CSR array");
    SC_REQUIRE(!(cflags & SC_CREATE_REORDER_BFS) || rename, SC_E_INVALID,
               "the BFS pre-order applies to whole graphs (shards keep the plan's order)");
    SC_REQUIRE(n >= 1 && n < (int64_t(1) << 31) - 1, SC_E_INVALID, "n=%lld out of range",
               (long long)n);
    SC_REQUIRE(nnz >= 0 && row_ptr[0] == 0 && row_ptr[n] == nnz, SC_E_RANGE,
               "row_ptr[0] must be 0 and row_ptr[n] must equal nnz=%lld", (long long)nnz);
    SC_REQUIRE(ncols >= n && ncols < (int64_t(1) << 32) - 1 && col_offset >= 0 &&
                   col_offset + n <= ncols,
               SC_E_RANGE, "bad z-space geometry ncols=%lld col_offset=%lld", (long long)ncols,
               (long long)col_offset);
    // large inputs are validated on the device (k_validate_rows for the row offsets and
    // degrees, k_col_range for the columns, overlapped with their copy); small ones here
    if (n < (int64_t(1) << 16)) {
        for (int64_t i = 0; i < n; ++i)
            SC_REQUIRE(row_ptr[i + 1] >= row_ptr[i], SC_E_RANGE, "row_ptr decreases at %lld",
                       (long long)i);
        for (int64_t i = 0; i < n; ++i)
            SC_REQUIRE(deg[i] > 0.0 && deg[i] < 1e308, SC_E_RANGE,
                       "degree of row %lld is not positive/finite", (long long)i);
    }
    if (col && nnz < (int64_t(1) << 20))
        for (int64_t j = 0; j < nnz; ++j)
            SC_REQUIRE(col[j] >= 0 && col[j] < ncols, SC_E_RANGE,
                       "col_indices[%lld]=%d out of range", (long long)j, col[j]);
    lap("host validation");
    int ndev = 0;
    SC_CUDA(cudaGetDeviceCount(&ndev));
    SC_REQUIRE(device >= 0 && device < ndev, SC_E_INVALID, "device %d not present (%d GPUs)",
               device, ndev);
    SC_CUDA(cudaSetDevice(device));

    sc_graph *g = new sc_graph();
    g->device = device;
    g->n = n;
    g->nnz = nnz;
    g->ncols = ncols;
    g->col_offset = col_offset;
    g->global_row0 = global_row0;
    cudaDeviceGetAttribute(&g->sm_count, cudaDevAttrMultiProcessorCount, device);
    {
        int l2 = 0;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
        g->l2_bytes = l2;
    }
    bool unit = (val == nullptr && dval == nullptr);
    if (val) {
        unit = true;
        for (int64_t j = 0; j < nnz && unit; ++j) unit = (val[j] == 1.0);
        if (cflags & SC_CREATE_KEEP_WEIGHTS) unit = false;
    }
    g->unit = unit;
    g->f32 = !unit && (cflags & SC_CREATE_FP32_VALUES);

    lap("unit check");
    int32_t st;
    // (worker thread of the staged column upload below; joined before any exit)
    struct Joiner {
        std::thread t;
        ~Joiner() {
            if (t.joinable()) t.join();
        }
    } col_up;
    cudaError_t col_up_err = cudaSuccess;
    auto join_up = [&]() {
        if (col_up.t.joinable()) col_up.t.join();
    };
    auto cleanup = [&](int32_t code) {
        join_up();
        sc_graph_destroy(g);
        return code;
    };
    {
        cudaMemPool_t pool;  // keep freed graph memory in the pool for the next graph
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&g->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&g->ev0) != cudaSuccess || cudaEventCreate(&g->ev1) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev_join, cudaEventDisableTiming) != cudaSuccess) {
        fail(SC_E_CUDA, "stream/event creation failed");
        return cleanup(SC_E_CUDA);
    }
    cudaStream_t s = g->stream, s2 = g->side;
    // staging: the original CSR on the device, freed once the SELL layout is built.  The
    // column / weight copies run on the side stream while the main stream validates the rows
    // and builds the renumbering from the row offsets (all on the device).
    int64_t *t_rp = nullptr, *t_sizes = nullptr, *t_stats = nullptr, *t_wlen = nullptr;
    int32_t *t_col = nullptr, *t_flag = nullptr;
    uint32_t *t_keys = nullptr, *t_keys2 = nullptr;
    int32_t *t_iota = nullptr;
    double *t_val = nullptr, *t_deg = nullptr;
    void *t_cub = nullptr;
    size_t cub_cap = 0;
    // pageable column / weight arrays are staged through pinned slots by host threads
    // (sc_hostcopy.cuh); that upload is host-bound, so it runs on a worker thread beside the
    // row validation and renumbering below, and is joined before the columns are used
    auto free_tmp = [&]() {
        join_up();
        for (void *p_ : {(void *)t_rp, (void *)t_sizes, (void *)t_stats, (void *)t_wlen,
                         (void *)t_flag, (void *)t_keys, (void *)t_keys2, (void *)t_iota,
                         (void *)t_deg, t_cub})
            if (p_) cudaFreeAsync(p_, s);
        if (t_col && !dcol) cudaFreeAsync(t_col, s);
        if (t_val && !dval) cudaFreeAsync(t_val, s);
    };
    auto need_cub = [&](size_t bytes) -> cudaError_t {
        if (bytes <= cub_cap) return cudaSuccess;
        if (t_cub) cudaFreeAsync(t_cub, s);
        cub_cap = bytes;
        return cudaMallocAsync(&t_cub, bytes, s);
    };
    auto bail = [&](cudaError_t err, const char *what) {
        join_up();
        cudaStreamSynchronize(s2);
        free_tmp();
        fail(err == cudaErrorMemoryAllocation ? SC_E_OOM : SC_E_CUDA, "%s: %s", what,
             cudaGetErrorString(err));
        return cleanup(err == cudaErrorMemoryAllocation ? SC_E_OOM : SC_E_CUDA);
    };
    cudaError_t e = cudaSuccess;
    if (dcol) t_col = const_cast<int32_t *>(dcol);
    else e = cudaMallocAsync((void **)&t_col, (size_t)std::max<int64_t>(nnz, 1) * 4, s);
    if (dval) t_val = const_cast<double *>(dval);
    else if (!e && !unit) e = cudaMallocAsync((void **)&t_val, (size_t)std::max<int64_t>(nnz, 1) * 8, s);
    if (!e) e = cudaMallocAsync((void **)&t_rp, (size_t)(n + 1) * 8, s);
    if (!e) e = cudaMallocAsync((void **)&t_deg, (size_t)n * 8, s);
    if (!e) e = cudaMallocAsync((void **)&t_flag, 64, s);
    if (!e) e = cudaMallocAsync((void **)&t_stats, 64, s);
    // row offsets and degrees first (they gate the renumbering), then the big arrays
    if (!e) e = h2d_upload(t_rp, row_ptr, (size_t)(n + 1) * 8, s);
    if (!e) e = h2d_upload(t_deg, deg, (size_t)n * 8, s);
    if (!e) e = cudaMemsetAsync(t_flag, 0, 64, s);
    if (!e) e = cudaEventRecord(g->ev_fork, s);  // allocations done -> side stream may copy
    if (!e) e = cudaStreamWaitEvent(s2, g->ev_fork, 0);
    auto upload_cols = [&, t_col, t_val]() -> cudaError_t {
        cudaError_t r = cudaSetDevice(device);
        if (!r && nnz && !dcol) r = h2d_upload(t_col, col, (size_t)nnz * 4, s2);
        if (!r && t_val && !dval) r = h2d_upload(t_val, val, (size_t)nnz * 8, s2);
        if (!r && nnz) {
            // flag[0]: any column index out of range (side stream, right after the copy)
            k_col_range<<<grid_for(g, nnz, 256), 256, 0, s2>>>(t_col, nnz, ncols, t_flag);
            r = cudaGetLastError();
        }
        if (!r) r = cudaEventRecord(g->ev_join, s2);
        return r;
    };
    if (!e) {
        const bool host_bound = (nnz && !dcol && h2d_staged(col, (size_t)nnz * 4)) ||
                                (t_val && !dval && h2d_staged(val, (size_t)nnz * 8));
        if (host_bound) col_up.t = std::thread([&, upload_cols]() { col_up_err = upload_cols(); });
        else e = upload_cols();
    }
    if (!e) e = cudaMemsetAsync(t_stats, 0, 64, s);
    if (!e) {
        k_validate_rows<<<grid_for(g, n, 256), 256, 0, s>>>(t_rp, t_deg, n, t_flag, t_stats);
        k_finish_stats<<<1, 1, 0, s>>>(t_stats, n);
        e = cudaGetLastError();
    }
    int64_t hst[8] = {0};
    int32_t hfl[4] = {0};
    if (!e) e = cudaMemcpyAsync(hst, t_stats, 64, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaMemcpyAsync(hfl, t_flag, 16, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) return bail(e, "graph upload");
    lap("H2D + row validation");
    if (hst[2] < n) {  // hst[2] = first row whose offsets decrease (n if none)
        cudaStreamSynchronize(s2);
        free_tmp();
        fail(SC_E_RANGE, "row_ptr decreases at %lld", (long long)hst[2]);
        return cleanup(SC_E_RANGE);
    }
    if (hst[3] < n) {  // first row with a non-positive / non-finite degree
        cudaStreamSynchronize(s2);
        free_tmp();
        fail(SC_E_RANGE, "degree of row %lld is not positive/finite", (long long)hst[3]);
        return cleanup(SC_E_RANGE);
    }
    // the SELL renumbering (see sell_order): windows of kSigma rows, or one global window
    // for heavy-tailed lengths (max > 4 x mean among rows <= kSellMax), rows sorted by
    // decreasing length inside a window (stable), wide rows last in their original order
    const int64_t cnt_rows = hst[0], sum_len = hst[1], max_len = hst[4];
    const int64_t sigma = (cnt_rows && max_len * cnt_rows > 4 * sum_len) ? n : kSigma;
    g->n_sell = cnt_rows;
    g->n_wide = n - g->n_sell;
    g->nslices = (g->n_sell + kSlice - 1) / kSlice;
    const int64_t nwin = (n + sigma - 1) / sigma;
    g->bfs_sigma = sigma;
    g->bfs_nwin = nwin;

    int end_bit = 1;
    while ((int64_t(1) << end_bit) <= nwin * 512 + kWideKeyMax) ++end_bit;
    if (!e) e = cudaMallocAsync((void **)&t_keys, (size_t)n * 4, s);
    if (!e) e = cudaMallocAsync((void **)&t_keys2, (size_t)n * 4, s);
    if (!e) e = cudaMallocAsync((void **)&t_iota, (size_t)n * 4, s);
    if (!e) e = cudaMallocAsync((void **)&t_sizes, (size_t)(g->nslices + 1) * 8, s);
    if (!e) e = cudaMallocAsync((void **)&t_wlen, (size_t)(g->n_wide + 1) * 8, s);
    if (e) return bail(e, "staging allocation");
    if ((st = dmalloc(g, (void **)&g->d_perm, (size_t)n * 4)) ||
        (st = dmalloc(g, (void **)&g->d_iperm, (size_t)n * 4)) ||
        (st = dmalloc(g, (void **)&g->d_slice_ptr, (size_t)(g->nslices + 1) * 8)) ||
        (st = dmalloc(g, (void **)&g->d_wide_ptr, (size_t)(g->n_wide + 1) * 8)) ||
        (st = dmalloc(g, (void **)&g->d_deg, (size_t)n * 8)) ||
        (st = dmalloc(g, (void **)&g->d_x0, (size_t)n * 8)) ||
        (st = dmalloc(g, (void **)&g->d_x[0], (size_t)n * 8)) ||
        (st = dmalloc(g, (void **)&g->d_x[1], (size_t)n * 8)) ||
        (st = dmalloc(g, (void **)&g->d_tmp, (size_t)n * 8)) ||
        (st = dmalloc(g, (void **)&g->d_f_orig, (size_t)n * 8))) {
        cudaStreamSynchronize(s2);
        free_tmp();
        return cleanup(st);
    }
    // both z buffers in one allocation so one L2 access-policy window covers them
    double *zz = nullptr;
    // z[1] 256-byte aligned (bulk copies of panels need 16-byte alignment), a zero slot
    // z[ncols] in both buffers (padding target of the panel layout; never written, also not
    // by peers), and 64 bytes of slack after z[1] (the last panel copy is rounded up to 16)
    g->zstride = (ncols + 32) & ~(int64_t)31;
    if ((st = dmalloc(g, (void **)&zz, (size_t)g->zstride * 16 + 64))) {
        cudaStreamSynchronize(s2);
        free_tmp();
        return cleanup(st);
    }
    g->d_z[0] = zz;
    g->d_z[1] = zz + g->zstride;
    e = cudaMemsetAsync(zz, 0, (size_t)g->zstride * 16 + 64, s);
    size_t cb = 0, cb2 = 0;
    // (a heavy-tailed graph is sorted by length globally, which would undo any pre-order)
    if (!e && (cflags & SC_CREATE_REORDER_BFS) && sigma < n) {
        // locality pre-order from a multi-source BFS (needs the columns on the device)
        join_up();
        if (!e) e = col_up_err;
        if (!e) e = reorder_bfs(g, s, t_rp, t_col, n, t_keys, t_iota, prof);
        lap("BFS pre-order");
    } else if (!e) {
        k_sell_keys<<<grid_for(g, n, 256), 256, 0, s>>>(t_rp, n, sigma, nwin, t_keys, t_iota);
        e = cudaGetLastError();
    }
    if (!e) e = cub::DeviceRadixSort::SortPairs(nullptr, cb, t_keys, t_keys2, t_iota, g->d_perm,
                                                n, 0, end_bit, s);
    if (!e) e = cub::DeviceScan::ExclusiveSum(nullptr, cb2, t_sizes, g->d_slice_ptr,
                                              g->nslices + 1, s);
    if (!e) e = need_cub(std::max(std::max(cb, cb2), (size_t)16));
    if (!e) e = cub::DeviceRadixSort::SortPairs(t_cub, cb, t_keys, t_keys2, t_iota, g->d_perm,
                                                n, 0, end_bit, s);
    if (!e) {
        k_inverse_perm<<<grid_for(g, n, 256), 256, 0, s>>>(g->d_perm, g->d_iperm, n);
        k_gather_perm<<<grid_for(g, n, 256), 256, 0, s>>>(t_deg, g->d_perm, g->d_deg, n);
        if (g->nslices)
            k_slice_sizes<<<grid_for(g, g->nslices, 256), 256, 0, s>>>(t_rp, g->d_perm, g->n_sell,
                                                                       g->nslices, t_sizes);
        k_wide_lens<<<grid_for(g, g->n_wide + 1, 256), 256, 0, s>>>(t_rp, g->d_perm + g->n_sell,
                                                                    g->n_wide, t_wlen);
        e = cudaGetLastError();
    }
    if (!e) e = cudaMemsetAsync(t_sizes + g->nslices, 0, 8, s);
    if (!e) e = cub::DeviceScan::ExclusiveSum(t_cub, cb2, t_sizes, g->d_slice_ptr,
                                              g->nslices + 1, s);
    size_t cb3 = 0;
    if (!e) e = cub::DeviceScan::ExclusiveSum(nullptr, cb3, t_wlen, g->d_wide_ptr, g->n_wide + 1, s);
    if (!e) e = need_cub(cb3);
    if (!e) e = cub::DeviceScan::ExclusiveSum(t_cub, cb3, t_wlen, g->d_wide_ptr, g->n_wide + 1, s);
    int64_t wide_total = 0;
    if (!e) e = cudaMemcpyAsync(&g->sell_entries, g->d_slice_ptr + g->nslices, 8,
                                cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaMemcpyAsync(&wide_total, g->d_wide_ptr + g->n_wide, 8, cudaMemcpyDeviceToHost, s);
    join_up();
    if (!e) e = col_up_err;
    if (!e) e = cudaStreamWaitEvent(s, g->ev_join, 0);  // columns copied and range-checked
    int32_t col_bad = 0;
    if (!e) e = cudaMemcpyAsync(&col_bad, t_flag, 4, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    lap("renumbering + slices");
    if (e) return bail(e, "graph layout");
    if (col_bad) {
        free_tmp();
        fail(SC_E_RANGE, "col_indices out of range [0, %lld)", (long long)ncols);
        for (int64_t j = 0; col && j < nnz; ++j)  // locate the culprit for the message
            if (col[j] < 0 || col[j] >= ncols) {
                fail(SC_E_RANGE, "col_indices[%lld]=%d out of range", (long long)j, col[j]);
                break;
            }
        return cleanup(SC_E_RANGE);
    }
    g->wide_entries = wide_total;
    if ((st = dmalloc(g, (void **)&g->d_col, (size_t)g->sell_entries * 4 + 16)) ||
        (!unit && !g->f32 &&
         (st = dmalloc(g, (void **)&g->d_val, (size_t)g->sell_entries * 8 + 16))) ||
        (g->f32 && (st = dmalloc(g, (void **)&g->d_val32, (size_t)g->sell_entries * 4 + 16))) ||
        (st = dmalloc(g, (void **)&g->d_wcol, (size_t)wide_total * 4 + 16)) ||
        (!unit && !g->f32 &&
         (st = dmalloc(g, (void **)&g->d_wval, (size_t)wide_total * 8 + 16))) ||
        (g->f32 && (st = dmalloc(g, (void **)&g->d_wval32, (size_t)wide_total * 4 + 16)))) {
        free_tmp();
        return cleanup(st);
    }
    if (g->n_sell)
        k_fill_sell<<<grid_for(g, g->nslices * kSlice, 256), 256, 0, s>>>(
            t_rp, t_col, t_val, g->d_perm, g->d_iperm, g->d_slice_ptr, g->n_sell, g->nslices,
            col_offset, n, rename, g->d_col, g->d_val, g->d_val32);
    if (g->n_wide)
        k_fill_wide<<<(unsigned)g->n_wide, 256, 0, s>>>(t_rp, t_col, t_val, g->d_perm, g->d_iperm,
                                                        g->d_wide_ptr, g->n_sell, g->n_wide,
                                                        col_offset, n, rename, g->d_wcol, g->d_wval,
                                                        g->d_wval32);
    e = cudaGetLastError();
    if (!e) e = cudaStreamSynchronize(s);
    free_tmp();
    lap("SELL fill + free");
    if (e) {
        fail(SC_E_CUDA, "graph layout: %s", cudaGetErrorString(e));
        return cleanup(SC_E_CUDA);
    }
    if ((cflags & SC_CREATE_PANELS) && rename) {
        if ((st = build_panels(g, prof))) return cleanup(st);
        lap("panel layout");
    }
    if ((cflags & SC_CREATE_WINDOWS) && !g->pan_ctas) {
        if ((st = build_windows(g, prof))) return cleanup(st);
        lap("window layout");
    }
    *out = g;
    return SC_OK;
}

static int32_t ensure_isd(sc_graph *g, cudaStream_t s) {
    if (g->d_isd) return SC_OK;
    int32_t st = dmalloc(g, (void **)&g->d_isd, (size_t)g->n * 8);
    if (st) return st;
    k_inv_sqrt<<<grid_for(g, g->n, 256), 256, 0, s>>>(g->d_deg, g->d_isd, g->n);
    SC_CUDA(cudaGetLastError());
    return SC_OK;
}

template <bool BIGZ>
static void launch_slices_t(const sc_graph *g, const StepArgs &a, bool sym, dim3 grid, cudaStream_t s) {
    if (g->unit) {
        if (sym) k_rw_step<true, true, false, BIGZ><<<grid, kStepTPB, 0, s>>>(a);
        else k_rw_step<true, false, false, BIGZ><<<grid, kStepTPB, 0, s>>>(a);
    } else if (g->f32) {
        if (sym) k_rw_step<false, true, true, BIGZ><<<grid, kStepTPB, 0, s>>>(a);
        else k_rw_step<false, false, true, BIGZ><<<grid, kStepTPB, 0, s>>>(a);
    } else {
        if (sym) k_rw_step<false, true, false, BIGZ><<<grid, kStepTPB, 0, s>>>(a);
        else k_rw_step<false, false, false, BIGZ><<<grid, kStepTPB, 0, s>>>(a);
    }
}
// the slice kernel with the 64-byte L2 fetch hint on its gathers when z does not fit the L2
static void launch_slices(const sc_graph *g, const StepArgs &a, bool sym, dim3 grid, cudaStream_t s) {
    if (a.zhint) launch_slices_t<true>(g, a, sym, grid, s);
    else launch_slices_t<false>(g, a, sym, grid, s);
}

// rows [row_lo, row_hi) of the renumbered shard; SELL boundaries must be slice-aligned
static int32_t launch_step(const sc_graph *g, const double *z_in, const double *x_in,
                           double *x_out, double *z_out, double sign, uint32_t flags,
                           cudaStream_t s, int64_t row_lo = 0, int64_t row_hi = -1) {
    const bool sym = flags & SC_SYM_VARIANT;
    if (row_hi < 0) row_hi = g->n;
    // whole-graph steps use the column-panel layout when the handle has one
    const bool panel = g->pan_ctas && !(flags & SC_FORCE_SELL) && row_lo == 0 && row_hi == g->n &&
                       (g->npeer == 0 || g->peer_events);
    // ... or the row-window layout (z_in must allow 16-byte aligned bulk copies)
    const bool window = !panel && g->win_items && !(flags & SC_FORCE_SELL) && row_lo == 0 &&
                        row_hi == g->n && ((uintptr_t)z_in & 15) == 0;
    StepArgs a;
    a.slice_lo = std::min(row_lo, g->n_sell) / kSlice;
    a.slice_hi = (std::min(row_hi, g->n_sell) + kSlice - 1) / kSlice;
    if (a.slice_hi < a.slice_lo) a.slice_hi = a.slice_lo;
    a.wide_lo = std::max<int64_t>(row_lo - g->n_sell, 0);
    a.wide_hi = std::max<int64_t>(row_hi - g->n_sell, 0);
    a.slice_ptr = g->d_slice_ptr;
    a.col = g->d_col;
    a.val = g->d_val;
    a.wide_ptr = g->d_wide_ptr;
    a.wcol = g->d_wcol;
    a.wval = g->d_wval;
    a.val32 = g->d_val32;
    a.wval32 = g->d_wval32;
    a.scale = sym ? g->d_isd : g->d_deg;
    a.x_in = x_in;
    a.z_in = z_in;
    a.x_out = x_out;
    a.z_out = z_out;
    a.n_sell = g->n_sell;
    a.n_wide = g->n_wide;
    a.nslices = g->nslices;
    a.col_offset = g->col_offset;
    a.hs = sign < 0 ? -0.5 : 0.5;
    // (SC_ZHINT=1 / 0 forces the 64-byte fetch hint on / off: tests run the hinted kernels on
    // small graphs)
    static const int zhint_env = [] {
        const char *e = getenv("SC_ZHINT");
        return e ? atoi(e) : -1;
    }();
    a.zhint = zhint_env >= 0 ? (zhint_env != 0) : (g->l2_bytes > 0 && g->ncols * 8 > g->l2_bytes);
    a.peer_base = g->d_peer_z;
    a.npeer = 0;
    a.peer_off = 0;
    if (g->npeer) {
        // the exchange mirrors the handle's own z allocation only
        SC_REQUIRE(z_out >= g->d_z[0] && z_out < g->d_z[0] + g->zstride + g->ncols, SC_E_STATE,
                   "peer exchange needs z_out inside the handle's z buffers (sc_shard_buffers)");
        a.npeer = g->npeer;
        a.peer_off = z_out - g->d_z[0];
    }
    if (panel) {
        SC_CUDA(launch_panel_step(g, a, sym, s));
        return SC_OK;
    }
    constexpr int wpb = kStepTPB / 32;
    a.wide_blocks = (int)((a.wide_hi - a.wide_lo + wpb - 1) / wpb);
    const int64_t sblocks = (a.slice_hi - a.slice_lo + wpb - 1) / wpb;
    // wide rows run concurrently on the side stream (fork / join through events, which a
    // CUDA-graph capture records as parallel branches)
    if (a.wide_blocks) {
        SC_CUDA(cudaEventRecord(g->ev_fork, s));
        SC_CUDA(cudaStreamWaitEvent(g->side, g->ev_fork, 0));
        // at most kWideCtasPerSM CTAs per SM (SC_WIDE_CAP overrides; 0 = one CTA per 8 rows)
        static const int wide_env = [] {
            const char *e = getenv("SC_WIDE_CAP");
            return e ? atoi(e) : -1;
        }();
        // (steps enqueued on a caller's stream -- the torchrun shard path -- keep the uncapped
        // grid: there the two kernels do not overlap and the cap only stretches the wide rows,
        // 293 -> 377 us per step at C3)
        const int wide_cap = wide_env >= 0 ? wide_env
                             : s != g->stream ? 0
                             : g->wide_entries * 4 >= g->nnz ? 2 * kWideCtasPerSM : kWideCtasPerSM;
        const int wide_grid = wide_cap > 0 ? std::min(a.wide_blocks, wide_cap * std::max(g->sm_count, 1))
                                           : a.wide_blocks;
        const dim3 wg((unsigned)wide_grid);
        if (g->unit) {
            if (sym) k_rw_wide<true, true><<<wg, kStepTPB, 0, g->side>>>(a);
            else k_rw_wide<true, false><<<wg, kStepTPB, 0, g->side>>>(a);
        } else if (g->f32) {
            if (sym) k_rw_wide<false, true, true><<<wg, kStepTPB, 0, g->side>>>(a);
            else k_rw_wide<false, false, true><<<wg, kStepTPB, 0, g->side>>>(a);
        } else {
            if (sym) k_rw_wide<false, true><<<wg, kStepTPB, 0, g->side>>>(a);
            else k_rw_wide<false, false><<<wg, kStepTPB, 0, g->side>>>(a);
        }
    }
    if (sblocks && window) {
        SC_CUDA(launch_window_step(g, a, sym, s));
    } else if (sblocks) {
        const dim3 grid((unsigned)sblocks);
        launch_slices(g, a, sym, grid, s);
    }
    if (a.wide_blocks) {
        SC_CUDA(cudaEventRecord(g->ev_join, g->side));
        SC_CUDA(cudaStreamWaitEvent(s, g->ev_join, 0));
    }
    SC_CUDA(cudaGetLastError());
    return SC_OK;
}

static int32_t enqueue_power(sc_graph *g, int32_t T, double sign, uint32_t flags) {
    const bool sym = flags & SC_SYM_VARIANT;
    cudaStream_t s = g->stream;
    k_scale<<<grid_for(g, g->n, 256), 256, 0, s>>>(g->d_x0, sym ? g->d_isd : g->d_deg,
                                                   g->d_z[0], g->n, g->col_offset, sym);
    SC_CUDA(cudaGetLastError());
    for (int32_t t = 0; t < T; ++t) {
        const int in = t & 1, out = in ^ 1;
        int32_t st = launch_step(g, g->d_z[in], t == 0 ? g->d_x0 : g->d_x[in], g->d_x[out],
                                 g->d_z[out], sign, flags, s);
        if (st) return st;
    }
    return SC_OK;
}

static void set_l2_window(sc_graph *g, bool on) {
    if (on == g->l2_window) return;
    cudaStreamAttrValue attr;
    std::memset(&attr, 0, sizeof attr);
    if (on) {
        int maxwin = 0, maxpersist = 0;
        cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, g->device);
        cudaDeviceGetAttribute(&maxpersist, cudaDevAttrMaxPersistingL2CacheSize, g->device);
        size_t bytes = (size_t)g->zstride * 16;
        size_t win = std::min<size_t>(bytes, (size_t)maxwin);
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(win, maxpersist));
        attr.accessPolicyWindow.base_ptr = g->d_z[0];
        attr.accessPolicyWindow.num_bytes = win;
        attr.accessPolicyWindow.hitRatio =
            win ? std::min(1.0f, (float)maxpersist / (float)win) : 0.f;
        attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    } else {
        attr.accessPolicyWindow.num_bytes = 0;
        cudaCtxResetPersistingL2Cache();
    }
    cudaStreamSetAttribute(g->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
    g->l2_window = on;
}

// device vector (renumbered order) -> host vector (original order)
static int32_t to_host_original(sc_graph *g, const double *dev, double *host) {
    k_gather_perm<<<grid_for(g, g->n, 256), 256, 0, g->stream>>>(dev, g->d_iperm, g->d_tmp, g->n);
    SC_CUDA(cudaGetLastError());
    SC_CUDA(cudaMemcpyAsync(host, g->d_tmp, (size_t)g->n * 8, cudaMemcpyDeviceToHost, g->stream));
    SC_CUDA(cudaStreamSynchronize(g->stream));
    return SC_OK;
}

int32_t csr_device_arrays(const sc_csr *h, const int64_t **rp, const int32_t **col,
                          const double **deg, const double **val, int32_t *device);  // sc_generate.cu

}  // namespace sc

// halo pack: dst[i] = src[idx[i]]
__global__ void k_gather_f64(const double *__restrict__ src, const int32_t *__restrict__ idx,
                             int64_t count, double *__restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[__ldg(idx + i)];
}

extern "C" {

int32_t sc_version(void) { return 2; }

const char *sc_last_error(void) { return sc::g_last_error.c_str(); }

int32_t sc_device_count(void) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        sc::set_error("cudaGetDeviceCount: %s", cudaGetErrorString(e));
        return 0;
    }
    return n;
}

int32_t sc_graph_create(const int64_t *row_ptr, const int32_t *col, const double *val,
                        const double *deg, int64_t n, int64_t nnz, int32_t device,
                        sc_graph **out) {
    return graph_init(row_ptr, col, val, deg, n, nnz, n, 0, 0, 1, 0u, device, out);
}

int32_t sc_graph_create_ex(const int64_t *row_ptr, const int32_t *col, const double *val,
                           const double *deg, int64_t n, int64_t nnz, int32_t device,
                           uint32_t create_flags, sc_graph **out) {
    SC_REQUIRE(!(create_flags & SC_CREATE_KEEP_WEIGHTS) || val || nnz == 0, SC_E_INVALID,
               "SC_CREATE_KEEP_WEIGHTS needs a weight array");
    return graph_init(row_ptr, col, val, deg, n, nnz, n, 0, 0, 1, create_flags, device, out);
}

int32_t sc_shard_create(const int64_t *row_ptr, const int32_t *col, const double *val,
                        const double *deg, int64_t n, int64_t nnz, int64_t ncols,
                        int64_t col_offset, int64_t global_row0, int32_t device,
                        sc_graph **out) {
    // columns arrive already renamed into the global renumbered z space (sc_sell_order)
    return graph_init(row_ptr, col, val, deg, n, nnz, ncols, col_offset, global_row0, 0, 0u, device,
                      out);
}

int32_t sc_graph_create_from_csr(const sc_csr *h, uint32_t create_flags, sc_graph **out) {
    SC_REQUIRE(h && out, SC_E_INVALID, "null argument");
    int64_t n = 0, nnz = 0;
    int32_t st = sc_csr_info(h, &n, &nnz, nullptr);
    if (st) return st;
    const int64_t *d_rp;
    const int32_t *d_col;
    const double *d_deg, *d_val;
    int32_t device;
    if ((st = sc::csr_device_arrays(h, &d_rp, &d_col, &d_deg, &d_val, &device))) return st;
    SC_CUDA(cudaSetDevice(device));
    // the renumbering is computed on the host from the row offsets (n + 1 words); the
    // column array stays on the device
    std::vector<int64_t> rp((size_t)n + 1);
    std::vector<double> deg((size_t)n);
    SC_CUDA(cudaMemcpy(rp.data(), d_rp, (size_t)(n + 1) * 8, cudaMemcpyDeviceToHost));
    SC_CUDA(cudaMemcpy(deg.data(), d_deg, (size_t)n * 8, cudaMemcpyDeviceToHost));
    return graph_init(rp.data(), nullptr, nullptr, deg.data(), n, nnz, n, 0, 0, 1, create_flags,
                      device, out, d_col, d_val);
}

int32_t sc_shard_create_from_csr(const sc_csr *h, int64_t row_lo, int64_t row_hi,
                                 const int32_t *d_slot_of, int64_t ncols, int64_t col_offset,
                                 sc_graph **out) {
    SC_REQUIRE(h && d_slot_of && out, SC_E_INVALID, "null argument");
    int64_t n = 0, nnz = 0;
    int32_t st = sc_csr_info(h, &n, &nnz, nullptr);
    if (st) return st;
    SC_REQUIRE(0 <= row_lo && row_lo < row_hi && row_hi <= n, SC_E_RANGE,
               "row range [%lld, %lld) outside [0, %lld)", (long long)row_lo, (long long)row_hi,
               (long long)n);
    const int64_t *d_rp;
    const int32_t *d_col;
    const double *d_deg, *d_val;
    int32_t device;
    if ((st = sc::csr_device_arrays(h, &d_rp, &d_col, &d_deg, &d_val, &device))) return st;
    SC_CUDA(cudaSetDevice(device));
    const int64_t nl = row_hi - row_lo;
    std::vector<int64_t> rp((size_t)nl + 1);
    std::vector<double> deg((size_t)nl);
    SC_CUDA(cudaMemcpy(rp.data(), d_rp + row_lo, (size_t)(nl + 1) * 8, cudaMemcpyDeviceToHost));
    SC_CUDA(cudaMemcpy(deg.data(), d_deg + row_lo, (size_t)nl * 8, cudaMemcpyDeviceToHost));
    const int64_t e0 = rp[0];
    for (auto &v : rp) v -= e0;
    const int64_t nnzl = rp[(size_t)nl];
    // the block's columns renamed into the z space on the device (range-checked there)
    int32_t *d_ren = nullptr;
    int32_t *d_bad = nullptr;
    SC_CUDA(cudaMalloc((void **)&d_ren, (size_t)std::max<int64_t>(nnzl, 1) * 4));
    cudaError_t e = cudaMalloc((void **)&d_bad, 4);
    if (!e) e = cudaMemset(d_bad, 0, 4);
    if (!e && nnzl) {
        sc::k_rename_cols<<<(unsigned)std::min<int64_t>((nnzl + 255) / 256, 148 * 16), 256>>>(
            d_col + e0, nnzl, d_slot_of, n, d_ren, d_bad);
        e = cudaGetLastError();
    }
    int32_t bad = 0;
    if (!e) e = cudaMemcpy(&bad, d_bad, 4, cudaMemcpyDeviceToHost);
    cudaFree(d_bad);
    if (e) {
        cudaFree(d_ren);
        return fail(SC_E_CUDA, "shard column renaming: %s", cudaGetErrorString(e));
    }
    if (bad) {
        cudaFree(d_ren);
        return fail(SC_E_RANGE, "a column index is outside [0, %lld)", (long long)n);
    }
    st = graph_init(rp.data(), nullptr, nullptr, deg.data(), nl, nnzl, ncols, col_offset, row_lo, 0,
                    0u, device, out, d_ren, d_val ? d_val + e0 : nullptr);
    cudaDeviceSynchronize();
    cudaFree(d_ren);
    return st;
}

int64_t sc_release_cached_memory(int32_t device) {
    // device < 0: every device
    return (int64_t)sc::cache_flush(device);
}

int32_t sc_sell_order(const int64_t *row_ptr, int64_t n, int32_t *perm_out) {
    SC_REQUIRE(row_ptr && perm_out && n >= 1, SC_E_INVALID, "null argument");
    std::vector<int32_t> perm;
    sell_order(row_ptr, n, perm);
    std::memcpy(perm_out, perm.data(), (size_t)n * 4);
    return SC_OK;
}

void sc_graph_destroy(sc_graph *g) {
    if (!g) return;
    if (g->multi) {
        sc::multi_free(g);
        delete g;
        return;
    }
    cudaSetDevice(g->device);
    if (g->stream) cudaStreamSynchronize(g->stream);
    if (g->side) cudaStreamSynchronize(g->side);
    if (g->gexec) cudaGraphExecDestroy(g->gexec);
    // a sticky error makes the stream query fail: do not recycle buffers of a broken context
    const bool healthy = !g->stream || cudaStreamQuery(g->stream) == cudaSuccess;
    for (auto &a : g->allocs) {
        if (healthy)
            cache_give(g->device, a.first, a.second);
        else
            cudaFree(a.first);
    }
    g->allocs.clear();
    if (g->ev0) cudaEventDestroy(g->ev0);
    if (g->ev1) cudaEventDestroy(g->ev1);
    if (g->ev_fork) cudaEventDestroy(g->ev_fork);
    if (g->ev_join) cudaEventDestroy(g->ev_join);
    if (g->side) {
        cudaStreamSynchronize(g->side);
        cudaStreamDestroy(g->side);
    }
    if (g->stream) cudaStreamDestroy(g->stream);
    delete g;
}

int32_t sc_graph_download_f(sc_graph *g, double *f_out) {
    SC_REQUIRE(g && f_out, SC_E_INVALID, "null argument");
    if (g->multi) return sc::multi_download_f(g, f_out);
    SC_REQUIRE(g->result >= 0, SC_E_STATE, "no power iteration has run on this handle");
    SC_CUDA(cudaSetDevice(g->device));
    return sc::to_host_original(g, g->d_z[g->result], f_out);
}

int32_t sc_graph_build_panels(sc_graph *g) {
    SC_REQUIRE(g, SC_E_INVALID, "null graph");
    SC_NOT_MULTI(g);  // (multi-GPU handles take SC_CREATE_PANELS at creation)
    if (g->pan_ctas) return SC_OK;
    SC_CUDA(cudaSetDevice(g->device));
    return sc::build_panels(g, getenv("SC_GRAPH_PROFILE") != nullptr);
}

int32_t sc_graph_build_windows(sc_graph *g) {
    SC_REQUIRE(g, SC_E_INVALID, "null graph");
    SC_NOT_MULTI(g);
    if (g->win_items) return SC_OK;
    SC_CUDA(cudaSetDevice(g->device));
    return sc::build_windows(g, getenv("SC_GRAPH_PROFILE") != nullptr);
}

int32_t sc_graph_info_get(const sc_graph *g, sc_graph_info *o) {
    SC_REQUIRE(g && o, SC_E_INVALID, "null argument");
    if (g->multi) return sc::multi_info(g, o);
    o->n = g->n;
    o->nnz = g->nnz;
    o->ncols = g->ncols;
    o->col_offset = g->col_offset;
    o->ntiles = g->nslices;
    o->long_rows = g->n_wide;
    o->unit_weights = g->unit;
    o->rp64 = 0;
    o->device_bytes = g->bytes;
    o->device = g->device;
    o->sm_count = g->sm_count;
    o->panel_groups = g->pan_ctas ? g->pan_groups : 0;
    o->panel_bytes = g->pan_ctas ? g->pan_bytes : 0;
    o->stored_entries = g->sell_entries;
    o->zstride = g->zstride;
    o->n_gpus = 1;
    o->window_items = g->win_items;
    return SC_OK;
}

int32_t sc_graph_order(const sc_graph *g, int32_t *perm_out) {
    SC_REQUIRE(g && perm_out, SC_E_INVALID, "null argument");
    SC_NOT_MULTI(g);
    SC_CUDA(cudaSetDevice(g->device));
    SC_CUDA(cudaMemcpy(perm_out, g->d_perm, (size_t)g->n * 4, cudaMemcpyDeviceToHost));
    return SC_OK;
}

int32_t sc_sample_irwin_hall(sc_graph *g, uint64_t key0, uint64_t key1, double *x0_out) {
    SC_REQUIRE(g, SC_E_INVALID, "null graph");
    if (g->multi) return sc::multi_sample(g, key0, key1, x0_out);
    SC_CUDA(cudaSetDevice(g->device));
    k_irwin_hall<<<grid_for(g, g->n, 128), 128, 0, g->stream>>>(g->d_deg, g->d_perm, g->d_x0,
                                                                g->n, g->global_row0, key0, key1);
    SC_CUDA(cudaGetLastError());
    if (x0_out) {
        int32_t st = to_host_original(g, g->d_x0, x0_out);
        if (st) return st;
    }
    SC_CUDA(cudaStreamSynchronize(g->stream));
    g->have_x0 = true;
    g->result = -1;
    return SC_OK;
}

int32_t sc_set_x0(sc_graph *g, const double *x0_host) {
    SC_REQUIRE(g && x0_host, SC_E_INVALID, "null argument");
    if (g->multi) return sc::multi_set_x0(g, x0_host);
    SC_CUDA(cudaSetDevice(g->device));
    SC_CUDA(cudaMemcpyAsync(g->d_tmp, x0_host, (size_t)g->n * 8, cudaMemcpyHostToDevice,
                            g->stream));
    k_gather_perm<<<grid_for(g, g->n, 256), 256, 0, g->stream>>>(g->d_tmp, g->d_perm, g->d_x0,
                                                                 g->n);
    SC_CUDA(cudaGetLastError());
    SC_CUDA(cudaStreamSynchronize(g->stream));
    g->have_x0 = true;
    g->result = -1;
    return SC_OK;
}

int32_t sc_power_iterate(sc_graph *g, int32_t T, double sign, uint32_t flags, double *xT_out,
                         double *f_out, sc_timing *t_out) {
    SC_REQUIRE(g, SC_E_INVALID, "null graph");
    SC_REQUIRE(T >= 0, SC_E_INVALID, "power method step count must be >= 0, got %d", T);
    SC_REQUIRE(sign == 1.0 || sign == -1.0, SC_E_INVALID, "sign must be +1 or -1");
    if (g->multi) return sc::multi_power(g, T, sign, flags, xT_out, f_out, t_out);
    SC_REQUIRE(g->have_x0, SC_E_STATE, "no start vector: call sc_sample_irwin_hall or sc_set_x0");
    SC_REQUIRE(g->ncols == g->n, SC_E_STATE,
               "sc_power_iterate needs a whole graph; shards use sc_shard_step");
    SC_CUDA(cudaSetDevice(g->device));
    int32_t st;
    if (flags & SC_SYM_VARIANT)
        if ((st = ensure_isd(g, g->stream))) return st;
    set_l2_window(g, flags & SC_L2_PERSIST);
    const uint32_t gflags = flags & ~(uint32_t)SC_NO_CUDA_GRAPH;
    SC_CUDA(cudaEventRecord(g->ev0, g->stream));
    if (flags & SC_NO_CUDA_GRAPH) {
        if ((st = enqueue_power(g, T, sign, flags))) return st;
    } else {
        if (!g->gexec || g->g_T != T || g->g_flags != gflags || g->g_sign != sign) {
            if (g->gexec) {
                cudaGraphExecDestroy(g->gexec);
                g->gexec = nullptr;
            }
            cudaGraph_t graph = nullptr;
            SC_CUDA(cudaStreamBeginCapture(g->stream, cudaStreamCaptureModeThreadLocal));
            st = enqueue_power(g, T, sign, flags);
            cudaError_t e = cudaStreamEndCapture(g->stream, &graph);
            if (st) {
                if (graph) cudaGraphDestroy(graph);
                return st;
            }
            SC_CUDA(e);
            e = cudaGraphInstantiate(&g->gexec, graph, 0);
            cudaGraphDestroy(graph);
            SC_CUDA(e);
            g->g_T = T;
            g->g_flags = gflags;
            g->g_sign = sign;
        }
        SC_CUDA(cudaGraphLaunch(g->gexec, g->stream));
    }
    SC_CUDA(cudaEventRecord(g->ev1, g->stream));
    SC_CUDA(cudaEventSynchronize(g->ev1));
    float ms = 0.f;
    SC_CUDA(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
    g->result = T & 1;
    const double *xT = T == 0 ? g->d_x0 : g->d_x[g->result];
    const double *f = g->d_z[g->result];
    auto h0 = std::chrono::steady_clock::now();
    if (xT_out && (st = to_host_original(g, xT, xT_out))) return st;
    if (f_out && (st = to_host_original(g, f, f_out))) return st;
    auto h1 = std::chrono::steady_clock::now();
    if (t_out) {
        t_out->power_ms = ms;
        t_out->kernel_ms = T ? ms / T : 0.0;
        t_out->d2h_ms = std::chrono::duration<double, std::milli>(h1 - h0).count();
    }
    return SC_OK;
}

}  // extern "C"

namespace sc {
template <int L>
static void launch_blk(const sc_graph *g, const BlkArgs &a, cudaStream_t s) {
    constexpr int wpb = kStepTPB / 32;
    if (g->n_wide) {
        cudaEventRecord(g->ev_fork, s);
        cudaStreamWaitEvent(g->side, g->ev_fork, 0);
        const unsigned wb = (unsigned)((g->n_wide + wpb - 1) / wpb);
        if (g->unit) k_blk_wide<L, true><<<wb, kStepTPB, 0, g->side>>>(a);
        else k_blk_wide<L, false><<<wb, kStepTPB, 0, g->side>>>(a);
    }
    if (g->nslices) {
        const unsigned sb = (unsigned)((g->nslices + wpb - 1) / wpb);
        if (g->unit) k_blk_step<L, true><<<sb, kStepTPB, 0, s>>>(a);
        else k_blk_step<L, false><<<sb, kStepTPB, 0, s>>>(a);
    }
    if (g->n_wide) {
        cudaEventRecord(g->ev_join, g->side);
        cudaStreamWaitEvent(s, g->ev_join, 0);
    }
}

template <int... Ls>
struct BlkDispatch;
template <>
struct BlkDispatch<> {
    static bool run(int, const sc_graph *, const BlkArgs &, cudaStream_t) { return false; }
};
template <int L0, int... Ls>
struct BlkDispatch<L0, Ls...> {
    static bool run(int L, const sc_graph *g, const BlkArgs &a, cudaStream_t s) {
        if (L == L0) {
            launch_blk<L0>(g, a, s);
            return true;
        }
        return BlkDispatch<Ls...>::run(L, g, a, s);
    }
};
using BlkAll = BlkDispatch<4, 8, 12, 16>;  // padded widths (32-byte rows)
constexpr int kMaxBlockCols = 16;
}  // namespace sc

extern "C" {

int32_t sc_power_iterate_block(sc_graph *g, int32_t T, int32_t L, const double *x0,
                               double *raw_out, double *scaled_out, sc_timing *t_out) {
    using namespace sc;
    SC_REQUIRE(g && x0, SC_E_INVALID, "null argument");
    SC_REQUIRE(T >= 0, SC_E_INVALID, "power method step count must be >= 0, got %d", T);
    SC_REQUIRE(L >= 1 && L <= kMaxBlockCols, SC_E_INVALID, "block width %d outside [1, %d]", L,
               kMaxBlockCols);
    SC_NOT_MULTI(g);
    SC_REQUIRE(g->ncols == g->n, SC_E_STATE, "block power method needs a whole graph");
    SC_REQUIRE(!g->f32, SC_E_STATE, "block power method needs fp64 weights (no SC_CREATE_FP32_VALUES)");
    SC_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = g->stream;
    int32_t st;
    if ((st = ensure_isd(g, s))) return st;
    // columns padded to a multiple of 4 so every row is 32-byte aligned and one 256-bit
    // load fetches four of a neighbour's values; the zero padding columns stay zero
    const int LP = (L + 3) / 4 * 4;
    const int64_t n = g->n, nl = n * LP;
    double *buf = nullptr;  // x0, x[2], z[2], staging: 6 [n][LP] blocks
    SC_CUDA(cudaMallocAsync((void **)&buf, (size_t)nl * 6 * 8, s));
    double *bx0 = buf, *bx[2] = {buf + nl, buf + 2 * nl}, *bz[2] = {buf + 3 * nl, buf + 4 * nl};
    double *stage = buf + 5 * nl;
    auto done = [&](int32_t code) {
        cudaFreeAsync(buf, s);
        cudaStreamSynchronize(s);
        return code;
    };
    cudaError_t e = cudaMemcpyAsync(stage, x0, (size_t)n * L * 8, cudaMemcpyHostToDevice, s);
    if (e) return done(fail(SC_E_CUDA, "block upload: %s", cudaGetErrorString(e)));
    const int gr = grid_for(g, nl, 256);
    k_gather_rows<<<gr, 256, 0, s>>>(stage, g->d_perm, bx0, n, L, L, LP);  // original -> renumbered
    k_scale_rows<<<gr, 256, 0, s>>>(bx0, g->d_isd, bz[0], n, LP);
    cudaEventRecord(g->ev0, s);
    BlkArgs a;
    a.slice_ptr = g->d_slice_ptr;
    a.col = g->d_col;
    a.val = g->d_val;
    a.wide_ptr = g->d_wide_ptr;
    a.wcol = g->d_wcol;
    a.wval = g->d_wval;
    a.isd = g->d_isd;
    a.n_sell = g->n_sell;
    a.nslices = g->nslices;
    a.n_wide = g->n_wide;
    for (int32_t t = 0; t < T; ++t) {
        const int in = t & 1, out = in ^ 1;
        a.x_in = t == 0 ? bx0 : bx[in];
        a.z_in = bz[in];
        a.x_out = bx[out];
        a.z_out = bz[out];
        BlkAll::run(LP, g, a, s);
    }
    cudaEventRecord(g->ev1, s);
    e = cudaGetLastError();
    if (!e) e = cudaEventSynchronize(g->ev1);
    if (e) return done(fail(SC_E_CUDA, "block power method: %s", cudaGetErrorString(e)));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, g->ev0, g->ev1);
    const double *xr = T == 0 ? bx0 : bx[T & 1];
    const double *zr = bz[T & 1];  // = d^-1/2 x_T: the scaled embedding (pipeline.py:157)
    for (int pass = 0; pass < 2; ++pass) {
        double *host = pass ? scaled_out : raw_out;
        if (!host) continue;
        k_gather_rows<<<gr, 256, 0, s>>>(pass ? zr : xr, g->d_iperm, stage, n, L, LP, L);
        e = cudaMemcpyAsync(host, stage, (size_t)n * L * 8, cudaMemcpyDeviceToHost, s);
        if (!e) e = cudaStreamSynchronize(s);
        if (e) return done(fail(SC_E_CUDA, "block download: %s", cudaGetErrorString(e)));
    }
    if (t_out) {
        t_out->power_ms = ms;
        t_out->kernel_ms = T ? ms / T : 0.0;
        t_out->sample_ms = 0.0;
        t_out->d2h_ms = 0.0;
    }
    return done(SC_OK);
}

int32_t sc_shard_step(sc_graph *g, const double *z_in, const double *x_in, double *x_out,
                      double *z_out, double sign, uint32_t flags, void *stream) {
    SC_REQUIRE(g && z_in && x_in && x_out && z_out, SC_E_INVALID, "null argument");
    SC_NOT_MULTI(g);
    SC_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = (cudaStream_t)stream;  // the caller's stream, 0 = legacy default stream
    int32_t st;
    if (flags & SC_SYM_VARIANT)
        if ((st = ensure_isd(g, s))) return st;
    return launch_step(g, z_in, x_in, x_out, z_out, sign, flags, s);
}

int32_t sc_shard_step_range(sc_graph *g, int64_t row_lo, int64_t row_hi, const double *z_in,
                            const double *x_in, double *x_out, double *z_out, double sign,
                            uint32_t flags, void *stream) {
    SC_REQUIRE(g && z_in && x_in && x_out && z_out, SC_E_INVALID, "null argument");
    SC_NOT_MULTI(g);
    SC_REQUIRE(0 <= row_lo && row_lo <= row_hi && row_hi <= g->n, SC_E_RANGE,
               "row range [%lld, %lld) outside [0, %lld)", (long long)row_lo, (long long)row_hi,
               (long long)g->n);
    SC_REQUIRE((row_lo >= g->n_sell || row_lo % kSlice == 0) &&
                   (row_hi >= g->n_sell || row_hi % kSlice == 0),
               SC_E_RANGE, "row range must be slice aligned (multiples of 32) below %lld",
               (long long)g->n_sell);
    SC_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = (cudaStream_t)stream;
    int32_t st;
    if (flags & SC_SYM_VARIANT)
        if ((st = ensure_isd(g, s))) return st;
    return launch_step(g, z_in, x_in, x_out, z_out, sign, flags, s, row_lo, row_hi);
}

int32_t sc_shard_scale_range(sc_graph *g, int64_t row_lo, int64_t row_hi, const double *x,
                             double *z_out, uint32_t flags, void *stream) {
    SC_REQUIRE(g && x && z_out, SC_E_INVALID, "null argument");
    SC_REQUIRE(0 <= row_lo && row_lo <= row_hi && row_hi <= g->n, SC_E_RANGE, "bad row range");
    SC_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = (cudaStream_t)stream;
    const bool sym = flags & SC_SYM_VARIANT;
    int32_t st;
    if (sym)
        if ((st = ensure_isd(g, s))) return st;
    int64_t poff = 0;
    if (g->npeer) {
        SC_REQUIRE(z_out >= g->d_z[0] && z_out < g->d_z[0] + g->zstride + g->ncols, SC_E_STATE,
                   "peer exchange needs z_out inside the handle's z buffers (sc_shard_buffers)");
        poff = z_out - g->d_z[0];
    }
    if (row_hi > row_lo)
        k_scale<<<grid_for(g, row_hi - row_lo, 256), 256, 0, s>>>(
            x + row_lo, (sym ? g->d_isd : g->d_deg) + row_lo, z_out, row_hi - row_lo,
            g->col_offset + row_lo, sym, g->d_peer_z, poff, g->npeer);
    SC_CUDA(cudaGetLastError());
    return SC_OK;
}

int32_t sc_shard_buffers(sc_graph *g, double **z_base, uint32_t **flags) {
    SC_REQUIRE(g && z_base && flags, SC_E_INVALID, "null argument");
    SC_NOT_MULTI(g);
    SC_CUDA(cudaSetDevice(g->device));
    if (!g->d_flags) {
        int32_t st = dmalloc(g, (void **)&g->d_flags, 64 * 4);
        if (st) return st;
        SC_CUDA(cudaMemset(g->d_flags, 0, 64 * 4));
    }
    *z_base = g->d_z[0];
    *flags = g->d_flags;
    return SC_OK;
}

int32_t sc_shard_set_peers(sc_graph *g, void *const *z_bases, void *const *flag_bases,
                           int32_t world, int32_t rank) {
    SC_REQUIRE(g && z_bases && flag_bases, SC_E_INVALID, "null argument");
    SC_NOT_MULTI(g);
    SC_REQUIRE(world >= 1 && world <= kMaxWorld && rank >= 0 && rank < world, SC_E_INVALID,
               "bad world/rank (%d/%d; at most %d ranks)", world, rank, kMaxWorld);
    SC_CUDA(cudaSetDevice(g->device));
    std::vector<double *> pz;
    std::vector<uint32_t *> pf((size_t)world, nullptr);
    for (int q = 0; q < world; ++q) {
        if (q == rank) continue;
        SC_REQUIRE(z_bases[q] && flag_bases[q], SC_E_INVALID, "null peer pointer for rank %d", q);
        pz.push_back(static_cast<double *>(z_bases[q]));
        pf[(size_t)q] = static_cast<uint32_t *>(flag_bases[q]);
    }
    if (!g->d_peer_z) {
        int32_t st;
        if ((st = dmalloc(g, (void **)&g->d_peer_z, kMaxWorld * sizeof(double *))) ||
            (st = dmalloc(g, (void **)&g->d_peer_flags, kMaxWorld * sizeof(uint32_t *))))
            return st;
    }
    if (!pz.empty())
        SC_CUDA(cudaMemcpy(g->d_peer_z, pz.data(), pz.size() * sizeof(double *),
                           cudaMemcpyHostToDevice));
    SC_CUDA(cudaMemcpy(g->d_peer_flags, pf.data(), pf.size() * sizeof(uint32_t *),
                       cudaMemcpyHostToDevice));
    g->npeer = (int)pz.size();
    g->world = world;
    g->rank = rank;
    return SC_OK;
}

int32_t sc_gather_f64(const double *src, const int32_t *idx, int64_t count, double *dst,
                      void *stream) {
    SC_REQUIRE(count >= 0, SC_E_INVALID, "negative count");
    if (count == 0) return SC_OK;
    SC_REQUIRE(src && idx && dst, SC_E_INVALID, "null argument");
    const int blocks = (int)std::min<int64_t>((count + 255) / 256, 148 * 16);
    k_gather_f64<<<blocks, 256, 0, (cudaStream_t)stream>>>(src, idx, count, dst);
    SC_CUDA(cudaGetLastError());
    return SC_OK;
}

int32_t sc_shard_barrier(sc_graph *g, void *stream) {
    SC_REQUIRE(g, SC_E_INVALID, "null graph");
    if (g->world <= 1) return SC_OK;
    SC_REQUIRE(g->d_flags, SC_E_STATE, "call sc_shard_buffers before the barrier");
    SC_CUDA(cudaSetDevice(g->device));
    k_peer_barrier<<<1, kMaxWorld, 0, (cudaStream_t)stream>>>(g->d_flags, g->d_peer_flags,
                                                               g->world, g->rank);
    SC_CUDA(cudaGetLastError());
    return SC_OK;
}

int32_t sc_ipc_export(const void *dptr, void *handle_out) {
    SC_REQUIRE(dptr && handle_out, SC_E_INVALID, "null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    SC_CUDA(cudaIpcGetMemHandle(&h, const_cast<void *>(dptr)));
    std::memcpy(handle_out, &h, 64);
    return SC_OK;
}

int32_t sc_ipc_import(const void *handle, int32_t device, void **dptr_out) {
    SC_REQUIRE(handle && dptr_out, SC_E_INVALID, "null argument");
    SC_CUDA(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    SC_CUDA(cudaIpcOpenMemHandle(dptr_out, h, cudaIpcMemLazyEnablePeerAccess));
    return SC_OK;
}

int32_t sc_ipc_release(void *dptr) {
    SC_REQUIRE(dptr, SC_E_INVALID, "null argument");
    SC_CUDA(cudaIpcCloseMemHandle(dptr));
    return SC_OK;
}

int32_t sc_shard_scale(sc_graph *g, const double *x, double *z_out, uint32_t flags,
                       void *stream) {
    SC_REQUIRE(g && x && z_out, SC_E_INVALID, "null argument");
    SC_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = (cudaStream_t)stream;  // the caller's stream, 0 = legacy default stream
    const bool sym = flags & SC_SYM_VARIANT;
    int32_t st;
    if (sym)
        if ((st = ensure_isd(g, s))) return st;
    int64_t poff = 0;
    if (g->npeer) {
        SC_REQUIRE(z_out >= g->d_z[0] && z_out < g->d_z[0] + g->zstride + g->ncols, SC_E_STATE,
                   "peer exchange needs z_out inside the handle's z buffers (sc_shard_buffers)");
        poff = z_out - g->d_z[0];
    }
    k_scale<<<grid_for(g, g->n, 256), 256, 0, s>>>(x, sym ? g->d_isd : g->d_deg, z_out, g->n,
                                                   g->col_offset, sym, g->d_peer_z, poff,
                                                   g->npeer);
    SC_CUDA(cudaGetLastError());
    return SC_OK;
}

int32_t sc_shard_irwin_hall(sc_graph *g, uint64_t key0, uint64_t key1, double *x_out,
                            void *stream) {
    SC_REQUIRE(g && x_out, SC_E_INVALID, "null argument");
    SC_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = (cudaStream_t)stream;  // the caller's stream, 0 = legacy default stream
    k_irwin_hall<<<grid_for(g, g->n, 128), 128, 0, s>>>(g->d_deg, g->d_perm, x_out, g->n,
                                                        g->global_row0, key0, key1);
    SC_CUDA(cudaGetLastError());
    return SC_OK;
}

}  // extern "C"

// internal accessors for sc_kmeans.cu
namespace sc {
// f (= z_T) in ORIGINAL vertex order, materialised on the device on demand
const double *graph_f_device(sc_graph *g) {
    if (g->multi) return multi_f_device(g);
    if (g->result < 0) return nullptr;
    if (!g->d_f_orig && dmalloc(g, (void **)&g->d_f_orig, (size_t)g->n * 8)) return nullptr;
    k_gather_perm<<<grid_for(g, g->n, 256), 256, 0, g->stream>>>(g->d_z[g->result], g->d_iperm,
                                                                 g->d_f_orig, g->n);
    if (cudaStreamSynchronize(g->stream) != cudaSuccess) return nullptr;
    return g->d_f_orig;
}
int64_t graph_n(const sc_graph *g) { return g->n; }
int graph_device(const sc_graph *g) { return g->device; }
}  // namespace sc

#include "sc_multi.cuh"
