// sc_graph.cu -- graph handle, Irwin-Hall start vector (K1) and the fused lazy-random-walk
// CSR SpMV (K2 + K3) for sm_100a.
//
// Reference semantics (paths under /root/reference/pkg/src/specluster):
//   power_method           spectral.py:87-102   x <- M x, t times, no normalisation
//   rw operator            SURVEY.md CS2        M x = 0.5*x + 0.5*(A @ (x/d))
//   SignlessLaplacianOp    spectral.py:52-57    M x = 0.5*x + 0.5*(s*(A @ (s*x)))
//   scipy csr_matvec       (sparsetools)        per row: sum = 0; sum += A_ij * v_j in
//                                               stored column order, no FMA
//
// Kernel design: the CSR is cut on the host into row tiles holding at most
// kChunk stored entries (rows longer than kChunk get a tile of their own).  One CTA per
// tile streams the tile's col/val with 128-bit evict-first loads, gathers z = D^-1 x
// through L1/L2, forms the products into shared memory, and then one thread per row adds
// its products left to right -- the scipy order, so the result is bit-identical to the
// reference.  The epilogue fuses the lazy blend 0.5 x + sign 0.5 s and the degree scaling
// of the next iterate: it writes x_{t+1} and z_{t+1} = x_{t+1} / d (the gathered vector
// of the next step, and after the last step the embedding f = D^-1 x_T itself).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <mutex>
#include <vector>

#include "sc_common.cuh"

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

constexpr int kTPB = 256;         // threads per tile CTA (8 warps)
constexpr int kChunk = 2048;      // stored entries per multi-row tile / per long-row chunk
constexpr int kRowsMax = 128;     // rows per multi-row tile (upper bound; see rows_cap)
constexpr int kPerThread = kChunk / kTPB;            // 8 entries per thread in phase A
constexpr int kPadded = kChunk + 16 * kRowsMax + 16; // padded product slots (32.1 KB)

struct StepArgs {
    const void *rp;        // int32 or int64 row offsets (local, rebased to 0)
    const uint32_t *col;   // packed: (tile-local row << col_bits) | column; padded (+8)
    const double *val;     // padded, or null for unit weights
    const double *scale;   // deg (rw) or deg^-1/2 (sym)
    const double *x_in;
    const double *z_in;    // gathered vector, indexed by column
    double *x_out;
    double *z_out;         // written at col_offset + row
    const int64_t *tile_b; // ntiles + 1 first stored entry of each tile
    const int32_t *tile_r; // ntiles + 1 first row of each tile
    int64_t col_offset;
    double hs;             // +0.5 or -0.5
    uint32_t col_mask;
    int col_bits;
};

// Shared-memory slot of row i's first product (pre = unpadded tile offset of the row).
// start == i (mod 16): the 16 lanes of a half-warp that read the t-th product of 16
// consecutive rows hit 16 distinct 8-byte bank pairs, so the sequential row sums of
// phase B are bank-conflict free; consecutive segments never overlap.
__device__ __forceinline__ int padded_start(int i, int pre) {
    return pre + 16 * i + ((i - pre) & 15);
}

// Long-row path: products of [cb, ce) into prod[0..), lane-linear coalesced loads.
template <bool UNIT>
__device__ __forceinline__ void gather_linear(const StepArgs &a, int64_t cb, int64_t ce,
                                              double *prod) {
    for (int64_t j = cb + threadIdx.x; j < ce; j += kTPB) {
        const uint32_t c = __ldcs(a.col + j) & a.col_mask;
        const double zv = __ldg(a.z_in + c);
        prod[j - cb] = UNIT ? zv : __dmul_rn(__ldcs(a.val + j), zv);
    }
}

template <bool SYM>
__device__ __forceinline__ void row_epilogue(const StepArgs &a, int64_t r, double s, double xr,
                                             double sc) {
    if (SYM) s = __dmul_rn(sc, s);
    const double y = __dadd_rn(__dmul_rn(0.5, xr), __dmul_rn(a.hs, s));
    __stcs(a.x_out + r, y);
    a.z_out[a.col_offset + r] = SYM ? __dmul_rn(sc, y) : __ddiv_rn(y, sc);
}

template <typename RP, bool UNIT, bool SYM>
__global__ void __launch_bounds__(kTPB) k_rw_step(StepArgs a) {
    __shared__ double prod[kPadded];
    __shared__ int pbase[kRowsMax + 1];  // padded_start(i, pre_i) - pre_i, then pre_i
    __shared__ int srp[kRowsMax + 1];    // tile-local row offsets
    const int tid = threadIdx.x;
    const int64_t b = a.tile_b[blockIdx.x], e = a.tile_b[blockIdx.x + 1];
    const int r0 = a.tile_r[blockIdx.x];
    const int nrows = a.tile_r[blockIdx.x + 1] - r0;
    if (e - b > kChunk) {
        // single long row: products chunk by chunk, one thread keeps the running sum
        double xr = 0.0, sc = 1.0;
        if (tid == 0) {
            xr = __ldcs(a.x_in + r0);
            sc = __ldcs(a.scale + r0);
        }
        double s = 0.0;
        for (int64_t cb = b; cb < e; cb += kChunk) {
            const int64_t ce = (e - cb > kChunk) ? cb + kChunk : e;
            gather_linear<UNIT>(a, cb, ce, prod);
            __syncthreads();
            if (tid == 0) {
                const int m = int(ce - cb);
                for (int j = 0; j < m; ++j) s = __dadd_rn(s, prod[j]);
            }
            __syncthreads();
        }
        if (tid == 0) row_epilogue<SYM>(a, r0, s, xr, sc);
        return;
    }
    const int nz = int(e - b);
    // phase A: warp w owns tile entries [256w, 256w + 256) as 8 lane-linear windows;
    // all col (+val) loads in flight first, then all gathers.  The tile-local row of each
    // entry travels in the high bits of the packed column word (no search).
    const int warp = tid >> 5, lane = tid & 31;
    const int wbase = warp * (32 * kPerThread);
    uint32_t cw[kPerThread];
    double v[kPerThread];
#pragma unroll
    for (int k = 0; k < kPerThread; ++k) {
        const int jl = wbase + 32 * k + lane;
        cw[k] = jl < nz ? __ldcs(a.col + b + jl) : 0u;
        v[k] = (!UNIT && jl < nz) ? __ldcs(a.val + b + jl) : 1.0;
    }
    // epilogue operands of this thread's row and the tile's row offsets (independent loads)
    double xr = 0.0, sc = 1.0;
    const RP *rp = static_cast<const RP *>(a.rp);
    if (tid < nrows) {
        xr = __ldcs(a.x_in + r0 + tid);
        sc = __ldcs(a.scale + r0 + tid);
    }
    if (tid <= nrows) {
        const int pre = int(rp[r0 + tid] - b);
        srp[tid] = pre;
        pbase[tid] = padded_start(tid, pre) - pre;
    }
#pragma unroll
    for (int k = 0; k < kPerThread; ++k) {
        const int jl = wbase + 32 * k + lane;
        if (jl < nz) {
            const double zv = __ldg(a.z_in + (cw[k] & a.col_mask));
            v[k] = UNIT ? zv : __dmul_rn(v[k], zv);
        }
    }
    __syncthreads();  // pbase ready
#pragma unroll
    for (int k = 0; k < kPerThread; ++k) {
        const int jl = wbase + 32 * k + lane;
        if (jl < nz) prod[pbase[cw[k] >> a.col_bits] + jl] = v[k];
    }
    __syncthreads();
    // phase B: one thread per row adds its products left to right (scipy csr_matvec order)
    if (tid < nrows) {
        const int pre = srp[tid], len = srp[tid + 1] - pre;
        const double *p = prod + pbase[tid] + pre;
        double s = 0.0;
        int t = 0;
        for (; t + 4 <= len; t += 4) {
            const double p0 = p[t], p1 = p[t + 1], p2 = p[t + 2], p3 = p[t + 3];
            s = __dadd_rn(s, p0);
            s = __dadd_rn(s, p1);
            s = __dadd_rn(s, p2);
            s = __dadd_rn(s, p3);
        }
        for (; t < len; ++t) s = __dadd_rn(s, p[t]);
        row_epilogue<SYM>(a, r0 + tid, s, xr, sc);
    }
}

// Stamp each stored entry of a multi-row tile with its tile-local row (high bits).
template <typename RP>
__global__ void k_pack_rows(const RP *__restrict__ rp, const int64_t *__restrict__ tile_b,
                            const int32_t *__restrict__ tile_r, uint32_t *__restrict__ col,
                            int col_bits) {
    const int64_t b = tile_b[blockIdx.x], e = tile_b[blockIdx.x + 1];
    if (e - b > kChunk) return;  // long-row tile: local row 0
    const int r0 = tile_r[blockIdx.x], nrows = tile_r[blockIdx.x + 1] - r0;
    for (int i = threadIdx.x >> 5; i < nrows; i += blockDim.x >> 5) {
        const int64_t lo = rp[r0 + i], hi = rp[r0 + i + 1];
        for (int64_t j = lo + (threadIdx.x & 31); j < hi; j += 32)
            col[j] |= (uint32_t)i << col_bits;
    }
}

// z[col_offset + i] = x[i] / d[i]   (rw)   or   x[i] * d[i]^-1/2   (sym)
__global__ void k_scale(const double *__restrict__ x, const double *__restrict__ scale,
                        double *__restrict__ z, int64_t n, int64_t off, int sym) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        z[off + i] = sym ? __dmul_rn(x[i], scale[i]) : __ddiv_rn(x[i], scale[i]);
}

// 1/sqrt(d), as numpy's 1.0 / np.sqrt(d) (spectral.py:49)
__global__ void k_inv_sqrt(const double *__restrict__ d, double *__restrict__ s, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        s[i] = __ddiv_rn(1.0, __dsqrt_rn(d[i]));
}

// K1: Irwin-Hall start vector.  Uniform j of global vertex u is word j%4 of
// Philox4x64-10(key, (j/4 + 1, u, 0, 0)); floor(deg) uniforms are summed left to right,
// a fractional degree adds frac * one more uniform (mean deg/2 for every degree).
__global__ void k_irwin_hall(const double *__restrict__ deg, double *__restrict__ x0, int64_t n,
                             int64_t global_row0, uint64_t k0, uint64_t k1) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double d = deg[i];
        const double fl = floor(d);
        const int64_t m = (int64_t)fl;
        const double frac = __dsub_rn(d, fl);
        const int64_t need = m + (frac > 0.0 ? 1 : 0);
        const uint64_t u = (uint64_t)(global_row0 + i);
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

}  // namespace sc

using namespace sc;

struct sc_graph {
    int device = 0;
    int sm_count = 0;
    int64_t n = 0, nnz = 0, ncols = 0, col_offset = 0, global_row0 = 0;
    bool unit = false, rp64 = false;
    void *d_rp = nullptr;
    uint32_t *d_col = nullptr;  // packed (local row << col_bits) | column
    double *d_val = nullptr;
    double *d_deg = nullptr;
    double *d_isd = nullptr;
    double *d_x0 = nullptr;
    double *d_x[2] = {nullptr, nullptr};
    double *d_z[2] = {nullptr, nullptr};
    int64_t *d_tile_b = nullptr;
    int32_t *d_tile_r = nullptr;
    int64_t ntiles = 0, long_rows = 0;
    int col_bits = 1, rows_cap = 1;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool have_x0 = false;
    int result = -1;  // buffer index holding x_T / f after the last power_iterate (2 = x0)
    cudaGraphExec_t gexec = nullptr;
    int32_t g_T = -1;
    uint32_t g_flags = 0;
    double g_sign = 0.0;
    int64_t bytes = 0;
    bool l2_window = false;
};

namespace sc {

static int32_t dmalloc(sc_graph *g, void **p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
    if (e != cudaSuccess)
        return fail(e == cudaErrorMemoryAllocation ? SC_E_OOM : SC_E_CUDA,
                    "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
    g->bytes += (int64_t)bytes;
    return SC_OK;
}

// Host tiling: greedy row packing, <= kChunk entries and <= rows_cap rows per tile;
// a row with more than kChunk entries is a tile of its own.
static void build_tiles(const int64_t *rp, int64_t n, int rows_cap, std::vector<int32_t> &tr,
                        std::vector<int64_t> &tb, int64_t &long_rows) {
    tr.clear();
    tb.clear();
    const size_t guess = (size_t)(rp[n] / kChunk + n / rows_cap + 16);
    tr.reserve(guess);
    tb.reserve(guess);
    auto cut = [&](int64_t r) {
        tr.push_back((int32_t)r);
        tb.push_back(rp[r]);
    };
    cut(0);
    int64_t cur_nnz = 0;
    int cur_rows = 0;
    long_rows = 0;
    for (int64_t r = 0; r < n; ++r) {
        const int64_t len = rp[r + 1] - rp[r];
        if (len > kChunk) {
            if (cur_rows) cut(r);
            cut(r + 1);
            ++long_rows;
            cur_nnz = 0;
            cur_rows = 0;
            continue;
        }
        if (cur_rows && (cur_nnz + len > kChunk || cur_rows == rows_cap)) {
            cut(r);
            cur_nnz = 0;
            cur_rows = 0;
        }
        cur_nnz += len;
        ++cur_rows;
    }
    if (cur_rows) cut(n);
}

static int32_t graph_init(const int64_t *row_ptr, const int32_t *col, const double *val,
                          const double *deg, int64_t n, int64_t nnz, int64_t ncols,
                          int64_t col_offset, int64_t global_row0, int32_t device,
                          sc_graph **out) {
    SC_REQUIRE(out, SC_E_INVALID, "out is null");
    *out = nullptr;
    SC_REQUIRE(row_ptr && deg && (col || nnz == 0), SC_E_INVALID, "null CSR array");
    SC_REQUIRE(n >= 1 && n < (int64_t(1) << 31) - 1, SC_E_INVALID, "n=%lld out of range",
               (long long)n);
    SC_REQUIRE(nnz >= 0 && row_ptr[0] == 0 && row_ptr[n] == nnz, SC_E_RANGE,
               "row_ptr[0] must be 0 and row_ptr[n] must equal nnz=%lld", (long long)nnz);
    SC_REQUIRE(ncols >= n && col_offset >= 0 && col_offset + n <= ncols, SC_E_RANGE,
               "bad z-space geometry ncols=%lld col_offset=%lld", (long long)ncols,
               (long long)col_offset);
    for (int64_t i = 0; i < n; ++i)
        SC_REQUIRE(row_ptr[i + 1] >= row_ptr[i], SC_E_RANGE, "row_ptr decreases at %lld",
                   (long long)i);
    for (int64_t i = 0; i < n; ++i)
        SC_REQUIRE(deg[i] > 0.0 && deg[i] < 1e308, SC_E_RANGE,
                   "degree of row %lld is not positive/finite", (long long)i);
    for (int64_t j = 0; j < nnz; ++j)
        SC_REQUIRE(col[j] >= 0 && col[j] < ncols, SC_E_RANGE, "col_indices[%lld]=%d out of range",
                   (long long)j, col[j]);
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
    bool unit = (val == nullptr);
    if (!unit) {
        unit = true;
        for (int64_t j = 0; j < nnz && unit; ++j) unit = (val[j] == 1.0);
    }
    g->unit = unit;
    g->rp64 = nnz >= (int64_t(1) << 31) - kChunk;

    g->col_bits = 1;
    while (g->col_bits < 31 && (int64_t(1) << g->col_bits) < ncols) ++g->col_bits;
    g->rows_cap = (int)std::min<int64_t>(kRowsMax, int64_t(1) << (32 - g->col_bits));
    std::vector<int32_t> tile_r;
    std::vector<int64_t> tile_b;
    build_tiles(row_ptr, n, g->rows_cap, tile_r, tile_b, g->long_rows);
    g->ntiles = (int64_t)tile_r.size() - 1;

    int32_t st;
    auto cleanup = [&](int32_t code) {
        sc_graph_destroy(g);
        return code;
    };
    const size_t rpb = (size_t)(n + 1) * (g->rp64 ? 8 : 4);
    if ((st = dmalloc(g, &g->d_rp, rpb))) return cleanup(st);
    if ((st = dmalloc(g, (void **)&g->d_col, (size_t)(nnz + 8) * 4))) return cleanup(st);
    if (val && !unit)
        if ((st = dmalloc(g, (void **)&g->d_val, (size_t)(nnz + 8) * 8))) return cleanup(st);
    if ((st = dmalloc(g, (void **)&g->d_deg, (size_t)n * 8))) return cleanup(st);
    if ((st = dmalloc(g, (void **)&g->d_x0, (size_t)n * 8))) return cleanup(st);
    for (int b = 0; b < 2; ++b) {
        if ((st = dmalloc(g, (void **)&g->d_x[b], (size_t)n * 8))) return cleanup(st);
    }
    // both z buffers in one allocation so one L2 access-policy window covers them
    double *zz = nullptr;
    if ((st = dmalloc(g, (void **)&zz, (size_t)ncols * 16))) return cleanup(st);
    g->d_z[0] = zz;
    g->d_z[1] = zz + ncols;
    if ((st = dmalloc(g, (void **)&g->d_tile_r, tile_r.size() * 4))) return cleanup(st);
    if ((st = dmalloc(g, (void **)&g->d_tile_b, tile_b.size() * 8))) return cleanup(st);

    cudaError_t e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&g->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&g->ev1);
    if (e == cudaSuccess) {
        if (g->rp64) {
            e = cudaMemcpyAsync(g->d_rp, row_ptr, rpb, cudaMemcpyHostToDevice, g->stream);
        } else {
            std::vector<int32_t> rp32((size_t)n + 1);
            for (int64_t i = 0; i <= n; ++i) rp32[i] = (int32_t)row_ptr[i];
            e = cudaMemcpyAsync(g->d_rp, rp32.data(), rpb, cudaMemcpyHostToDevice, g->stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
        }
    }
    if (e == cudaSuccess && nnz)
        e = cudaMemcpyAsync(g->d_col, col, (size_t)nnz * 4, cudaMemcpyHostToDevice, g->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(g->d_col + nnz, 0, 32, g->stream);
    if (e == cudaSuccess && g->d_val) {
        e = cudaMemcpyAsync(g->d_val, val, (size_t)nnz * 8, cudaMemcpyHostToDevice, g->stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(g->d_val + nnz, 0, 64, g->stream);
    }
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(g->d_deg, deg, (size_t)n * 8, cudaMemcpyHostToDevice, g->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(g->d_tile_r, tile_r.data(), tile_r.size() * 4, cudaMemcpyHostToDevice,
                            g->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(g->d_tile_b, tile_b.data(), tile_b.size() * 8, cudaMemcpyHostToDevice,
                            g->stream);
    if (e == cudaSuccess && g->ntiles) {
        if (g->rp64)
            k_pack_rows<int64_t><<<(unsigned)g->ntiles, 256, 0, g->stream>>>(
                (const int64_t *)g->d_rp, g->d_tile_b, g->d_tile_r, g->d_col, g->col_bits);
        else
            k_pack_rows<int32_t><<<(unsigned)g->ntiles, 256, 0, g->stream>>>(
                (const int32_t *)g->d_rp, g->d_tile_b, g->d_tile_r, g->d_col, g->col_bits);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(zz, 0, (size_t)ncols * 16, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    if (e != cudaSuccess) {
        fail(SC_E_CUDA, "graph upload failed: %s", cudaGetErrorString(e));
        return cleanup(SC_E_CUDA);
    }
    *out = g;
    return SC_OK;
}

static int grid_for(const sc_graph *g, int64_t n, int tpb) {
    int64_t want = (n + tpb - 1) / tpb;
    int64_t cap = (int64_t)std::max(g->sm_count, 1) * 8;
    return (int)std::max<int64_t>(1, std::min(want, cap));
}

static int32_t ensure_isd(sc_graph *g, cudaStream_t s) {
    if (g->d_isd) return SC_OK;
    int32_t st = dmalloc(g, (void **)&g->d_isd, (size_t)g->n * 8);
    if (st) return st;
    k_inv_sqrt<<<grid_for(g, g->n, 256), 256, 0, s>>>(g->d_deg, g->d_isd, g->n);
    SC_CUDA(cudaGetLastError());
    return SC_OK;
}

static int32_t launch_step(const sc_graph *g, const double *z_in, const double *x_in,
                           double *x_out, double *z_out, double sign, uint32_t flags,
                           cudaStream_t s) {
    if (g->ntiles == 0) return SC_OK;
    const bool sym = flags & SC_SYM_VARIANT;
    const bool unit = g->unit && !(flags & SC_FORCE_WEIGHTED && g->d_val);
    StepArgs a;
    a.rp = g->d_rp;
    a.col = g->d_col;
    a.val = g->d_val;
    a.scale = sym ? g->d_isd : g->d_deg;
    a.x_in = x_in;
    a.z_in = z_in;
    a.x_out = x_out;
    a.z_out = z_out;
    a.tile_b = g->d_tile_b;
    a.tile_r = g->d_tile_r;
    a.col_offset = g->col_offset;
    a.col_bits = g->col_bits;
    a.col_mask = g->col_bits >= 32 ? 0xffffffffu : ((1u << g->col_bits) - 1u);
    a.hs = sign < 0 ? -0.5 : 0.5;
    const dim3 grid((unsigned)g->ntiles);
#define SC_LAUNCH(RP, U, S) k_rw_step<RP, U, S><<<grid, kTPB, 0, s>>>(a)
    if (g->rp64) {
        if (unit) { if (sym) SC_LAUNCH(int64_t, true, true); else SC_LAUNCH(int64_t, true, false); }
        else { if (sym) SC_LAUNCH(int64_t, false, true); else SC_LAUNCH(int64_t, false, false); }
    } else {
        if (unit) { if (sym) SC_LAUNCH(int32_t, true, true); else SC_LAUNCH(int32_t, true, false); }
        else { if (sym) SC_LAUNCH(int32_t, false, true); else SC_LAUNCH(int32_t, false, false); }
    }
#undef SC_LAUNCH
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
        size_t bytes = (size_t)g->ncols * 16;
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

}  // namespace sc

extern "C" {

int32_t sc_version(void) { return 1; }

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
    return graph_init(row_ptr, col, val, deg, n, nnz, n, 0, 0, device, out);
}

int32_t sc_shard_create(const int64_t *row_ptr, const int32_t *col, const double *val,
                        const double *deg, int64_t n, int64_t nnz, int64_t ncols,
                        int64_t col_offset, int64_t global_row0, int32_t device,
                        sc_graph **out) {
    return graph_init(row_ptr, col, val, deg, n, nnz, ncols, col_offset, global_row0, device,
                      out);
}

void sc_graph_destroy(sc_graph *g) {
    if (!g) return;
    cudaSetDevice(g->device);
    if (g->stream) cudaStreamSynchronize(g->stream);
    if (g->gexec) cudaGraphExecDestroy(g->gexec);
    cudaFree(g->d_rp);
    cudaFree(g->d_col);
    cudaFree(g->d_val);
    cudaFree(g->d_deg);
    cudaFree(g->d_isd);
    cudaFree(g->d_x0);
    cudaFree(g->d_x[0]);
    cudaFree(g->d_x[1]);
    cudaFree(g->d_z[0]);
    cudaFree(g->d_tile_b);
    cudaFree(g->d_tile_r);
    if (g->ev0) cudaEventDestroy(g->ev0);
    if (g->ev1) cudaEventDestroy(g->ev1);
    if (g->stream) cudaStreamDestroy(g->stream);
    delete g;
}

int32_t sc_graph_info_get(const sc_graph *g, sc_graph_info *o) {
    SC_REQUIRE(g && o, SC_E_INVALID, "null argument");
    o->n = g->n;
    o->nnz = g->nnz;
    o->ncols = g->ncols;
    o->col_offset = g->col_offset;
    o->ntiles = g->ntiles;
    o->long_rows = g->long_rows;
    o->unit_weights = g->unit;
    o->rp64 = g->rp64;
    o->device_bytes = g->bytes;
    o->device = g->device;
    o->sm_count = g->sm_count;
    return SC_OK;
}

int32_t sc_sample_irwin_hall(sc_graph *g, uint64_t key0, uint64_t key1, double *x0_out) {
    SC_REQUIRE(g, SC_E_INVALID, "null graph");
    SC_CUDA(cudaSetDevice(g->device));
    k_irwin_hall<<<grid_for(g, g->n, 128), 128, 0, g->stream>>>(g->d_deg, g->d_x0, g->n,
                                                                g->global_row0, key0, key1);
    SC_CUDA(cudaGetLastError());
    if (x0_out)
        SC_CUDA(cudaMemcpyAsync(x0_out, g->d_x0, (size_t)g->n * 8, cudaMemcpyDeviceToHost,
                                g->stream));
    SC_CUDA(cudaStreamSynchronize(g->stream));
    g->have_x0 = true;
    g->result = -1;
    return SC_OK;
}

int32_t sc_set_x0(sc_graph *g, const double *x0_host) {
    SC_REQUIRE(g && x0_host, SC_E_INVALID, "null argument");
    SC_CUDA(cudaSetDevice(g->device));
    SC_CUDA(cudaMemcpyAsync(g->d_x0, x0_host, (size_t)g->n * 8, cudaMemcpyHostToDevice,
                            g->stream));
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
    if (xT_out)
        SC_CUDA(cudaMemcpy(xT_out, xT, (size_t)g->n * 8, cudaMemcpyDeviceToHost));
    if (f_out) SC_CUDA(cudaMemcpy(f_out, f, (size_t)g->n * 8, cudaMemcpyDeviceToHost));
    auto h1 = std::chrono::steady_clock::now();
    if (t_out) {
        t_out->power_ms = ms;
        t_out->kernel_ms = T ? ms / T : 0.0;
        t_out->d2h_ms = std::chrono::duration<double, std::milli>(h1 - h0).count();
    }
    return SC_OK;
}

int32_t sc_shard_step(sc_graph *g, const double *z_in, const double *x_in, double *x_out,
                      double *z_out, double sign, uint32_t flags, void *stream) {
    SC_REQUIRE(g && z_in && x_in && x_out && z_out, SC_E_INVALID, "null argument");
    SC_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = stream ? (cudaStream_t)stream : g->stream;
    int32_t st;
    if (flags & SC_SYM_VARIANT)
        if ((st = ensure_isd(g, s))) return st;
    return launch_step(g, z_in, x_in, x_out, z_out, sign, flags, s);
}

int32_t sc_shard_scale(sc_graph *g, const double *x, double *z_out, uint32_t flags,
                       void *stream) {
    SC_REQUIRE(g && x && z_out, SC_E_INVALID, "null argument");
    SC_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = stream ? (cudaStream_t)stream : g->stream;
    const bool sym = flags & SC_SYM_VARIANT;
    int32_t st;
    if (sym)
        if ((st = ensure_isd(g, s))) return st;
    k_scale<<<grid_for(g, g->n, 256), 256, 0, s>>>(x, sym ? g->d_isd : g->d_deg, z_out, g->n,
                                                   g->col_offset, sym);
    SC_CUDA(cudaGetLastError());
    return SC_OK;
}

int32_t sc_shard_irwin_hall(sc_graph *g, uint64_t key0, uint64_t key1, double *x_out,
                            void *stream) {
    SC_REQUIRE(g && x_out, SC_E_INVALID, "null argument");
    SC_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = stream ? (cudaStream_t)stream : g->stream;
    k_irwin_hall<<<grid_for(g, g->n, 128), 128, 0, s>>>(g->d_deg, x_out, g->n, g->global_row0,
                                                        key0, key1);
    SC_CUDA(cudaGetLastError());
    return SC_OK;
}

}  // extern "C"

// internal accessors for sc_kmeans.cu
namespace sc {
const double *graph_f_device(const sc_graph *g) {
    return g->result < 0 ? nullptr : g->d_z[g->result];
}
int64_t graph_n(const sc_graph *g) { return g->n; }
int graph_device(const sc_graph *g) { return g->device; }
}  // namespace sc
