// sc_generate_wt.cu -- device generators for the weighted benchmark graphs (BASELINE.json
// configs 3 and 4).  The reference has no generator for either (its
// kNN builder is brute force, unit weights and refuses n > 50,000: generate.py:176-220); the
// laws below are ours, realised on counter-based Philox streams and elementary functions built
// from correctly rounded operations (sc_genmath.cuh), so oracle/oracle.py (numpy, the same
// operation sequence) reproduces every graph bit for bit.
//
// Config 4, weighted random geometric cluster graph (sc_generate_knn3d):
//   centre j (< k):  (U0, U1, U2) of Philox(key, (b + 1, j, kTagCentres, 0))
//   point i (< n):   stream Philox(key, (b + 1, i, kTagPoints, 0)), 40 words: label
//                    floor(U0 * k); coordinate c = centre[label][c] + sigma * z_c with
//                    z_c = (U_{1+12c} + ... + U_{12+12c}) - 6, summed left to right (the
//                    Irwin-Hall(12) stand-in for a standard normal: mean 0, variance 1)
//   U = (raw >> 11) * 2^-53 for every word
//   neighbours:      the knn points j != i with the smallest (d2(i, j), j), where
//                    d2 = ((dx*dx + dy*dy) + dz*dz), dx = xi - xj, every operation rounded
//   edges:           the union of the neighbour pairs, symmetric, weight
//                    max(sc_exp(-(d2 / scale)), DBL_MIN) (d2 is symmetric: negation is exact)
// The kNN search buckets the points in a uniform grid over their bounding box and grows a
// cube of cells around each point until the knn-th distance cannot be beaten outside it.
//
// Config 3, degree-corrected SBM (sc_generate_dcsbm; block offsets from the host):
//   vertex i, stream Philox(key, (b + 1, i, kTagDegrees, 0)): U0 -> expected degree
//            d_i = clamp(floor(sc_exp(sc_log(A + U0 * (B - A)) / a)), dmin, dmax) with
//            a = 1 - gamma, A = dmin^a, B = dmax^a (truncated power law, inverse CDF);
//            U1 -> stubs m_i = d_i / 2 (+1 if d_i is odd and U1 < 0.5)
//   stub s of i, stream Philox(key, (b + 1, i, kTagStubs, 0)), words 3s..3s+2: inside =
//            U >= mix; target t = floor(U' * W) over the inclusive prefix sums of the integer
//            degrees of i's block (inside) or of all vertices; partner = the first vertex
//            whose prefix sum exceeds t (searchsorted 'right'); weight wlo + (whi - wlo) * U''
//   edges:   self loops dropped; of the stubs joining the same pair only the first (stub
//            order) counts; symmetric; isolated vertices dropped, ids compacted
// Degrees of both graphs: the row's weights summed left to right in column order.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cfloat>
#include <vector>

#include "sc_common.cuh"
#include "sc_csr.cuh"
#include "sc_genmath.cuh"

namespace sc {

constexpr uint64_t kTagCentres = 0x43454e54u, kTagPoints = 0x504f494eu;
constexpr uint64_t kTagDegrees = 0x44454752u, kTagStubs = 0x53545542u;
constexpr int kMaxKnn = 32;

__device__ __forceinline__ double u53w(uint64_t w) {
    return (double)(w >> 11) * 1.1102230246251565e-16;
}

struct Stream {
    uint64_t id, tag, k0, k1;
    uint64_t blk = 0;
    int idx = 4;
    uint64_t w[4];
    __device__ uint64_t next() {
        if (idx == 4) {
            const u64x4 r = philox4x64_10(u64x4{blk + 1, id, tag, 0}, k0, k1);
            w[0] = r.x;
            w[1] = r.y;
            w[2] = r.z;
            w[3] = r.w;
            idx = 0;
            ++blk;
        }
        return w[idx++];
    }
    __device__ void seek(uint64_t word) {  // position the stream at word `word`
        blk = word / 4;
        idx = 4;
        const int skip = (int)(word % 4);
        if (skip) {
            next();
            idx = skip;
        }
    }
};

// ---------------------------------------------------------------------------------------
// config 4

__global__ void k_knn_points(int64_t n, int k, double sigma, uint64_t k0, uint64_t k1,
                             double *__restrict__ px, double *__restrict__ py,
                             double *__restrict__ pz, int32_t *__restrict__ plab) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        Stream st{(uint64_t)i, kTagPoints, k0, k1};
        int lab = (int)floor(u53w(st.next()) * (double)k);
        lab = lab < k ? lab : k - 1;
        Stream cs{(uint64_t)lab, kTagCentres, k0, k1};
        double cen[3], z[3];
        for (int c = 0; c < 3; ++c) cen[c] = u53w(cs.next());
        for (int c = 0; c < 3; ++c) {
            double acc = 0.0;
            for (int t = 0; t < 12; ++t) acc = __dadd_rn(acc, u53w(st.next()));
            z[c] = __dsub_rn(acc, 6.0);
        }
        px[i] = __dadd_rn(cen[0], __dmul_rn(sigma, z[0]));
        py[i] = __dadd_rn(cen[1], __dmul_rn(sigma, z[1]));
        pz[i] = __dadd_rn(cen[2], __dmul_rn(sigma, z[2]));
        plab[i] = lab;
    }
}

struct GridBox {
    double lo[3], inv[3], w[3];  // cell index = floor((x - lo) * inv), cell width w
    int G;
};

__device__ __forceinline__ int cell_of(double v, const GridBox &g, int ax) {
    int c = (int)floor((v - g.lo[ax]) * g.inv[ax]);
    return c < 0 ? 0 : (c >= g.G ? g.G - 1 : c);
}

__global__ void k_knn_cells(int64_t n, GridBox g, const double *__restrict__ px,
                            const double *__restrict__ py, const double *__restrict__ pz,
                            uint32_t *__restrict__ cell, int32_t *__restrict__ iota) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t cx = cell_of(px[i], g, 0), cy = cell_of(py[i], g, 1), cz = cell_of(pz[i], g, 2);
        cell[i] = (cz * (uint32_t)g.G + cy) * (uint32_t)g.G + cx;
        iota[i] = (int32_t)i;
    }
}

__global__ void k_cell_starts(int64_t n, const uint32_t *__restrict__ cell_sorted,
                              int64_t ncell, int32_t *__restrict__ start) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= n;
         t += (int64_t)gridDim.x * blockDim.x) {
        // start[c] = first sorted position with cell >= c
        const int64_t a = t == 0 ? -1 : (int64_t)cell_sorted[t - 1];
        const int64_t b = t == n ? ncell : (int64_t)cell_sorted[t];
        for (int64_t c = a + 1; c <= b; ++c) start[c] = (int32_t)t;
    }
}

__device__ __forceinline__ double d2exact(double xi, double yi, double zi, double xj, double yj,
                                          double zj) {
    const double dx = __dsub_rn(xi, xj), dy = __dsub_rn(yi, yj), dz = __dsub_rn(zi, zj);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// thread per point: the knn nearest (d2, id), cubes of cells grown until the knn-th distance is
// provably below the distance to every unsearched cell
template <int K>
__global__ void __launch_bounds__(128) k_knn_search(
    int64_t n, GridBox g, const double *__restrict__ px, const double *__restrict__ py,
    const double *__restrict__ pz, const int32_t *__restrict__ order,
    const int32_t *__restrict__ start, int32_t *__restrict__ nb, double *__restrict__ nd2) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double xi = px[i], yi = py[i], zi = pz[i];
        const int cx = cell_of(xi, g, 0), cy = cell_of(yi, g, 1), cz = cell_of(zi, g, 2);
        double bd[K];
        int bj[K];
#pragma unroll
        for (int q = 0; q < K; ++q) {
            bd[q] = INFINITY;
            bj[q] = INT32_MAX;
        }
        for (int r = 0; r <= g.G; ++r) {
            for (int z = cz - r; z <= cz + r; ++z) {
                if (z < 0 || z >= g.G) continue;
                for (int y = cy - r; y <= cy + r; ++y) {
                    if (y < 0 || y >= g.G) continue;
                    const bool zy_edge = z == cz - r || z == cz + r || y == cy - r || y == cy + r;
                    for (int x = cx - r; x <= cx + r; x += (zy_edge || r == 0) ? 1 : 2 * r) {
                        if (x < 0 || x >= g.G) continue;
                        const int64_t c = ((int64_t)z * g.G + y) * g.G + x;
                        for (int p = start[c]; p < start[c + 1]; ++p) {
                            const int j = order[p];
                            if (j == i) continue;
                            const double d = d2exact(xi, yi, zi, px[j], py[j], pz[j]);
                            if (d < bd[K - 1] || (d == bd[K - 1] && j < bj[K - 1])) {
                                double cd = d;
                                int cj = j;
#pragma unroll
                                for (int q = 0; q < K; ++q) {  // sorted insert
                                    const bool before = cd < bd[q] || (cd == bd[q] && cj < bj[q]);
                                    const double td = bd[q];
                                    const int tj = bj[q];
                                    bd[q] = before ? cd : bd[q];
                                    bj[q] = before ? cj : bj[q];
                                    cd = before ? td : cd;
                                    cj = before ? tj : cj;
                                }
                            }
                        }
                    }
                }
            }
            // smallest distance from the point to a cell outside the searched cube (cube faces
            // at the grid border have nothing beyond them)
            double m = INFINITY;
            const int cc[3] = {cx, cy, cz};
            const double vv[3] = {xi, yi, zi};
            for (int ax = 0; ax < 3; ++ax) {
                if (cc[ax] - r > 0) m = fmin(m, vv[ax] - (g.lo[ax] + (cc[ax] - r) * g.w[ax]));
                if (cc[ax] + r < g.G - 1) m = fmin(m, (g.lo[ax] + (cc[ax] + r + 1) * g.w[ax]) - vv[ax]);
            }
            if (m == INFINITY) break;  // the whole grid was searched
            m = fmax(m - 1e-9 * (g.w[0] + g.w[1] + g.w[2]), 0.0);  // cell rounding margin
            if (bd[K - 1] < m * m * (1.0 - 1e-9)) break;
        }
#pragma unroll
        for (int q = 0; q < K; ++q) {
            nb[i * K + q] = bj[q];
            nd2[i * K + q] = bd[q];
        }
    }
}

// both directions of every neighbour pair: key (row << 32 | col), weight
__global__ void k_knn_pairs(int64_t n, int K, double scale, const int32_t *__restrict__ nb,
                            const double *__restrict__ nd2, uint64_t *__restrict__ key,
                            double *__restrict__ w) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * K;
         t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t i = (uint64_t)(t / K), j = (uint64_t)nb[t];
        double v = sc_exp(-__ddiv_rn(nd2[t], scale));
        v = v < DBL_MIN ? DBL_MIN : v;
        key[2 * t] = (i << 32) | j;
        key[2 * t + 1] = (j << 32) | i;
        w[2 * t] = v;
        w[2 * t + 1] = v;
    }
}

// ---------------------------------------------------------------------------------------
// config 3

__global__ void k_dc_degrees(int64_t n, double A, double BmA, double inv_a, int dmin, int dmax,
                             uint64_t k0, uint64_t k1, int64_t *__restrict__ deg,
                             int64_t *__restrict__ stubs) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        Stream st{(uint64_t)i, kTagDegrees, k0, k1};
        const double u0 = u53w(st.next()), u1 = u53w(st.next());
        const double x = sc_exp(__dmul_rn(sc_log(__dadd_rn(A, __dmul_rn(u0, BmA))), inv_a));
        double fl = floor(x);
        fl = fl < (double)dmin ? (double)dmin : (fl > (double)dmax ? (double)dmax : fl);
        const int64_t d = (int64_t)fl;
        deg[i] = d;
        stubs[i] = d / 2 + ((d & 1) && u1 < 0.5 ? 1 : 0);
    }
}

__device__ __forceinline__ int64_t upper_bound(const int64_t *__restrict__ a, int64_t lo,
                                               int64_t hi, int64_t t) {
    while (lo < hi) {  // first index in [lo, hi) with a[idx] > t
        const int64_t mid = (lo + hi) / 2;
        if (a[mid] > t) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

// stub s of vertex i -> unordered pair key (min << 32 | max) or ~0 (self loop), weight
__global__ void k_dc_stubs(int64_t n, const int64_t *__restrict__ boff, int nblk, double mix,
                           double wlo, double wspan, uint64_t k0, uint64_t k1,
                           const int64_t *__restrict__ cum, const int64_t *__restrict__ stub_off,
                           const int64_t *__restrict__ stubs, uint64_t *__restrict__ key,
                           double *__restrict__ w) {
    const int64_t W = cum[n - 1];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        // block of i
        int lo = 0, hi = nblk;
        while (hi - lo > 1) {
            const int mid = (lo + hi) / 2;
            if (boff[mid] <= i) lo = mid;
            else hi = mid;
        }
        const int64_t b0 = boff[lo], b1 = boff[lo + 1];
        const int64_t before = b0 > 0 ? cum[b0 - 1] : 0;
        const int64_t Wb = cum[b1 - 1] - before;
        Stream st{(uint64_t)i, kTagStubs, k0, k1};
        const int64_t o = stub_off[i], m = stubs[i];
        for (int64_t s = 0; s < m; ++s) {
            const double ua = u53w(st.next()), ub = u53w(st.next()), uc = u53w(st.next());
            int64_t p;
            if (ua >= mix) {
                const int64_t t = before + (int64_t)floor(__dmul_rn(ub, (double)Wb));
                p = upper_bound(cum, b0, b1, t);
            } else {
                const int64_t t = (int64_t)floor(__dmul_rn(ub, (double)W));
                p = upper_bound(cum, 0, n, t);
            }
            const uint64_t a = (uint64_t)min(i, p), bb = (uint64_t)max(i, p);
            key[o + s] = p == i ? ~0ull : ((a << 32) | bb);
            w[o + s] = __dadd_rn(wlo, __dmul_rn(wspan, uc));
        }
    }
}

// keep the first of each run of equal keys (sorted, stable); drop ~0 keys
__global__ void k_unique_flags(int64_t m, const uint64_t *__restrict__ key, int32_t *__restrict__ flag) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
         t += (int64_t)gridDim.x * blockDim.x)
        flag[t] = key[t] != ~0ull && (t == 0 || key[t] != key[t - 1]);
}

__global__ void k_unique_both(int64_t m, const uint64_t *__restrict__ key, const double *__restrict__ w,
                              const int32_t *__restrict__ flag, const int64_t *__restrict__ pos,
                              uint64_t *__restrict__ okey, double *__restrict__ ow) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
         t += (int64_t)gridDim.x * blockDim.x) {
        if (!flag[t]) continue;
        const uint64_t a = key[t] >> 32, b = key[t] & 0xffffffffull;
        const int64_t o = 2 * pos[t];
        okey[o] = key[t];
        okey[o + 1] = (b << 32) | a;
        ow[o] = w[t];
        ow[o + 1] = w[t];
    }
}

__global__ void k_unique_copy(int64_t m, const uint64_t *__restrict__ key, const double *__restrict__ w,
                              const int32_t *__restrict__ flag, const int64_t *__restrict__ pos,
                              uint64_t *__restrict__ okey, double *__restrict__ ow) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
         t += (int64_t)gridDim.x * blockDim.x) {
        if (!flag[t]) continue;
        okey[pos[t]] = key[t];
        ow[pos[t]] = w[t];
    }
}

// ---------------------------------------------------------------------------------------
// shared assembly: sorted unique (row << 32 | col) keys with weights -> compacted CSR

__global__ void k_row_len(int64_t m, const uint64_t *__restrict__ key, int64_t *__restrict__ len) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
         t += (int64_t)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long *)&len[key[t] >> 32], 1ull);
}

__global__ void k_keep_rows(int64_t n, const int64_t *__restrict__ len, int32_t *__restrict__ keep) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x)
        keep[u] = len[u] > 0;
}

__global__ void k_fill_csr(int64_t m, const uint64_t *__restrict__ key, const double *__restrict__ w,
                           const int32_t *__restrict__ newid, int32_t *__restrict__ col,
                           double *__restrict__ val) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
         t += (int64_t)gridDim.x * blockDim.x) {
        col[t] = newid[key[t] & 0xffffffffull];
        val[t] = w[t];
    }
}

__global__ void k_rows_out(int64_t n, const int64_t *__restrict__ len, const int64_t *__restrict__ off,
                           const int32_t *__restrict__ keep, const int32_t *__restrict__ newid,
                           const double *__restrict__ val, int64_t *__restrict__ rp,
                           double *__restrict__ deg, int32_t *__restrict__ orig) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        if (!keep[u]) continue;
        const int32_t id = newid[u];
        const int64_t b = off[u], e = b + len[u];
        rp[id] = b;
        orig[id] = (int32_t)u;
        double s = 0.0;  // left to right in column order
        for (int64_t t = b; t < e; ++t) s = __dadd_rn(s, val[t]);
        deg[id] = s;
    }
}

__global__ void k_set_last64(int64_t *rp, int64_t idx, int64_t v) { rp[idx] = v; }

struct GenCtx {
    cudaStream_t s = nullptr;
    int grid = 148 * 8;
    std::vector<void *> tmp;
    void *cub = nullptr;
    size_t cub_bytes = 0;
    cudaError_t e = cudaSuccess;
    template <typename T>
    T *alloc(size_t count) {
        T *p = nullptr;
        if (e) return nullptr;
        e = cudaMallocAsync((void **)&p, std::max<size_t>(count, 1) * sizeof(T), s);
        if (!e) tmp.push_back(p);
        return p;
    }
    void release(void *p) {
        for (auto &q : tmp)
            if (q == p) {
                cudaFreeAsync(p, s);
                q = nullptr;
            }
    }
    void *need(size_t b) {
        if (e) return nullptr;
        if (b > cub_bytes) {
            if (cub) cudaFreeAsync(cub, s);
            cub = nullptr;
            e = cudaMallocAsync(&cub, b, s);
            cub_bytes = e ? 0 : b;
        }
        return cub;
    }
    ~GenCtx() {
        for (void *p : tmp)
            if (p) cudaFreeAsync(p, s);
        if (cub) cudaFreeAsync(cub, s);
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

// sort (key, weight) pairs by key (stable), in place through alternate buffers
static void sort_pairs(GenCtx &G, uint64_t *&key, double *&w, int64_t m, int end_bit) {
    if (G.e || m <= 1) return;
    uint64_t *k2 = G.alloc<uint64_t>(m);
    double *w2 = G.alloc<double>(m);
    if (G.e) return;
    size_t b = 0;
    cub::DoubleBuffer<uint64_t> dk(key, k2);
    cub::DoubleBuffer<double> dv(w, w2);
    G.e = cub::DeviceRadixSort::SortPairs(nullptr, b, dk, dv, m, 0, end_bit, G.s);
    void *t = G.need(b);
    if (!G.e) G.e = cub::DeviceRadixSort::SortPairs(t, b, dk, dv, m, 0, end_bit, G.s);
    if (G.e) return;
    if (dk.Current() != key) {
        G.release(key);
        G.release(w);
        key = dk.Current();
        w = dv.Current();
    } else {
        G.release(k2);
        G.release(w2);
    }
}

template <typename In, typename Out>
static void excl_scan(GenCtx &G, const In *in, Out *out, int64_t m) {
    if (G.e) return;
    size_t b = 0;
    G.e = cub::DeviceScan::ExclusiveSum(nullptr, b, in, out, m, G.s);
    void *t = G.need(b);
    if (!G.e) G.e = cub::DeviceScan::ExclusiveSum(t, b, in, out, m, G.s);
}

template <typename T>
static T fetch(GenCtx &G, const T *p) {
    T v{};
    if (G.e) return v;
    G.e = cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, G.s);
    if (!G.e) G.e = cudaStreamSynchronize(G.s);
    return v;
}

// sorted unique symmetric (key, w) with m entries -> sc_csr (rows without entries dropped)
static int32_t assemble(GenCtx &G, int64_t n, const uint64_t *key, const double *w, int64_t m,
                        int device, sc_csr **out) {
    int64_t *len = G.alloc<int64_t>(n), *off = G.alloc<int64_t>(n + 1);
    int32_t *keep = G.alloc<int32_t>(n), *newid = G.alloc<int32_t>(n);
    if (!G.e) G.e = cudaMemsetAsync(len, 0, (size_t)n * 8, G.s);
    if (!G.e) {
        k_row_len<<<G.grid, 256, 0, G.s>>>(m, key, len);
        k_keep_rows<<<G.grid, 256, 0, G.s>>>(n, len, keep);
        G.e = cudaGetLastError();
    }
    excl_scan(G, len, off, n);
    excl_scan(G, keep, newid, n);
    const int64_t nk = (int64_t)fetch(G, newid + n - 1) + fetch(G, keep + n - 1);
    if (G.e) return fail(G.e == cudaErrorMemoryAllocation ? SC_E_OOM : SC_E_CUDA,
                         "generator assembly: %s", cudaGetErrorString(G.e));
    SC_REQUIRE(nk > 0, SC_E_INVALID, "the sampled graph has no edges");
    sc_csr *h = new sc_csr();
    h->device = device;
    h->n_gen = n;
    h->n = nk;
    h->nnz = m;
    cudaError_t e = cudaMalloc((void **)&h->d_rp, (size_t)(nk + 1) * 8);
    if (!e) e = cudaMalloc((void **)&h->d_col, (size_t)std::max<int64_t>(m, 1) * 4);
    if (!e) e = cudaMalloc((void **)&h->d_val, (size_t)std::max<int64_t>(m, 1) * 8);
    if (!e) e = cudaMalloc((void **)&h->d_deg, (size_t)nk * 8);
    if (!e) e = cudaMalloc((void **)&h->d_orig, (size_t)nk * 4);
    if (!e) {
        k_fill_csr<<<G.grid, 256, 0, G.s>>>(m, key, w, newid, h->d_col, h->d_val);
        k_rows_out<<<G.grid, 256, 0, G.s>>>(n, len, off, keep, newid, h->d_val, h->d_rp, h->d_deg,
                                            h->d_orig);
        k_set_last64<<<1, 1, 0, G.s>>>(h->d_rp, nk, m);
        e = cudaGetLastError();
    }
    if (!e) e = cudaStreamSynchronize(G.s);
    if (e) {
        cudaFree(h->d_rp);
        cudaFree(h->d_col);
        cudaFree(h->d_val);
        cudaFree(h->d_deg);
        cudaFree(h->d_orig);
        delete h;
        return fail(e == cudaErrorMemoryAllocation ? SC_E_OOM : SC_E_CUDA, "generator output: %s",
                    cudaGetErrorString(e));
    }
    *out = h;
    return SC_OK;
}

static int32_t gen_begin(GenCtx &G, int device) {
    int ndev = 0;
    SC_CUDA(cudaGetDeviceCount(&ndev));
    SC_REQUIRE(device >= 0 && device < ndev, SC_E_INVALID, "device %d not present", device);
    SC_CUDA(cudaSetDevice(device));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    G.grid = sms * 8;
    SC_CUDA(cudaStreamCreateWithFlags(&G.s, cudaStreamNonBlocking));
    return SC_OK;
}

}  // namespace sc

extern "C" {

int32_t sc_generate_knn3d(int64_t n, int32_t k, double sigma, int32_t knn, double scale,
                          uint64_t key0, uint64_t key1, int32_t device, sc_csr **out) {
    using namespace sc;
    SC_REQUIRE(out, SC_E_INVALID, "out is null");
    *out = nullptr;
    SC_REQUIRE(n >= 2 && n < (int64_t(1) << 31) - 1, SC_E_INVALID, "n=%lld out of range", (long long)n);
    SC_REQUIRE(k >= 1, SC_E_INVALID, "k must be >= 1");
    SC_REQUIRE(knn == 16 && n > knn, SC_E_INVALID, "knn must be 16 and below n (got %d)", knn);
    SC_REQUIRE(sigma >= 0.0 && scale > 0.0, SC_E_INVALID, "need sigma >= 0 and scale > 0");
    GenCtx G;
    int32_t st = gen_begin(G, device);
    if (st) return st;
    double *px = G.alloc<double>(n), *py = G.alloc<double>(n), *pz = G.alloc<double>(n);
    int32_t *plab = G.alloc<int32_t>(n);
    if (!G.e) {
        k_knn_points<<<G.grid, 256, 0, G.s>>>(n, k, sigma, key0, key1, px, py, pz, plab);
        G.e = cudaGetLastError();
    }
    // bounding box and grid (about two points per cell)
    double *mm = G.alloc<double>(6);
    for (int ax = 0; ax < 3 && !G.e; ++ax) {
        const double *v = ax == 0 ? px : ax == 1 ? py : pz;
        size_t b = 0;
        G.e = cub::DeviceReduce::Min(nullptr, b, v, mm + 2 * ax, n, G.s);
        void *t = G.need(b);
        if (!G.e) G.e = cub::DeviceReduce::Min(t, b, v, mm + 2 * ax, n, G.s);
        if (!G.e) G.e = cub::DeviceReduce::Max(t, b, v, mm + 2 * ax + 1, n, G.s);
    }
    double hmm[6] = {0, 0, 0, 0, 0, 0};
    if (!G.e) G.e = cudaMemcpyAsync(hmm, mm, 48, cudaMemcpyDeviceToHost, G.s);
    if (!G.e) G.e = cudaStreamSynchronize(G.s);
    GridBox gb;
    gb.G = std::max(1, std::min(1024, (int)std::cbrt((double)n / 2.0)));
    for (int ax = 0; ax < 3; ++ax) {
        const double span = std::max(hmm[2 * ax + 1] - hmm[2 * ax], 1e-300);
        gb.lo[ax] = hmm[2 * ax];
        gb.w[ax] = span / gb.G;
        gb.inv[ax] = gb.G / span;
    }
    const int64_t ncell = (int64_t)gb.G * gb.G * gb.G;
    uint32_t *cell = G.alloc<uint32_t>(n), *cell_s = G.alloc<uint32_t>(n);
    int32_t *iota = G.alloc<int32_t>(n), *order = G.alloc<int32_t>(n);
    int32_t *start = G.alloc<int32_t>(ncell + 1);
    if (!G.e) {
        k_knn_cells<<<G.grid, 256, 0, G.s>>>(n, gb, px, py, pz, cell, iota);
        G.e = cudaGetLastError();
    }
    int cbits = 1;
    while ((int64_t(1) << cbits) < ncell) ++cbits;
    if (!G.e) {
        size_t b = 0;
        G.e = cub::DeviceRadixSort::SortPairs(nullptr, b, cell, cell_s, iota, order, n, 0, cbits, G.s);
        void *t = G.need(b);
        if (!G.e) G.e = cub::DeviceRadixSort::SortPairs(t, b, cell, cell_s, iota, order, n, 0, cbits, G.s);
    }
    if (!G.e) {
        k_cell_starts<<<G.grid, 256, 0, G.s>>>(n, cell_s, ncell, start);
        G.e = cudaGetLastError();
    }
    int32_t *nb = G.alloc<int32_t>((size_t)n * 16);
    double *nd2 = G.alloc<double>((size_t)n * 16);
    if (!G.e) {
        k_knn_search<16><<<G.grid, 128, 0, G.s>>>(n, gb, px, py, pz, order, start, nb, nd2);
        G.e = cudaGetLastError();
    }
    // both directions of every pair, sorted, unique
    const int64_t m2 = 2 * 16 * n;
    uint64_t *key = G.alloc<uint64_t>(m2);
    double *w = G.alloc<double>(m2);
    if (!G.e) {
        k_knn_pairs<<<G.grid, 256, 0, G.s>>>(n, 16, scale, nb, nd2, key, w);
        G.e = cudaGetLastError();
    }
    G.release(nb);
    G.release(nd2);
    int kbits = 32;
    while ((int64_t(1) << (kbits - 32)) < n) ++kbits;
    sort_pairs(G, key, w, m2, kbits);
    int32_t *flag = G.alloc<int32_t>(m2);
    int64_t *pos = G.alloc<int64_t>(m2 + 1);
    if (!G.e) {
        k_unique_flags<<<G.grid, 256, 0, G.s>>>(m2, key, flag);
        G.e = cudaGetLastError();
    }
    excl_scan(G, flag, pos, m2);
    const int64_t m = fetch(G, pos + m2 - 1) + fetch(G, flag + m2 - 1);
    uint64_t *ukey = G.alloc<uint64_t>(m);
    double *uw = G.alloc<double>(m);
    if (!G.e) {
        k_unique_copy<<<G.grid, 256, 0, G.s>>>(m2, key, w, flag, pos, ukey, uw);
        G.e = cudaGetLastError();
    }
    if (G.e)
        return fail(G.e == cudaErrorMemoryAllocation ? SC_E_OOM : SC_E_CUDA, "knn3d: %s",
                    cudaGetErrorString(G.e));
    return assemble(G, n, ukey, uw, m, device, out);
}

int32_t sc_generate_dcsbm(int64_t n, const int64_t *block_offsets, int32_t nblocks, double A,
                          double B, double inv_a, int32_t dmin, int32_t dmax, double mix,
                          double wlo, double whi, uint64_t key0, uint64_t key1, int32_t device,
                          sc_csr **out) {
    using namespace sc;
    SC_REQUIRE(out && block_offsets, SC_E_INVALID, "null argument");
    *out = nullptr;
    SC_REQUIRE(n >= 2 && n < (int64_t(1) << 31) - 1, SC_E_INVALID, "n=%lld out of range", (long long)n);
    SC_REQUIRE(nblocks >= 1, SC_E_INVALID, "need at least one block");
    SC_REQUIRE(block_offsets[0] == 0 && block_offsets[nblocks] == n, SC_E_INVALID,
               "block offsets must run from 0 to n");
    for (int b = 0; b < nblocks; ++b)
        SC_REQUIRE(block_offsets[b + 1] > block_offsets[b], SC_E_INVALID, "empty block %d", b);
    SC_REQUIRE(1 <= dmin && dmin <= dmax, SC_E_INVALID, "need 1 <= dmin <= dmax");
    SC_REQUIRE(0.0 <= mix && mix <= 1.0 && wlo > 0.0 && whi >= wlo, SC_E_INVALID,
               "need 0 <= mix <= 1 and 0 < wlo <= whi");
    GenCtx G;
    int32_t st = gen_begin(G, device);
    if (st) return st;
    int64_t *boff = G.alloc<int64_t>(nblocks + 1);
    if (!G.e) G.e = cudaMemcpyAsync(boff, block_offsets, (size_t)(nblocks + 1) * 8,
                                    cudaMemcpyHostToDevice, G.s);
    int64_t *deg = G.alloc<int64_t>(n), *stubs = G.alloc<int64_t>(n);
    int64_t *cum = G.alloc<int64_t>(n), *soff = G.alloc<int64_t>(n + 1);
    if (!G.e) {
        k_dc_degrees<<<G.grid, 256, 0, G.s>>>(n, A, B - A, inv_a, dmin, dmax, key0, key1, deg, stubs);
        G.e = cudaGetLastError();
    }
    if (!G.e) {  // inclusive prefix of the integer degrees
        size_t b = 0;
        G.e = cub::DeviceScan::InclusiveSum(nullptr, b, deg, cum, n, G.s);
        void *t = G.need(b);
        if (!G.e) G.e = cub::DeviceScan::InclusiveSum(t, b, deg, cum, n, G.s);
    }
    excl_scan(G, stubs, soff, n);
    const int64_t ns = fetch(G, soff + n - 1) + fetch(G, stubs + n - 1);
    uint64_t *key = G.alloc<uint64_t>(ns);
    double *w = G.alloc<double>(ns);
    if (!G.e) {
        k_dc_stubs<<<G.grid, 256, 0, G.s>>>(n, boff, nblocks, mix, wlo, whi - wlo, key0, key1, cum,
                                            soff, stubs, key, w);
        G.e = cudaGetLastError();
    }
    int kbits = 32;
    while ((int64_t(1) << (kbits - 32)) < n) ++kbits;
    sort_pairs(G, key, w, ns, 64);  // ~0 (self loops) sorts last
    int32_t *flag = G.alloc<int32_t>(ns);
    int64_t *pos = G.alloc<int64_t>(ns + 1);
    if (!G.e) {
        k_unique_flags<<<G.grid, 256, 0, G.s>>>(ns, key, flag);
        G.e = cudaGetLastError();
    }
    excl_scan(G, flag, pos, ns);
    const int64_t mu = fetch(G, pos + ns - 1) + fetch(G, flag + ns - 1);
    uint64_t *k2 = G.alloc<uint64_t>(2 * mu);
    double *w2 = G.alloc<double>(2 * mu);
    if (!G.e) {
        k_unique_both<<<G.grid, 256, 0, G.s>>>(ns, key, w, flag, pos, k2, w2);
        G.e = cudaGetLastError();
    }
    G.release(key);
    G.release(w);
    sort_pairs(G, k2, w2, 2 * mu, kbits);
    if (G.e)
        return fail(G.e == cudaErrorMemoryAllocation ? SC_E_OOM : SC_E_CUDA, "dcsbm: %s",
                    cudaGetErrorString(G.e));
    return assemble(G, n, k2, w2, 2 * mu, device, out);
}

}  // extern "C"
