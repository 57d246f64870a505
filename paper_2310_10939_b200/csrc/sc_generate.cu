// sc_generate.cu -- device generator for the planted-partition graphs of the benchmark
// configs too large for the host (config 5: n = 1e8, ~1.8e9 stored
// entries), and the device-resident CSR handle that feeds sc_graph_create_from_csr without a
// host round trip of the column array.
//
// Law (the reference's SBM, specluster/generate.py:112-149): vertices in k consecutive blocks
// of s = n/k; every pair u < v is an edge independently with probability p (same block) or q
// (different blocks); no self loops; unit weights; isolated vertices are dropped and the
// remaining ids compacted (generate.py:137).  The realisation is ours (the reference's
// per-block-pair numpy streams cannot be replayed at 5e5 block pairs): row u walks its
// upper-triangle candidates v > u with geometric skips, first inside its block (prob p), then
// over the later blocks (prob q).  Skip j of row u uses word j%4 of
// Philox4x64-10(key, (j/4 + 1, u, kGenTag, 0)) -- numpy.random.Philox(key, counter=[0, u,
// kGenTag, 0]) reproduces the stream -- as U = (raw >> 11 + 1) * 2^-53 in (0, 1], and
// G = 1 + floor(sc_log(U) * inv_log1m), inv_log1m = 1 / log1p(-prob) computed by the caller.
// sc_log uses only correctly rounded +,-,*,/ so the host oracle (numpy, same op sequence)
// reproduces every skip bit for bit.
//
// Assembly: count pass -> scan -> fill pass (upper lists, row-major, sorted) -> stable radix
// sort of the transposed pairs by column (gives every row's lower neighbours in ascending
// order) -> row = lower ++ upper (already globally sorted) -> drop isolated rows, compact ids.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <vector>

#include "sc_common.cuh"

#include "sc_csr.cuh"
#include "sc_genmath.cuh"

namespace sc {

constexpr uint64_t kGenTag = 0x5bd1e995u;

struct RowStream {
    uint64_t u, k0, k1;
    uint64_t blk = 0;
    int idx = 4;
    uint64_t w[4];
    __device__ uint64_t next() {
        if (idx == 4) {
            const u64x4 r = philox4x64_10(u64x4{blk + 1, u, kGenTag, 0}, k0, k1);
            w[0] = r.x;
            w[1] = r.y;
            w[2] = r.z;
            w[3] = r.w;
            idx = 0;
            ++blk;
        }
        return w[idx++];
    }
    // geometric skip >= 1 (returns a huge value for prob 0: inv = -0.0 -> caller's bound)
    __device__ int64_t skip(double inv_log1m) {
        const double U = (double)((next() >> 11) + 1) * 1.1102230246251565e-16;
        const double g = floor(sc_log(U) * inv_log1m);
        return g >= 4.0e18 ? INT64_MAX / 2 : 1 + (int64_t)g;
    }
};

// count (FILL = false) or write (FILL = true) the upper neighbours of every row
template <bool FILL>
__global__ void k_sbm_upper(int64_t n, int64_t s, double inv_p, double inv_q, int has_p,
                            int has_q, uint64_t k0, uint64_t k1, int32_t *__restrict__ cnt,
                            const int64_t *__restrict__ ptr, int32_t *__restrict__ col,
                            int32_t *__restrict__ src, int32_t *__restrict__ lowcnt) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        RowStream rs{(uint64_t)u, k0, k1};
        const int64_t hi = (u / s + 1) * s;
        int64_t c = 0, o = FILL ? ptr[u] : 0;
        auto emit = [&](int64_t v) {
            if (FILL) {
                col[o + c] = (int32_t)v;
                src[o + c] = (int32_t)u;
                atomicAdd(&lowcnt[v], 1);
            }
            ++c;
        };
        if (has_p)
            for (int64_t v = u + rs.skip(inv_p); v < hi; v += rs.skip(inv_p)) emit(v);
        if (has_q)
            for (int64_t v = hi - 1 + rs.skip(inv_q); v < n; v += rs.skip(inv_q)) emit(v);
        if (!FILL) cnt[u] = (int32_t)c;
    }
}

__global__ void k_keep(int64_t n, const int32_t *__restrict__ up, const int32_t *__restrict__ low,
                       int64_t *__restrict__ deg64, int32_t *__restrict__ keep) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = (int64_t)up[u] + low[u];
        deg64[u] = d;
        keep[u] = d > 0;
    }
}

// row u (kept) = lower neighbours (sorted transposed pairs) ++ upper neighbours, renamed
__global__ void k_assemble(int64_t n, const int32_t *__restrict__ up, const int64_t *__restrict__ up_ptr,
                           const int32_t *__restrict__ up_col, const int32_t *__restrict__ low,
                           const int64_t *__restrict__ low_ptr, const int32_t *__restrict__ low_src,
                           const int64_t *__restrict__ full_ptr, const int32_t *__restrict__ newid,
                           const int32_t *__restrict__ keep, int64_t *__restrict__ rp,
                           int32_t *__restrict__ col, double *__restrict__ deg,
                           int32_t *__restrict__ orig) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        if (!keep[u]) continue;
        const int32_t id = newid[u];
        const int64_t b = full_ptr[u];
        const int32_t nl = low[u], nu = up[u];
        rp[id] = b;
        deg[id] = (double)(nl + nu);
        orig[id] = (int32_t)u;
        const int64_t lp = low_ptr[u], upp = up_ptr[u];
        for (int32_t i = 0; i < nl; ++i) col[b + i] = newid[low_src[lp + i]];
        for (int32_t i = 0; i < nu; ++i) col[b + nl + i] = newid[up_col[upp + i]];
    }
}

__global__ void k_set_last(int64_t *rp, int64_t idx, int64_t v) { rp[idx] = v; }

template <typename T>
static cudaError_t dalloc(T **p, size_t count, cudaStream_t s) {
    return cudaMallocAsync((void **)p, std::max<size_t>(count, 1) * sizeof(T), s);
}

}  // namespace sc

extern "C" {

int32_t sc_generate_sbm(int64_t n, int32_t k, double p, double q, double inv_log1m_p,
                        double inv_log1m_q, uint64_t key0, uint64_t key1, int32_t device,
                        sc_csr **out) {
    using namespace sc;
    SC_REQUIRE(out, SC_E_INVALID, "out is null");
    *out = nullptr;
    SC_REQUIRE(n >= 1 && n < (int64_t(1) << 31) - 1, SC_E_INVALID, "n=%lld out of range",
               (long long)n);
    SC_REQUIRE(k >= 1 && n % k == 0, SC_E_INVALID, "k must divide n (n=%lld, k=%d)",
               (long long)n, k);
    SC_REQUIRE(0.0 <= q && q <= p && p <= 1.0, SC_E_INVALID, "need 0 <= q <= p <= 1");
    int ndev = 0;
    SC_CUDA(cudaGetDeviceCount(&ndev));
    SC_REQUIRE(device >= 0 && device < ndev, SC_E_INVALID, "device %d not present", device);
    SC_CUDA(cudaSetDevice(device));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int grid = sms * 8;
    cudaStream_t s;
    SC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const int64_t bs = n / k;
    const int has_p = p > 0.0 && bs > 1, has_q = q > 0.0 && k > 1;
    int32_t *up = nullptr, *low = nullptr, *up_col = nullptr, *up_src = nullptr,
            *low_src = nullptr, *keys_sorted = nullptr, *keep = nullptr, *newid = nullptr;
    int64_t *up_ptr = nullptr, *low_ptr = nullptr, *deg64 = nullptr, *full_ptr = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    sc_csr *h = new sc_csr();
    h->device = device;
    h->n_gen = n;
    auto cleanup = [&](int32_t code) {
        for (void *ptr : {(void *)up, (void *)low, (void *)up_col, (void *)up_src,
                          (void *)low_src, (void *)keys_sorted, (void *)keep, (void *)newid,
                          (void *)up_ptr, (void *)low_ptr, (void *)deg64, (void *)full_ptr,
                          tmp})
            if (ptr) cudaFreeAsync(ptr, s);
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
        return code;
    };
    auto need_tmp = [&](size_t b) -> cudaError_t {
        if (b <= tmp_bytes) return cudaSuccess;
        if (tmp) cudaFreeAsync(tmp, s);
        tmp_bytes = b;
        return cudaMallocAsync(&tmp, b, s);
    };
    cudaError_t e = dalloc(&up, n, s);
    if (!e) e = dalloc(&low, n, s);
    if (!e) e = dalloc(&up_ptr, n + 1, s);
    if (!e) e = cudaMemsetAsync(low, 0, (size_t)n * 4, s);
    if (!e) {
        k_sbm_upper<false><<<grid, 256, 0, s>>>(n, bs, inv_log1m_p, inv_log1m_q, has_p, has_q,
                                                key0, key1, up, nullptr, nullptr, nullptr,
                                                nullptr);
        e = cudaGetLastError();
    }
    // exclusive scan of the int32 counts into int64 offsets (+ total at [n])
    size_t b = 0;
    if (!e) e = cub::DeviceScan::ExclusiveSum(nullptr, b, up, up_ptr, n, s);
    if (!e) e = need_tmp(b);
    if (!e) e = cub::DeviceScan::ExclusiveSum(tmp, b, up, up_ptr, n, s);
    int64_t last_ptr = 0;
    int32_t last_cnt = 0;
    if (!e) e = cudaMemcpyAsync(&last_ptr, up_ptr + n - 1, 8, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaMemcpyAsync(&last_cnt, up + n - 1, 4, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) {
        delete h;
        fail(e == cudaErrorMemoryAllocation ? SC_E_OOM : SC_E_CUDA, "sbm count: %s",
             cudaGetErrorString(e));
        return cleanup(e == cudaErrorMemoryAllocation ? SC_E_OOM : SC_E_CUDA);
    }
    const int64_t m = last_ptr + last_cnt;  // upper-triangle edges
    if (m > (int64_t(1) << 31) - 1) {
        delete h;
        fail(SC_E_RANGE, "too many edges (%lld)", (long long)m);
        return cleanup(SC_E_RANGE);
    }
    e = dalloc(&up_col, m, s);
    if (!e) e = dalloc(&up_src, m, s);
    if (!e) {
        k_sbm_upper<true><<<grid, 256, 0, s>>>(n, bs, inv_log1m_p, inv_log1m_q, has_p, has_q,
                                               key0, key1, nullptr, up_ptr, up_col, up_src, low);
        e = cudaGetLastError();
    }
    // transposed pairs (col, src) stably sorted by col: lower neighbours, ascending
    int end_bit = 1;
    while ((int64_t(1) << end_bit) < n) ++end_bit;
    if (!e) e = dalloc(&keys_sorted, m, s);
    if (!e) e = dalloc(&low_src, m, s);
    if (!e) e = cub::DeviceRadixSort::SortPairs(nullptr, b, up_col, keys_sorted, up_src, low_src,
                                                (int)m, 0, end_bit, s);
    if (!e) e = need_tmp(b);
    if (!e) e = cub::DeviceRadixSort::SortPairs(tmp, b, up_col, keys_sorted, up_src, low_src,
                                                (int)m, 0, end_bit, s);
    if (keys_sorted) cudaFreeAsync(keys_sorted, s);
    keys_sorted = nullptr;
    if (up_src) cudaFreeAsync(up_src, s);
    up_src = nullptr;
    if (!e) e = dalloc(&low_ptr, n + 1, s);
    if (!e) e = cub::DeviceScan::ExclusiveSum(nullptr, b, low, low_ptr, n, s);
    if (!e) e = need_tmp(b);
    if (!e) e = cub::DeviceScan::ExclusiveSum(tmp, b, low, low_ptr, n, s);
    // degrees, kept rows, new ids, row offsets of the full rows
    if (!e) e = dalloc(&deg64, n, s);
    if (!e) e = dalloc(&keep, n, s);
    if (!e) e = dalloc(&newid, n, s);
    if (!e) e = dalloc(&full_ptr, n, s);
    if (!e) {
        k_keep<<<grid, 256, 0, s>>>(n, up, low, deg64, keep);
        e = cudaGetLastError();
    }
    if (!e) e = cub::DeviceScan::ExclusiveSum(nullptr, b, deg64, full_ptr, n, s);
    if (!e) e = need_tmp(b);
    if (!e) e = cub::DeviceScan::ExclusiveSum(tmp, b, deg64, full_ptr, n, s);
    if (!e) e = cub::DeviceScan::ExclusiveSum(nullptr, b, keep, newid, n, s);
    if (!e) e = need_tmp(b);
    if (!e) e = cub::DeviceScan::ExclusiveSum(tmp, b, keep, newid, n, s);
    int32_t last_id = 0, last_keep = 0;
    if (!e) e = cudaMemcpyAsync(&last_id, newid + n - 1, 4, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaMemcpyAsync(&last_keep, keep + n - 1, 4, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    const int64_t nk = (int64_t)last_id + last_keep, nnz = 2 * m;
    if (!e && nk == 0) {
        delete h;
        fail(SC_E_INVALID, "the sampled graph has no edges");
        return cleanup(SC_E_INVALID);
    }
    if (!e) e = cudaMalloc((void **)&h->d_rp, (size_t)(nk + 1) * 8);
    if (!e) e = cudaMalloc((void **)&h->d_col, (size_t)std::max<int64_t>(nnz, 1) * 4);
    if (!e) e = cudaMalloc((void **)&h->d_deg, (size_t)nk * 8);
    if (!e) e = cudaMalloc((void **)&h->d_orig, (size_t)nk * 4);
    if (!e) {
        k_assemble<<<grid, 256, 0, s>>>(n, up, up_ptr, up_col, low, low_ptr, low_src, full_ptr,
                                        newid, keep, h->d_rp, h->d_col, h->d_deg, h->d_orig);
        k_set_last<<<1, 1, 0, s>>>(h->d_rp, nk, nnz);
        e = cudaGetLastError();
    }
    if (!e) e = cudaStreamSynchronize(s);
    if (e) {
        cudaFree(h->d_rp);
        cudaFree(h->d_col);
        cudaFree(h->d_deg);
        cudaFree(h->d_orig);
        delete h;
        fail(e == cudaErrorMemoryAllocation ? SC_E_OOM : SC_E_CUDA, "sbm assembly: %s",
             cudaGetErrorString(e));
        return cleanup(e == cudaErrorMemoryAllocation ? SC_E_OOM : SC_E_CUDA);
    }
    h->n = nk;
    h->nnz = nnz;
    *out = h;
    return cleanup(SC_OK);
}

int32_t sc_csr_info(const sc_csr *h, int64_t *n, int64_t *nnz, int64_t *n_generated) {
    SC_REQUIRE(h, SC_E_INVALID, "null csr");
    if (n) *n = h->n;
    if (nnz) *nnz = h->nnz;
    if (n_generated) *n_generated = h->n_gen;
    return SC_OK;
}

int32_t sc_csr_download_weights(const sc_csr *h, double *val) {
    SC_REQUIRE(h && val, SC_E_INVALID, "null argument");
    SC_REQUIRE(h->d_val, SC_E_STATE, "the CSR has unit weights");
    SC_CUDA(cudaSetDevice(h->device));
    if (h->nnz) SC_CUDA(cudaMemcpy(val, h->d_val, (size_t)h->nnz * 8, cudaMemcpyDeviceToHost));
    return SC_OK;
}

int32_t sc_csr_download(const sc_csr *h, int64_t *row_ptr, int32_t *col, double *deg,
                        int32_t *orig_ids) {
    SC_REQUIRE(h, SC_E_INVALID, "null csr");
    SC_CUDA(cudaSetDevice(h->device));
    if (row_ptr) SC_CUDA(cudaMemcpy(row_ptr, h->d_rp, (size_t)(h->n + 1) * 8, cudaMemcpyDeviceToHost));
    if (col && h->nnz) SC_CUDA(cudaMemcpy(col, h->d_col, (size_t)h->nnz * 4, cudaMemcpyDeviceToHost));
    if (deg) SC_CUDA(cudaMemcpy(deg, h->d_deg, (size_t)h->n * 8, cudaMemcpyDeviceToHost));
    if (orig_ids) SC_CUDA(cudaMemcpy(orig_ids, h->d_orig, (size_t)h->n * 4, cudaMemcpyDeviceToHost));
    return SC_OK;
}

void sc_csr_destroy(sc_csr *h) {
    if (!h) return;
    cudaSetDevice(h->device);
    cudaFree(h->d_rp);
    cudaFree(h->d_col);
    cudaFree(h->d_deg);
    cudaFree(h->d_orig);
    if (h->d_val) cudaFree(h->d_val);
    delete h;
}

}  // extern "C"

namespace sc {
// device-side view for sc_graph_create_from_csr (sc_graph.cu)
int32_t csr_device_arrays(const sc_csr *h, const int64_t **rp, const int32_t **col,
                          const double **deg, const double **val, int32_t *device) {
    SC_REQUIRE(h, SC_E_INVALID, "null csr");
    *val = h->d_val;
    *rp = h->d_rp;
    *col = h->d_col;
    *deg = h->d_deg;
    *device = h->device;
    return SC_OK;
}
}  // namespace sc
