// dsmem_bench.cu -- random 8-byte gathers served from a thread-block cluster's distributed
// shared memory vs from L2.  A window of W doubles (one SBM block of z) is spread over the
// cluster's CTAs; every thread gathers z[c] for random c in the window.
// Usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bench dsmem_bench.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); \
            return 1;                                                           \
        }                                                                       \
    } while (0)

// each cluster handles windows w = cluster_id, cluster_id + nclusters, ...; per window it
// loads z[w*W .. (w+1)*W) spread over its CTAs, then gathers `per_win` random entries.
template <int CS>
__global__ void k_dsmem(const double *z, const int *idx, int64_t per_win, int nwin, int W,
                        double *out) {
    extern __shared__ double slice[];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = cl.block_rank();
    const int nclus = gridDim.x / CS;
    const int cid = blockIdx.x / CS;
    const int sl = (W + CS - 1) / CS;
    double acc = 0.0;
    for (int w = cid; w < nwin; w += nclus) {
        for (int i = threadIdx.x; i < sl; i += blockDim.x) {
            const int64_t g = (int64_t)w * W + (int64_t)rank * sl + i;
            slice[i] = (rank * sl + i < W) ? z[g] : 0.0;
        }
        cl.sync();
        const int *my = idx + (int64_t)w * per_win;
        const int64_t per_cta = per_win / CS;
        const int *mine = my + rank * per_cta;
        for (int64_t j = threadIdx.x; j < per_cta; j += 4 * blockDim.x) {
            int c[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) c[q] = j + q * blockDim.x < per_cta ? __ldcs(mine + j + q * blockDim.x) : 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int r = c[q] / sl, o = c[q] - r * sl;
                const double *p = cl.map_shared_rank(slice, r);
                acc += p[o];
            }
        }
        cl.sync();
    }
    if (acc == -1.0) out[0] = acc;
}

__global__ void k_l2(const double *z, const int *idx, int64_t per_win, int nwin, int W, double *out) {
    double acc = 0.0;
    const int64_t tot = per_win * nwin;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < tot; j += 4 * (int64_t)gridDim.x * blockDim.x) {
        int c[4];
        int64_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t jj = j + q * (int64_t)gridDim.x * blockDim.x;
            c[q] = jj < tot ? __ldcs(idx + jj) : 0;
            w[q] = jj < tot ? jj / per_win : 0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) acc += __ldg(z + w[q] * W + c[q]);
    }
    if (acc == -1.0) out[0] = acc;
}

template <int CS>
int run(const double *dz, const int *didx, int64_t per_win, int nwin, int W, double *dout, int sms) {
    const int sl = (W + CS - 1) / CS;
    const size_t smem = (size_t)sl * 8;
    auto kern = k_dsmem<CS>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (CS > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    const int nclus = sms / CS;
    cfg.gridDim = dim3(nclus * CS);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 2; ++i) CK(cudaLaunchKernelEx(&cfg, kern, dz, didx, per_win, nwin, W, dout));
    cudaEventRecord(e0);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) cudaLaunchKernelEx(&cfg, kern, dz, didx, per_win, nwin, W, dout);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double g = (double)per_win * nwin;
    printf("dsmem CS=%2d clusters=%3d smem/CTA=%6zu B: %8.1f us  %7.1f Ggather/s\n", CS, nclus, smem,
           ms * 1e3, g / ms / 1e6);
    return 0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int W = 100000, nwin = 10;
    const int64_t per_win = 4000000;  // 40 in-block gathers x 1e5 rows
    std::vector<int> idx((size_t)per_win * nwin);
    uint64_t s = 88172645463325252ULL;
    for (auto &v : idx) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        v = (int)(s % W);
    }
    double *dz, *dout;
    int *didx;
    CK(cudaMalloc(&dz, (size_t)W * nwin * 8));
    CK(cudaMalloc(&dout, 64));
    CK(cudaMalloc(&didx, idx.size() * 4));
    CK(cudaMemcpy(didx, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(dz, 0, (size_t)W * nwin * 8));
    run<8>(dz, didx, per_win, nwin, W, dout, sms);
    run<16>(dz, didx, per_win, nwin, W, dout, sms);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 2; ++i) k_l2<<<sms * 4, 512>>>(dz, didx, per_win, nwin, W, dout);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) k_l2<<<sms * 4, 512>>>(dz, didx, per_win, nwin, W, dout);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 10;
    printf("l2 gathers: %8.1f us  %7.1f Ggather/s\n", ms * 1e3, per_win * nwin / ms / 1e6);
    return 0;
}
