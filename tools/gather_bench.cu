// gather_bench.cu -- ceiling measurements for the SpMV's random gathers on one B200.
//
// Builds an SBM-like column array like config 2 (n = 1e6 rows, blocks of 1e5, 40 random
// in-block + 4 random out-of-block neighbours per row, sorted per row), then times:
//   copy      : HBM copy of the col array (read+write bytes)        -> streaming ceiling
//   stream    : read col only (sum of indices)                      -> HBM read ceiling
//   gather    : acc += z[col[j]] over all j, lane-linear            -> gather ceiling (L1 path)
//   gather_na : same with ld.global.nc.L1::no_allocate gathers
//   gather_u4 : 4 gathers per thread from one int4 col load
// Usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e = (x);                                                      \
        if (e != cudaSuccess) {                                                   \
            printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e));   \
            return 1;                                                             \
        }                                                                         \
    } while (0)

__global__ void k_copy(const int4 *a, int4 *b, int64_t n4) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = __ldcs(a + i);
}

__global__ void k_stream(const int *col, int64_t nnz, double *out) {
    int64_t acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
        acc += __ldcs(col + i);
    if (acc == 42) out[0] = 1.0;
}

template <int MODE>
__global__ void k_gather(const int *col, const double *z, int64_t nnz, double *out) {
    double acc = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < nnz; i += 4 * stride) {
        int c[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = __ldcs(col + i + q * stride);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double v;
            if (MODE == 0) v = __ldg(z + c[q]);
            else asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(z + c[q]));
            acc += v;
        }
    }
    for (; i < nnz; i += stride) acc += __ldg(z + __ldcs(col + i));
    if (acc == -1.0) out[0] = acc;
}

int main() {
    const int64_t n = 1000000, blk = 100000;
    std::vector<int> col;
    col.reserve(n * 44);
    uint64_t s = 0x9E3779B97F4A7C15ULL;
    auto rnd = [&]() {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        return s;
    };
    std::vector<int> row;
    for (int64_t i = 0; i < n; ++i) {
        row.clear();
        const int64_t b = i / blk;
        for (int t = 0; t < 40; ++t) row.push_back((int)(b * blk + rnd() % blk));
        for (int t = 0; t < 4; ++t) row.push_back((int)(rnd() % n));
        std::sort(row.begin(), row.end());
        col.insert(col.end(), row.begin(), row.end());
    }
    const int64_t nnz = (int64_t)col.size();
    int *dcol, *dcol2;
    double *dz, *dout;
    CK(cudaMalloc(&dcol, nnz * 4 + 64));
    CK(cudaMalloc(&dcol2, nnz * 4 + 64));
    CK(cudaMalloc(&dz, n * 8));
    CK(cudaMalloc(&dout, 64));
    CK(cudaMemcpy(dcol, col.data(), nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(dz, 0, n * 8));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char *name, auto fn, double bytes, double gathers) {
        for (int w = 0; w < 3; ++w) fn();
        cudaEventRecord(e0);
        const int reps = 20;
        for (int r = 0; r < reps; ++r) fn();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= reps;
        printf("%-12s %9.1f us  %8.1f GB/s  %8.1f Ggather/s\n", name, ms * 1e3, bytes / ms / 1e6,
               gathers / ms / 1e6);
    };
    for (int tpb : {256, 512, 1024}) {
        for (int mult : {4, 8, 16}) {
            const int grid = sms * mult * 256 / tpb;
            printf("-- tpb %d grid %d (x%d)\n", tpb, grid, mult);
            timeit("gather", [&] { k_gather<0><<<grid, tpb>>>(dcol, dz, nnz, dout); }, nnz * 4.0, (double)nnz);
            timeit("gather_na", [&] { k_gather<1><<<grid, tpb>>>(dcol, dz, nnz, dout); }, nnz * 4.0, (double)nnz);
        }
    }
    const int grid = sms * 8;
    timeit("copy", [&] { k_copy<<<grid, 256>>>((const int4 *)dcol, (int4 *)dcol2, nnz / 4); }, nnz * 8.0, 0);
    timeit("stream", [&] { k_stream<<<grid, 256>>>(dcol, nnz, dout); }, nnz * 4.0, 0);
    CK(cudaGetLastError());
    printf("nnz=%lld\n", (long long)nnz);
    return 0;
}
