// tma_gather_bench.cu -- can the TMA engine serve the SpMV's random 8-byte gathers faster than
// the LSU/L1 request path (~288 G gathers/s measured by gather_bench.cu)?
//
// Same synthetic column array as gather_bench.cu (config-2 shaped: 1e6 rows, 40 in-block +
// 4 random neighbours).  Variants, all summing z[col[j]] over 44M entries:
//   ldg      : __ldg gathers (baseline)
//   cg       : ld.global.cg gathers (L2 only)
//   bulk16   : per-lane cp.async.bulk global->shared of the 16-byte pair holding z[c],
//              completion on a per-stage mbarrier, 4-stage pipeline per warp
//   gather4  : cp.async.bulk.tensor.2d ... tile::gather4 of four 16-byte rows of z viewed as
//              [n/2][2] doubles (one instruction per 4 gathers), same pipeline
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_gather_bench
//        tma_gather_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); \
            return 1;                                                           \
        }                                                                       \
    } while (0)

template <int CG>
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
            if (CG) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(z + c[q]));
            else v = __ldg(z + c[q]);
            acc += v;
        }
    }
    for (; i < nnz; i += stride) acc += __ldg(z + __ldcs(col + i));
    if (acc == -1.0) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *m, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t *m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}\n" ::"r"(smem_u32(m)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk16(void *dst, const void *src, uint64_t *m) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(smem_u32(m))
        : "memory");
}
__device__ __forceinline__ void gather4(void *dst, const CUtensorMap *tm, int r0, int r1, int r2,
                                        int r3, uint64_t *m) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(m))
        : "memory");
}

// one warp streams a contiguous range of entries; per stage every lane moves E entries
constexpr int E = 4, STAGES = 2, WPB = 4, LS = 16;  // LS: doubles per lane slot (128 B)

template <int MODE>  // 0 bulk16, 1 gather4
__global__ void __launch_bounds__(32 * WPB) k_tma(const int *col, const double *z,
                                                  const __grid_constant__ CUtensorMap tm,
                                                  int64_t nnz, double *out) {
    __shared__ alignas(128) double buf[WPB][STAGES][32 * LS];
    __shared__ uint64_t bar[WPB][STAGES];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t nw = (int64_t)gridDim.x * WPB, gw = (int64_t)blockIdx.x * WPB + w;
    const int64_t per = 32 * E;  // entries per stage
    const int64_t chunks = (nnz + per - 1) / per;
    if (lane == 0)
        for (int s = 0; s < STAGES; ++s) mbar_init(&bar[w][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    double acc = 0.0;
    int cs[STAGES][E];
    auto issue = [&](int64_t ch, int s) {
        const int64_t b = ch * per;
        if (lane == 0) mbar_expect(&bar[w][s], (uint32_t)(per * 16));
        __syncwarp();
        if (MODE == 0) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int64_t j = b + e * 32 + lane;
                const int c = j < nnz ? __ldcs(col + j) : 0;
                cs[s][e] = c;
                bulk16(&buf[w][s][lane * LS + e * 2], z + (c & ~1), &bar[w][s]);
            }
        } else {
            // lane handles 4 consecutive entries -> one gather4 of 4 rows
            int c4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int64_t j = b + lane * 4 + e;
                c4[e] = j < nnz ? __ldcs(col + j) : 0;
                cs[s][e] = c4[e];
            }
            gather4(&buf[w][s][lane * LS], &tm, c4[0] >> 1, c4[1] >> 1, c4[2] >> 1, c4[3] >> 1,
                    &bar[w][s]);
        }
    };
    int64_t ch = gw;
    int issued = 0;
    for (int s = 0; s < STAGES && ch + (int64_t)s * nw < chunks; ++s) {
        issue(ch + (int64_t)s * nw, s);
        ++issued;
    }
    uint32_t phase[STAGES] = {};
    for (int64_t k = 0; ch + k * nw < chunks; ++k) {
        const int s = (int)(k % STAGES);
        mbar_wait(&bar[w][s], phase[s]);
        phase[s] ^= 1;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int c = cs[s][e];
            acc += buf[w][s][lane * LS + e * 2 + (c & 1)];
        }
        __syncwarp();
        const int64_t nxt = ch + (k + STAGES) * nw;
        if (nxt < chunks) issue(nxt, s);
    }
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
    int *dcol;
    double *dz, *dout;
    CK(cudaMalloc(&dcol, nnz * 4 + 64));
    CK(cudaMalloc(&dz, n * 8 + 64));
    CK(cudaMalloc(&dout, 64));
    CK(cudaMemcpy(dcol, col.data(), nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(dz, 0, n * 8));
    // z as a [n/2][2] double tensor: 16-byte rows
    CUtensorMap tm;
    cuuint64_t dims[2] = {2, (cuuint64_t)(n / 2)};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dz, dims, strides,
                                         box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("tensor map encode: %d\n", (int)cr);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char *name, auto fn) {
        for (int w = 0; w < 3; ++w) fn();
        cudaError_t e = cudaDeviceSynchronize();
        if (e) {
            printf("%-10s failed: %s\n", name, cudaGetErrorString(e));
            return;
        }
        cudaEventRecord(e0);
        const int reps = 20;
        for (int r = 0; r < reps; ++r) fn();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= reps;
        printf("%-10s %9.1f us  %8.1f Ggather/s\n", name, ms * 1e3, nnz / ms / 1e6);
    };
    timeit("ldg", [&] { k_gather<0><<<sms * 4, 1024>>>(dcol, dz, nnz, dout); });
    timeit("cg", [&] { k_gather<1><<<sms * 4, 1024>>>(dcol, dz, nnz, dout); });
    for (int mult : {4, 8, 16}) {
        char nm[32];
        snprintf(nm, sizeof nm, "bulk16x%d", mult);
        if (cr == CUDA_SUCCESS) {
            snprintf(nm, sizeof nm, "gather4x%d", mult);
            timeit(nm, [&] { k_tma<1><<<sms * mult, 32 * WPB>>>(dcol, dz, tm, nnz, dout); });
        }
        snprintf(nm, sizeof nm, "bulk16x%d", mult);
        timeit(nm, [&] { k_tma<0><<<sms * mult, 32 * WPB>>>(dcol, dz, tm, nnz, dout); });
    }
    // both paths at once on two streams (are the LSU and TMA request paths independent?)
    cudaStream_t s1, s2;
    cudaEvent_t fork, j1, j2;
    cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&j1, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&j2, cudaEventDisableTiming);
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    for (double f : {0.5, 0.6, 0.7}) {
        int64_t na = ((int64_t)(nnz * f) / 512) * 512;
        char nm[32];
        snprintf(nm, sizeof nm, "hybrid%.1f", f);
        timeit(nm, [&] {  // fork from / join into the legacy stream timeit brackets
            cudaEventRecord(fork, 0);
            cudaStreamWaitEvent(s1, fork, 0);
            cudaStreamWaitEvent(s2, fork, 0);
            k_gather<0><<<sms * 2, 1024, 0, s1>>>(dcol, dz, na, dout);
            k_tma<1><<<sms * 8, 32 * WPB, 0, s2>>>(dcol + na, dz, tm, nnz - na, dout);
            cudaEventRecord(j1, s1);
            cudaEventRecord(j2, s2);
            cudaStreamWaitEvent(0, j1, 0);
            cudaStreamWaitEvent(0, j2, 0);
        });
    }
    printf("nnz=%lld\n", (long long)nnz);
    return 0;
}
