// sc_common.cuh -- shared plumbing for the sm_100a one-vector path: status/error
// reporting behind the C-ABI, CUDA checks, and the exact-arithmetic device helpers.
//
// All floating-point work that must match the reference bit for bit is written with
// explicit round-to-nearest intrinsics (__dadd_rn/__dmul_rn/__ddiv_rn) and the library is
// compiled with -fmad=false, so no FMA contraction can change a rounding.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/sc_b200.h"

namespace sc {

void set_error(const char *fmt, ...);
int32_t fail(int32_t code, const char *fmt, ...);

struct Status {
    int32_t code = SC_OK;
};

}  // namespace sc

#define SC_CUDA(call)                                                                    \
    do {                                                                                 \
        cudaError_t _e = (call);                                                         \
        if (_e != cudaSuccess) {                                                         \
            return ::sc::fail(_e == cudaErrorMemoryAllocation ? SC_E_OOM : SC_E_CUDA,    \
                              "%s:%d %s: %s", __FILE__, __LINE__, #call,                 \
                              cudaGetErrorString(_e));                                   \
        }                                                                                \
    } while (0)

#define SC_REQUIRE(cond, code, ...)                 \
    do {                                            \
        if (!(cond)) return ::sc::fail(code, __VA_ARGS__); \
    } while (0)

namespace sc {

constexpr int kSmCountB200 = 148;

// ---------------------------------------------------------------------------
// Philox4x64-10 (numpy.random.Philox); round constants from Salmon et al. 2011.
struct u64x4 {
    uint64_t x, y, z, w;
};

__host__ __device__ inline u64x4 philox4x64_10(u64x4 c, uint64_t k0, uint64_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ULL;
            k1 += 0xBB67AE8584CAA73BULL;
        }
#ifdef __CUDA_ARCH__
        uint64_t h0 = __umul64hi(0xD2E7470EE14C6C93ULL, c.x), l0 = 0xD2E7470EE14C6C93ULL * c.x;
        uint64_t h1 = __umul64hi(0xCA5A826395121157ULL, c.z), l1 = 0xCA5A826395121157ULL * c.z;
#else
        __uint128_t p0 = (__uint128_t)0xD2E7470EE14C6C93ULL * c.x;
        __uint128_t p1 = (__uint128_t)0xCA5A826395121157ULL * c.z;
        uint64_t h0 = (uint64_t)(p0 >> 64), l0 = (uint64_t)p0;
        uint64_t h1 = (uint64_t)(p1 >> 64), l1 = (uint64_t)p1;
#endif
        c = u64x4{h1 ^ c.y ^ k0, l1, h0 ^ c.w ^ k1, l0};
    }
    return c;
}

__device__ __forceinline__ double u53(uint64_t r) {
    return __dmul_rn((double)(r >> 11), 1.1102230246251565e-16);  // 2^-53, exact
}

// _sq_dists_to (specluster/kmeans.py:106-113) for d = 1:
// ((x*x) - ((2x)*c)) + (c*c), clipped at zero, every operation rounded separately.
__device__ __forceinline__ double d2ref(double x, double c) {
    double v = __dadd_rn(__dsub_rn(__dmul_rn(x, x), __dmul_rn(__dmul_rn(2.0, x), c)),
                         __dmul_rn(c, c));
    return v < 0.0 ? 0.0 : v;
}

// streaming (evict-first) and read-only cached loads
__device__ __forceinline__ int4 ld_stream_int4(const int4 *p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream_d2(const double2 *p) { return __ldcs(p); }

}  // namespace sc

// labels widened to the int64 the reference's Partition holds (kmeans.py:41), on several host
// threads for large n (a scalar loop costs ~60 ms at 1e8 points)
#include <thread>
#include <vector>
namespace sc {
template <typename T>
inline void widen_labels(const T *src, int64_t *dst, int64_t n) {
    const int64_t kMin = int64_t(1) << 19;
    int nthr = (int)std::min<int64_t>(8, std::max<int64_t>(1, n / kMin));
    nthr = std::min<int>(nthr, std::max(1u, std::thread::hardware_concurrency()));
    auto work = [&](int t) {
        const int64_t lo = n * t / nthr, hi = n * (t + 1) / nthr;
        for (int64_t i = lo; i < hi; ++i) dst[i] = (int64_t)src[i];
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nthr; ++t) th.emplace_back(work, t);
    work(0);
    for (auto &x : th) x.join();
}
}  // namespace sc
