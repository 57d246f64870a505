// sc_kmeans_small.cu -- the exact k-means replica for SMALL 1-D inputs (n <= 4096, k <= 256;
// config 1 is n = 1000, k = 5): one CTA per restart holds the points, the D^2 weights or own
// distances, the labels and the centres in shared memory, and runs every k-means++ round
// (kmeans.py:121-137) or every Lloyd iteration of its restart (kmeans.py:194-210) without
// leaving the kernel.  At these sizes the general path is bound by launches and host round
// trips (~30 launches for the seeding, a cooperative kernel with grid barriers for Lloyd);
// here the whole clustering is two launches.
//
// Arithmetic contract, element by element the one of oracle/sc_oracle.c (orc_kmeanspp,
// orc_lloyd_restart, orc_einsum_sumsq), i.e. of the reference's numpy calls:
//   weights / distances  d2ref = ((x*x) - (2x)*c) + c*c clipped at 0 (kmeans.py:106-113)
//   k-means++ draw       cumsum sequential in index order, first j with cum[j] > u * cum[-1]
//                        (searchsorted 'right', kmeans.py:116-118), n - 1 if none; a round
//                        whose weights are all 0 is reported (degen) for the host replay
//   assignment           argmin, lowest index on ties (:199)
//   repair               empties in increasing order, each takes the first point of maximal
//                        own distance, whose own distance is then 0 (:151-164)
//   means                np.add.at: per cluster a sequential sum in index order, / count,
//                        empty -> 0 (:86-93)
//   cost                 numpy einsum order (8192-element buffers, two lanes, 8-element
//                        steps 6|7, 4|5, 2|3, 0|1, zero-filled tail) (:96-103)
//   stop                 kmeans.py:202-210 incl. the :206 assertion (optional)
// Nothing here is approximate; tests/test_gpu_parity.py runs the reference's own k-means
// edge cases (degenerate seeding, repairs, negative values, k = 50) through this path.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "sc_common.cuh"

namespace sc {

constexpr int kSmallMaxN = 4096;
constexpr int kSmallMaxK = 256;
constexpr int kSmallTPB = 1024;

bool small_kmeans_eligible(int l, int k, int64_t n) {
    return l == 1 && n >= 1 && n <= kSmallMaxN && k >= 1 && k <= kSmallMaxK &&
           getenv("SC_KMEANS_NO_SMALL") == nullptr;
}

// block-wide: the lowest index j with flag(j), or `none`
__device__ __forceinline__ int block_first(bool flag, int j, int none, int *slot) {
    if (threadIdx.x == 0) *slot = none;
    __syncthreads();
    if (flag) atomicMin(slot, j);
    __syncthreads();
    const int v = *slot;
    __syncthreads();
    return v;
}

// k-means++ rounds start[r]..k-1 of restart r = blockIdx.x (same contract as sc_kmeans_pp)
__global__ void __launch_bounds__(kSmallTPB) k_kpp_small(const double *__restrict__ x, int n, int k,
                                                         const int32_t *__restrict__ start,
                                                         const double *__restrict__ u,
                                                         int64_t *__restrict__ chosen,
                                                         int32_t *__restrict__ degen) {
    extern __shared__ __align__(16) double sm[];
    double *xs = sm, *best = sm + n, *cum = sm + 2 * n;
    __shared__ int slot;
    __shared__ double s_tot;
    const int r = blockIdx.x;
    const int s0 = start[r];
    if (s0 >= k) return;
    int64_t *ch = chosen + (int64_t)r * k;
    for (int j = threadIdx.x; j < n; j += kSmallTPB) xs[j] = x[j];
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += kSmallTPB) {
        double b = d2ref(xs[j], xs[ch[0]]);
        for (int i = 1; i < s0; ++i) {
            const double d = d2ref(xs[j], xs[ch[i]]);
            if (d < b) b = d;
        }
        best[j] = b;
    }
    __syncthreads();
    for (int i = s0; i < k; ++i) {
        int any = 0;
        for (int j = threadIdx.x; j < n; j += kSmallTPB) any |= best[j] > 0.0;
        if (!__syncthreads_or(any)) {
            if (threadIdx.x == 0) degen[r] = i;
            return;
        }
        if (threadIdx.x == 0) {
            // np.cumsum: one left-to-right chain (loads run ahead of the adds)
            double c = 0.0;
#pragma unroll 8
            for (int j = 0; j < n; ++j) {
                c = __dadd_rn(c, best[j]);
                cum[j] = c;
            }
            s_tot = c;
        }
        __syncthreads();
        const double target = __dmul_rn(u[(int64_t)r * (k - 1) + (i - 1)], s_tot);
        int idx = n;
        for (int j0 = 0; j0 < n; j0 += kSmallTPB) {
            const int j = j0 + threadIdx.x;
            const int f = block_first(j < n && cum[j] > target, j, n, &slot);
            if (f < n) {
                idx = f;
                break;
            }
        }
        if (idx >= n) idx = n - 1;
        if (threadIdx.x == 0) ch[i] = idx;
        const double c = xs[idx];
        for (int j = threadIdx.x; j < n; j += kSmallTPB) {
            const double d = d2ref(xs[j], c);
            if (d < best[j]) best[j] = d;
        }
        __syncthreads();
    }
}

// Lloyd of restart r = blockIdx.x from the centres x[chosen[r*k + c]]
__global__ void __launch_bounds__(kSmallTPB) k_lloyd_small(const double *__restrict__ x, int n, int k,
                                                           const int64_t *__restrict__ chosen,
                                                           int max_iters, double tol, int assert_cost,
                                                           int32_t *__restrict__ lab_out,
                                                           double *__restrict__ cost_out,
                                                           int32_t *__restrict__ iters_out,
                                                           int32_t *__restrict__ err_out) {
    extern __shared__ __align__(16) double sm[];
    double *xs = sm, *own = sm + n, *cen = sm + 2 * n, *ncen = cen + k;
    uint8_t *lab = reinterpret_cast<uint8_t *>(ncen + k);
    uint8_t *prv = lab + ((n + 15) & ~15);
    int *cnt = reinterpret_cast<int *>(prv + ((n + 15) & ~15));
    int *elist = cnt + k;
    __shared__ int slot, s_ne, s_chg;
    __shared__ unsigned long long s_far;
    __shared__ double s_a[2];
    const int r = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int j = tid; j < n; j += kSmallTPB) {
        xs[j] = x[j];
        prv[j] = 0;  // labels = np.zeros(n) (kmeans.py:195)
    }
    for (int c = tid; c < k; c += kSmallTPB) cen[c] = x[chosen[(int64_t)r * k + c]];
    __syncthreads();
    double prev = INFINITY;
    int it = 0, err = 0;
    while (it < max_iters) {
        ++it;
        // assignment (argmin, lowest index on ties)
        for (int j = tid; j < n; j += kSmallTPB) {
            const double xv = xs[j];
            int bi = 0;
            double bd = d2ref(xv, cen[0]);
            for (int c = 1; c < k; ++c) {
                const double d = d2ref(xv, cen[c]);
                if (d < bd) {
                    bd = d;
                    bi = c;
                }
            }
            lab[j] = (uint8_t)bi;
            own[j] = bd;
        }
        for (int c = tid; c < k; c += kSmallTPB) cnt[c] = 0;
        __syncthreads();
        for (int j = tid; j < n; j += kSmallTPB) atomicAdd(&cnt[lab[j]], 1);
        __syncthreads();
        // _repair_empty: the empties listed once, in order
        if (tid == 0) {
            int ne = 0;
            for (int c = 0; c < k; ++c)
                if (cnt[c] == 0) elist[ne++] = c;
            s_ne = ne;
        }
        __syncthreads();
        const int ne = s_ne;
        for (int e = 0; e < ne; ++e) {
            // first index of the maximal own distance (own >= 0: its bits order like the value)
            if (tid == 0) s_far = 0ull;
            __syncthreads();
            unsigned long long key = 0ull;
            for (int j = tid; j < n; j += kSmallTPB) {
                const unsigned long long kb = (unsigned long long)__double_as_longlong(own[j]);
                key = kb > key ? kb : key;
            }
            atomicMax(&s_far, key);
            __syncthreads();
            const double omax = __longlong_as_double((long long)s_far);
            int far = n;
            for (int j0 = 0; j0 < n; j0 += kSmallTPB) {
                const int j = j0 + tid;
                const int f = block_first(j < n && own[j] == omax, j, n, &slot);
                if (f < n) {
                    far = f;
                    break;
                }
            }
            if (tid == 0) {
                cnt[lab[far]] -= 1;
                lab[far] = (uint8_t)elist[e];
                cnt[elist[e]] = 1;
                own[far] = 0.0;
            }
            __syncthreads();
        }
        // unchanged labels (kmeans.py:201), then keep them as the previous labels
        if (tid == 0) s_chg = 0;
        __syncthreads();
        int chg = 0;
        for (int j = tid; j < n; j += kSmallTPB) {
            chg |= lab[j] != prv[j];
            prv[j] = lab[j];
        }
        if (chg) s_chg = 1;
        // cluster_means: warp w sums the clusters w, w+32, ... in index order
        for (int c = warp; c < k; c += kSmallTPB / 32) {
            double sum = 0.0;
            for (int j0 = 0; j0 < n; j0 += 32) {
                const int j = j0 + lane;
                unsigned m = __ballot_sync(0xffffffffu, j < n && lab[j] == c);
                if (lane == 0)
                    while (m) {
                        const int b = __ffs(m) - 1;
                        m &= m - 1;
                        sum = __dadd_rn(sum, xs[j0 + b]);
                    }
            }
            if (lane == 0) ncen[c] = cnt[c] > 0 ? __ddiv_rn(sum, (double)cnt[c]) : sum;
        }
        __syncthreads();
        const bool unchanged = std::isfinite(prev) && !s_chg;
        for (int c = tid; c < k; c += kSmallTPB) cen[c] = ncen[c];
        __syncthreads();
        // diff = x - mu[label], kept in own[]
        for (int j = tid; j < n; j += kSmallTPB) own[j] = __dsub_rn(xs[j], cen[lab[j]]);
        __syncthreads();
        // kmeans_cost: numpy einsum order, lane chains a0 (thread 0) and a1 (thread 1)
        if (tid < 2) {
            double out = 0.0;
            for (int c0 = 0; c0 < n; c0 += 8192) {
                const int m = n - c0 < 8192 ? n - c0 : 8192;
                const double *p = own + c0;
                double acc = 0.0;
                int i = 0;
                for (; m - i >= 8; i += 8)
                    for (int b = 3; b >= 0; --b) {
                        const double v = p[i + 2 * b + tid];
                        acc = __dadd_rn(__dmul_rn(v, v), acc);
                    }
                for (; i < m; i += 2) {
                    const double v = (i + tid < m) ? p[i + tid] : 0.0;
                    acc = __dadd_rn(__dmul_rn(v, v), acc);
                }
                s_a[tid] = acc;
                __syncwarp(0x3u);
                if (tid == 0) out = __dadd_rn(__dadd_rn(s_a[0], s_a[1]), out);
                __syncwarp(0x3u);
            }
            if (tid == 0) s_a[0] = out;
        }
        __syncthreads();
        const double cost = s_a[0];
        __syncthreads();
        // kmeans.py:206-210
        if (!(cost <= __dadd_rn(__dmul_rn(prev, 1.0 + 1e-12), 1e-12)) && assert_cost) {
            err = it;
            prev = cost;
            break;
        }
        const bool small_gain = std::isfinite(prev) &&
                                __dsub_rn(prev, cost) <= __dmul_rn(tol, fmax(prev, 1e-300));
        prev = cost;
        if (unchanged || small_gain) break;
    }
    for (int j = tid; j < n; j += kSmallTPB) lab_out[(int64_t)r * n + j] = lab[j];
    if (tid == 0) {
        cost_out[r] = prev;
        iters_out[r] = it;
        err_out[r] = err;
    }
}

static size_t kpp_smem(int n) { return (size_t)3 * n * 8; }
static size_t lloyd_smem(int n, int k) {
    return (size_t)2 * n * 8 + (size_t)2 * k * 8 + (size_t)((n + 15) & ~15) * 2 + (size_t)2 * k * 4;
}

int32_t small_kpp(int device, cudaStream_t s, const double *d_x, int64_t n, int k, int R,
                  const int32_t *d_start, const double *d_u, int64_t *d_chosen, int32_t *d_degen) {
    const size_t sm = kpp_smem((int)n);
    if (sm > 48 * 1024)
        SC_CUDA(cudaFuncSetAttribute(k_kpp_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_kpp_small<<<R, kSmallTPB, sm, s>>>(d_x, (int)n, k, d_start, d_u, d_chosen, d_degen);
    SC_CUDA(cudaGetLastError());
    (void)device;
    return SC_OK;
}

// Lloyd for all R restarts; d_lab (R*n int32), d_cost (R), d_iters (R), d_err (R) are
// device workspaces.  Writes the winner's labels (first strictly smallest cost) to labels_out.
int32_t small_lloyd(cudaStream_t s, const double *d_x, int64_t n, int k, int R,
                    const int64_t *d_chosen, int max_iters, double tol, bool assert_cost,
                    int32_t *d_lab, double *d_cost, int32_t *d_iters, int32_t *d_err,
                    int64_t *labels_out, double *costs_out, int32_t *iters_out, int32_t *best_out) {
    const size_t sm = lloyd_smem((int)n, k);
    if (sm > 48 * 1024)
        SC_CUDA(cudaFuncSetAttribute(k_lloyd_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_lloyd_small<<<R, kSmallTPB, sm, s>>>(d_x, (int)n, k, d_chosen, max_iters, tol,
                                           assert_cost ? 1 : 0, d_lab, d_cost, d_iters, d_err);
    SC_CUDA(cudaGetLastError());
    std::vector<double> cost((size_t)R);
    std::vector<int32_t> its((size_t)R), err((size_t)R);
    SC_CUDA(cudaMemcpyAsync(cost.data(), d_cost, (size_t)R * 8, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaMemcpyAsync(its.data(), d_iters, (size_t)R * 4, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaMemcpyAsync(err.data(), d_err, (size_t)R * 4, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaStreamSynchronize(s));
    for (int r = 0; r < R; ++r)
        if (err[r]) return fail(SC_E_INTERNAL, "k-means cost increased (restart %d, iteration %d)", r, err[r] - 1);
    int best = -1;
    double bc = INFINITY;
    for (int r = 0; r < R; ++r)
        if (cost[r] < bc) {
            bc = cost[r];
            best = r;
        }
    SC_REQUIRE(best >= 0, SC_E_INTERNAL, "no restart produced a finite cost");
    std::vector<int32_t> lab((size_t)n);
    SC_CUDA(cudaMemcpy(lab.data(), d_lab + (size_t)best * n, (size_t)n * 4, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i) labels_out[i] = lab[(size_t)i];
    if (costs_out)
        for (int r = 0; r < R; ++r) costs_out[r] = cost[r];
    if (iters_out)
        for (int r = 0; r < R; ++r) iters_out[r] = its[r];
    if (best_out) *best_out = best;
    return SC_OK;
}

}  // namespace sc
