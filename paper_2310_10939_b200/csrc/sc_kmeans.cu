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
#include <cub/device/device_radix_sort.cuh>
#include <vector>

#include "sc_common.cuh"

namespace sc {
const double *graph_f_device(const sc_graph *g);
int64_t graph_n(const sc_graph *g);
int graph_device(const sc_graph *g);
}  // namespace sc

struct sc_kmeans {
    int device = 0;
    int sm_count = 148;
    int64_t n = 0;
    double *d_x = nullptr;
    cudaStream_t stream = nullptr;
    // workspaces (grown on demand)
    int cap_r = 0, cap_k = 0;
    double *d_best = nullptr;      // [R][n] k-means++ D^2 weights
    int32_t *d_lab[2] = {nullptr, nullptr};  // [R][n] labels (current / previous)
    int32_t *d_keys = nullptr;     // [R*n] sort keys (r*k + label)
    int32_t *d_keys_alt = nullptr;
    double *d_vals = nullptr;      // [R*n] sorted points
    double *d_vals_alt = nullptr;
    double *d_own = nullptr;       // [n] repair scratch
    void *d_cub = nullptr;
    size_t cub_bytes = 0;
    int64_t *d_chosen = nullptr;   // [R][k]
    double *d_u = nullptr;         // [R][k-1]
    int32_t *d_start = nullptr;    // [R]
    int32_t *d_degen = nullptr;    // [R]
    double *d_cen = nullptr;       // [R][k]
    int32_t *d_cnt = nullptr;      // [R][k]
    int64_t *d_seg = nullptr;      // [R*k + 1] segment offsets into the sorted arrays
    double *d_part = nullptr;      // [R][nchunks][2] einsum lane partials
    double *d_cost = nullptr;      // [R]
    int32_t *d_changed = nullptr;  // [R]
    int32_t *d_active = nullptr;   // [R]
    int32_t *d_empty = nullptr;    // [R]
};

namespace sc {

constexpr int kEinsumBuf = 8192;  // numpy nditer buffer size (elements)

// ---------------------------------------------------------------------------
// k-means++

// best[r][j] = min over chosen[r][0..start_r-1] of d2(x_j, x[chosen])
__global__ void k_kpp_init(const double *__restrict__ x, int64_t n, int k,
                           const int64_t *__restrict__ chosen, const int32_t *__restrict__ start,
                           double *__restrict__ best) {
    const int r = blockIdx.y;
    const int s = start[r];
    double *b = best + (int64_t)r * n;
    const int64_t *ch = chosen + (int64_t)r * k;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double xj = x[j];
        double v = d2ref(xj, x[ch[0]]);
        for (int i = 1; i < s; ++i) v = fmin(v, d2ref(xj, x[ch[i]]));
        b[j] = v;
    }
}

// best = min(best, d2(x, x[chosen[r][i]])) for restarts whose round i just picked
__global__ void k_kpp_update(const double *__restrict__ x, int64_t n, int k, int i,
                             const int64_t *__restrict__ chosen, const int32_t *__restrict__ start,
                             const int32_t *__restrict__ degen, double *__restrict__ best) {
    const int r = blockIdx.y;
    if (i < start[r] || degen[r] >= 0) return;
    const double c = x[chosen[(int64_t)r * k + i]];
    double *b = best + (int64_t)r * n;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double v = d2ref(x[j], c);
        if (v < b[j]) b[j] = v;
    }
}

// One CTA per restart: round i of _kmeans_pp_indices.  v0: the sequential cumsum is one
// thread walking the weights with 8-deep prefetch (np.cumsum order); "any weight > 0" is a
// block reduction (== best_d2.sum() > 0 for nonnegative weights).
__global__ void __launch_bounds__(256) k_kpp_pick(int64_t n, int k, int i,
                                                  const double *__restrict__ best,
                                                  const double *__restrict__ u,
                                                  int64_t *__restrict__ chosen,
                                                  const int32_t *__restrict__ start,
                                                  int32_t *__restrict__ degen) {
    const int r = blockIdx.x;
    if (i < start[r] || degen[r] >= 0) return;
    const double *b = best + (int64_t)r * n;
    __shared__ int any;
    if (threadIdx.x == 0) any = 0;
    __syncthreads();
    int mine = 0;
    for (int64_t j = threadIdx.x; j < n && !mine; j += blockDim.x) mine = b[j] > 0.0;
    if (mine) any = 1;
    __syncthreads();
    if (threadIdx.x != 0) return;
    if (!any) {
        degen[r] = i;
        return;
    }
    double tot = 0.0;
    int64_t j = 0;
    for (; j + 8 <= n; j += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = b[j + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) tot = __dadd_rn(tot, v[q]);
    }
    for (; j < n; ++j) tot = __dadd_rn(tot, b[j]);
    const double target = __dmul_rn(u[(int64_t)r * (k - 1) + (i - 1)], tot);
    double cum = 0.0;
    int64_t idx = n - 1;
    for (j = 0; j + 8 <= n; j += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = b[j + q];
        bool hit = false;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (!hit) {
                cum = __dadd_rn(cum, v[q]);
                if (cum > target) {
                    hit = true;
                    idx = j + q;
                }
            }
        }
        if (hit) break;
    }
    if (j + 8 > n) {
        for (; j < n; ++j) {
            cum = __dadd_rn(cum, b[j]);
            if (cum > target) {
                idx = j;
                break;
            }
        }
    }
    chosen[(int64_t)r * k + i] = idx;
}

// ---------------------------------------------------------------------------
// Lloyd

// assignment: labels, counts, changed vs previous labels
__global__ void k_assign(const double *__restrict__ x, int64_t n, int k,
                         const double *__restrict__ cen, const int32_t *__restrict__ active,
                         const int32_t *__restrict__ prev, int32_t *__restrict__ lab,
                         int32_t *__restrict__ cnt, int32_t *__restrict__ changed) {
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
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double xj = x[j];
        int bi = 0;
        double bd = d2ref(xj, c[0]);
        for (int q = 1; q < k; ++q) {
            const double d = d2ref(xj, c[q]);
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

// _repair_empty (kmeans.py:151-164), one CTA per restart; returns at once when no
// cluster is empty (the common case).  Clusters empty after assignment are repaired in
// increasing order: the first point of maximal own distance moves in, its own distance
// becomes 0.  Then counts and the changed-label count of the restart are recomputed.
__global__ void __launch_bounds__(1024) k_repair(const double *__restrict__ x, int64_t n, int k,
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
    const double *cc = cen + (int64_t)r * k;
    double *own = own_all + (int64_t)r * n;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) own[j] = d2ref(x[j], cc[lb[j]]);
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

__global__ void k_make_keys(int64_t n, int k, const int32_t *__restrict__ lab,
                            int32_t *__restrict__ keys, double *__restrict__ vals,
                            const double *__restrict__ x, int R) {
    const int64_t tot = (int64_t)R * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / n, j = t - r * n;
        keys[t] = (int32_t)(r * k + lab[t]);
        vals[t] = x[j];
    }
}

// segment offsets: seg[t] = first position of key >= t in the sorted keys
__global__ void k_seg_offsets(int rk, int64_t total, const int32_t *__restrict__ keys,
                              int64_t *__restrict__ seg) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > rk) return;
    int64_t lo = 0, hi = total;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < t) lo = mid + 1;
        else hi = mid;
    }
    seg[t] = lo;
}

// ordered per-cluster sums (np.add.at order) and means; v0: one thread per segment
__global__ void k_seg_means(int rk, int k, const int64_t *__restrict__ seg,
                            const double *__restrict__ vals, const int32_t *__restrict__ active,
                            double *__restrict__ cen) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rk) return;
    if (!active[t / k]) return;
    const int64_t lo = seg[t], hi = seg[t + 1];
    double s = 0.0;
    int64_t j = lo;
    for (; j + 8 <= hi; j += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = vals[j + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) s = __dadd_rn(s, v[q]);
    }
    for (; j < hi; ++j) s = __dadd_rn(s, vals[j]);
    const int64_t c = hi - lo;
    cen[t] = c > 0 ? __ddiv_rn(s, (double)c) : s;
}

// einsum lane partials: thread (r, buffer, lane) sums its lane of one 8192-element buffer
__global__ void k_cost_lanes(const double *__restrict__ x, int64_t n, int k,
                             const int32_t *__restrict__ lab, const double *__restrict__ cen,
                             const int32_t *__restrict__ active, int64_t nbuf,
                             double *__restrict__ part) {
    const int r = blockIdx.y;
    if (!active[r]) return;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nbuf * 2) return;
    const int64_t bufi = t >> 1;
    const int lane = (int)(t & 1);
    const int32_t *lb = lab + (int64_t)r * n;
    const double *c = cen + (int64_t)r * k;
    const int64_t base = bufi * kEinsumBuf;
    const int64_t m = std::min<int64_t>(kEinsumBuf, n - base);
    double acc = 0.0;
    int64_t i = 0;
    for (; m - i >= 8; i += 8) {
#pragma unroll
        for (int blk = 3; blk >= 0; --blk) {
            const int64_t j = base + i + 2 * blk + lane;
            const double d = __dsub_rn(x[j], c[lb[j]]);
            acc = __dadd_rn(__dmul_rn(d, d), acc);
        }
    }
    for (; i < m; i += 2) {
        double d = 0.0;
        if (i + lane < m) {
            const int64_t j = base + i + lane;
            d = __dsub_rn(x[j], c[lb[j]]);
        }
        acc = __dadd_rn(__dmul_rn(d, d), acc);
    }
    part[((int64_t)r * nbuf + bufi) * 2 + lane] = acc;
}

// buffer totals (l0 + l1) added into the running output in buffer order
__global__ void k_cost_combine(int64_t nbuf, const double *__restrict__ part,
                               const int32_t *__restrict__ active, double *__restrict__ cost) {
    const int r = blockIdx.x;
    if (threadIdx.x != 0 || !active[r]) return;
    double out = 0.0;
    const double *p = part + (int64_t)r * nbuf * 2;
    for (int64_t b = 0; b < nbuf; ++b) out = __dadd_rn(__dadd_rn(p[2 * b], p[2 * b + 1]), out);
    cost[r] = out;
}

__global__ void k_gather_centers(const double *__restrict__ x, const int64_t *__restrict__ chosen,
                                 int rk, double *__restrict__ cen) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < rk) cen[t] = x[chosen[t]];
}

template <typename T>
static int32_t grow(T **p, size_t count) {
    if (*p) cudaFree(*p);
    *p = nullptr;
    cudaError_t e = cudaMalloc((void **)p, std::max<size_t>(count, 1) * sizeof(T));
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
    const int64_t nbuf = (n + kEinsumBuf - 1) / kEinsumBuf;
    int32_t st;
    if ((st = grow(&km->d_best, (size_t)R * n))) return st;
    if ((st = grow(&km->d_lab[0], (size_t)R * n))) return st;
    if ((st = grow(&km->d_lab[1], (size_t)R * n))) return st;
    if ((st = grow(&km->d_keys, (size_t)R * n))) return st;
    if ((st = grow(&km->d_keys_alt, (size_t)R * n))) return st;
    if ((st = grow(&km->d_vals, (size_t)R * n))) return st;
    if ((st = grow(&km->d_vals_alt, (size_t)R * n))) return st;
    if ((st = grow(&km->d_own, (size_t)n))) return st;
    if ((st = grow(&km->d_chosen, (size_t)R * k))) return st;
    if ((st = grow(&km->d_u, (size_t)R * k))) return st;
    if ((st = grow(&km->d_start, (size_t)R))) return st;
    if ((st = grow(&km->d_degen, (size_t)R))) return st;
    if ((st = grow(&km->d_cen, (size_t)R * k))) return st;
    if ((st = grow(&km->d_cnt, (size_t)R * k))) return st;
    if ((st = grow(&km->d_seg, (size_t)R * k + 1))) return st;
    if ((st = grow(&km->d_part, (size_t)R * nbuf * 2))) return st;
    if ((st = grow(&km->d_cost, (size_t)R))) return st;
    if ((st = grow(&km->d_changed, (size_t)R))) return st;
    if ((st = grow(&km->d_active, (size_t)R))) return st;
    if ((st = grow(&km->d_empty, (size_t)R))) return st;
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, km->d_keys, km->d_keys_alt, km->d_vals,
                                    km->d_vals_alt, (int64_t)R * n, 0, 31, km->stream);
    if ((st = grow((unsigned char **)&km->d_cub, need))) return st;
    km->cub_bytes = need;
    km->cap_r = R;
    km->cap_k = k;
    return SC_OK;
}

static int grid_1d(const sc_kmeans *km, int64_t work, int tpb) {
    const int64_t want = (work + tpb - 1) / tpb;
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)km->sm_count * 8));
}

static int32_t km_init(int device, int64_t n, sc_kmeans **out) {
    sc_kmeans *km = new sc_kmeans();
    km->device = device;
    km->n = n;
    cudaDeviceGetAttribute(&km->sm_count, cudaDevAttrMultiProcessorCount, device);
    cudaError_t e = cudaStreamCreateWithFlags(&km->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&km->d_x, (size_t)n * 8);
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

int32_t sc_kmeans_create(const double *points_host, int64_t n, int32_t device,
                         sc_kmeans **out) {
    SC_REQUIRE(out && points_host, SC_E_INVALID, "null argument");
    SC_REQUIRE(n >= 1, SC_E_INVALID, "need n >= 1 points");
    for (int64_t i = 0; i < n; ++i)
        SC_REQUIRE(std::isfinite(points_host[i]), SC_E_INVALID, "points contain NaN or Inf");
    SC_CUDA(cudaSetDevice(device));
    int32_t st = km_init(device, n, out);
    if (st) return st;
    SC_CUDA(cudaMemcpy((*out)->d_x, points_host, (size_t)n * 8, cudaMemcpyHostToDevice));
    return SC_OK;
}

int32_t sc_kmeans_create_from_graph(sc_graph *g, sc_kmeans **out) {
    SC_REQUIRE(g && out, SC_E_INVALID, "null argument");
    const double *f = graph_f_device(g);
    SC_REQUIRE(f, SC_E_STATE, "graph has no embedding yet: call sc_power_iterate first");
    SC_CUDA(cudaSetDevice(graph_device(g)));
    int32_t st = km_init(graph_device(g), graph_n(g), out);
    if (st) return st;
    SC_CUDA(cudaMemcpy((*out)->d_x, f, (size_t)graph_n(g) * 8, cudaMemcpyDeviceToDevice));
    return SC_OK;
}

void sc_kmeans_destroy(sc_kmeans *km) {
    if (!km) return;
    cudaSetDevice(km->device);
    if (km->stream) cudaStreamSynchronize(km->stream);
    void *ptrs[] = {km->d_x, km->d_best, km->d_lab[0], km->d_lab[1], km->d_keys, km->d_keys_alt,
                    km->d_vals, km->d_vals_alt, km->d_own, km->d_cub, km->d_chosen, km->d_u,
                    km->d_start, km->d_degen, km->d_cen, km->d_cnt, km->d_seg, km->d_part,
                    km->d_cost, km->d_changed, km->d_active, km->d_empty};
    for (void *p : ptrs) cudaFree(p);
    if (km->stream) cudaStreamDestroy(km->stream);
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
    for (int r = 0; r < R; ++r) smin = std::min(smin, start_round[r]);
    const dim3 g2(grid_1d(km, n, 256) / std::max(1, std::min(R, 8)) + 1, R);
    k_kpp_init<<<g2, 256, 0, s>>>(km->d_x, n, k, km->d_chosen, km->d_start, km->d_best);
    SC_CUDA(cudaGetLastError());
    for (int i = smin; i < k; ++i) {
        k_kpp_pick<<<R, 256, 0, s>>>(n, k, i, km->d_best, km->d_u, km->d_chosen, km->d_start,
                                      km->d_degen);
        k_kpp_update<<<g2, 256, 0, s>>>(km->d_x, n, k, i, km->d_chosen, km->d_start,
                                         km->d_degen, km->d_best);
    }
    SC_CUDA(cudaGetLastError());
    SC_CUDA(cudaMemcpyAsync(chosen, km->d_chosen, (size_t)R * k * 8, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaMemcpyAsync(degenerate_out, km->d_degen, (size_t)R * 4, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaStreamSynchronize(s));
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
    const int64_t nbuf = (n + kEinsumBuf - 1) / kEinsumBuf;
    const int rk = R * k;
    SC_CUDA(cudaMemcpyAsync(km->d_chosen, chosen, (size_t)rk * 8, cudaMemcpyHostToDevice, s));
    k_gather_centers<<<(rk + 255) / 256, 256, 0, s>>>(km->d_x, km->d_chosen, rk, km->d_cen);
    // labels start at zero (kmeans.py:195)
    SC_CUDA(cudaMemsetAsync(km->d_lab[0], 0, (size_t)R * n * 4, s));
    std::vector<int32_t> active(R, 1), changed(R), iters(R, 0), final_buf(R, 0);
    std::vector<double> prev(R, INFINITY), cost(R, INFINITY);
    int cur = 0;  // d_lab[cur] = labels of the previous iteration
    int end_bit = 1;
    while ((1ll << end_bit) < (long long)rk) ++end_bit;
    const size_t smem_assign = (size_t)k * 12;
    SC_REQUIRE(smem_assign <= 200 * 1024, SC_E_INVALID, "k=%d too large for the assign kernel", k);
    if (smem_assign > 48 * 1024)
        SC_CUDA(cudaFuncSetAttribute(k_assign, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_assign));
    if (k > 48 * 1024)
        SC_CUDA(cudaFuncSetAttribute(k_repair, cudaFuncAttributeMaxDynamicSharedMemorySize, k));
    const dim3 ga(grid_1d(km, n, 256) / std::max(1, std::min(R, 8)) + 1, R);
    const dim3 gc((unsigned)((nbuf * 2 + 127) / 128), R);
    for (int it = 0; it < max_iters; ++it) {
        int nact = 0;
        for (int r = 0; r < R; ++r) nact += active[r];
        if (!nact) break;
        const int nxt = cur ^ 1;
        SC_CUDA(cudaMemcpyAsync(km->d_active, active.data(), (size_t)R * 4, cudaMemcpyHostToDevice, s));
        SC_CUDA(cudaMemsetAsync(km->d_cnt, 0, (size_t)rk * 4, s));
        SC_CUDA(cudaMemsetAsync(km->d_changed, 0, (size_t)R * 4, s));
        k_assign<<<ga, 256, smem_assign, s>>>(km->d_x, n, k, km->d_cen, km->d_active,
                                               km->d_lab[cur], km->d_lab[nxt], km->d_cnt,
                                               km->d_changed);
        k_repair<<<R, 1024, (size_t)k, s>>>(km->d_x, n, k, km->d_cen, km->d_active,
                                              km->d_lab[cur], km->d_lab[nxt], km->d_cnt,
                                              km->d_changed, km->d_best);
        // inactive restarts carry their final labels forward so every restart's labels
        // live in d_lab[nxt] (the sort below covers all restarts)
        for (int r = 0; r < R; ++r)
            if (!active[r])
                SC_CUDA(cudaMemcpyAsync(km->d_lab[nxt] + (size_t)r * n, km->d_lab[cur] + (size_t)r * n,
                                        (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
        // np.add.at order: stable radix sort on (restart, label) keeps point-index order
        // inside every cluster; then ordered segment sums
        k_make_keys<<<grid_1d(km, (int64_t)R * n, 256), 256, 0, s>>>(
            n, k, km->d_lab[nxt], km->d_keys, km->d_vals, km->d_x, R);
        size_t tb = km->cub_bytes;
        SC_CUDA(cub::DeviceRadixSort::SortPairs(km->d_cub, tb, km->d_keys, km->d_keys_alt,
                                                km->d_vals, km->d_vals_alt, (int64_t)R * n, 0,
                                                end_bit, s));
        k_seg_offsets<<<(rk + 1 + 255) / 256, 256, 0, s>>>(rk, (int64_t)R * n, km->d_keys_alt,
                                                           km->d_seg);
        k_seg_means<<<(rk + 127) / 128, 128, 0, s>>>(rk, k, km->d_seg, km->d_vals_alt,
                                                     km->d_active, km->d_cen);
        k_cost_lanes<<<gc, 128, 0, s>>>(km->d_x, n, k, km->d_lab[nxt], km->d_cen, km->d_active,
                                        nbuf, km->d_part);
        k_cost_combine<<<R, 32, 0, s>>>(nbuf, km->d_part, km->d_active, km->d_cost);
        SC_CUDA(cudaGetLastError());
        SC_CUDA(cudaMemcpyAsync(cost.data(), km->d_cost, (size_t)R * 8, cudaMemcpyDeviceToHost, s));
        SC_CUDA(cudaMemcpyAsync(changed.data(), km->d_changed, (size_t)R * 4, cudaMemcpyDeviceToHost, s));
        SC_CUDA(cudaStreamSynchronize(s));
        for (int r = 0; r < R; ++r) {
            if (!active[r]) continue;
            // kmeans.py:202-210, in the same double arithmetic
            const bool fin = std::isfinite(prev[r]);
            const bool unchanged = changed[r] == 0 && fin;
            const double c = cost[r];
            const bool small_gain = fin && (prev[r] - c <= tol * std::max(prev[r], 1e-300));
            prev[r] = c;
            iters[r] += 1;
            final_buf[r] = nxt;
            if (unchanged || small_gain) active[r] = 0;
        }
        cur = nxt;
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
    for (int64_t j = 0; j < n; ++j) labels_out[j] = lab32[(size_t)j];
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
