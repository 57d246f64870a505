// panel_bench.cu -- feasibility probe for a column-panel SpMV (dense panels of z staged in
// shared memory by TMA, sparse remainder gathered from L2), against the config-2 pattern.
//
// Layout: rows split into CTA row blocks of SPB 32-row slices; lane l of slice i owns one row
// for the whole step (partial sum in a register, so entries are added in stored order without
// any cross-thread ordering). Columns split into panels of Z doubles. Per row block a panel is
// "dense" if the block has >= thresh entries in it: the panel is bulk-copied into shared memory
// and its entries are 16-bit panel-local indices; runs of non-dense panels form "sparse" groups
// with 32-bit global indices gathered from L2. Each (group, slice) is an ELL tile: width =
// max entries of its 32 rows, entries column-major, padding points at a zero slot.
// Usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o panel_bench panel_bench.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                            \
        }                                                                       \
    } while (0)

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
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *m) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(m))
        : "memory");
}

template <typename T>
static T *up(const std::vector<T> &v) {
    T *d;
    CK(cudaMalloc(&d, v.size() * sizeof(T) + 64));
    CK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}

// ---- version 3: register prefetch of the next tile's entries (chunk-major uint4 packing) ----
struct Layout3 {
    int spb, G, S, Z;
    std::vector<int> blk_g, grp_panel, blk_dense, dense_panel;
    std::vector<int64_t> tbase;  // per (block, warp) + 1: tile range
    std::vector<uint2> tiles;    // (offset in 512-B units, width | dense << 16)
    std::vector<uint32_t> grp_off;  // per group + 1: first byte / 512
    std::vector<uint8_t> bytes;
};

template <bool DENSE>
__device__ __forceinline__ int ent(const uint4 &a, const uint4 &b, int e) {
    if (DENSE) {
        const uint32_t wv = e < 8 ? (&a.x)[(e & 7) >> 1] : (&b.x)[(e & 7) >> 1];
        return (e & 1) ? (int)(wv >> 16) : (int)(wv & 0xffff);
    } else {
        return e < 4 ? (int)(&a.x)[e & 3] : (int)(&b.x)[e & 3];
    }
}

template <int Z, int MAXS>
__global__ void __launch_bounds__(1024, 1)
    k_panel3(const int *blk_g, const int *grp_panel, const int *blk_dense, const int *dense_panel,
             const int64_t *tbase, const uint2 *tiles, const uint4 *ent16, const double *z, int spb,
             int64_t n, double *out) {
    extern __shared__ __align__(128) double zs[];
    __shared__ uint64_t full[2];
    const int b = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    constexpr int kStride = Z + 16;
    const int g0 = blk_g[b], g1 = blk_g[b + 1];
    const int d0 = blk_dense[b], d1 = blk_dense[b + 1];
    constexpr uint32_t kChunk = 16384;
    auto issue_z = [&](int d) {
        const int buf = (d - d0) & 1;
        const double *src = z + (int64_t)dense_panel[d] * Z;
        mbar_expect(&full[buf], Z * 8);
        for (uint32_t o = 0; o < Z * 8u; o += kChunk)
            bulk_g2s((char *)(zs + buf * kStride) + o, (const char *)src + o, min(kChunk, Z * 8u - o),
                     &full[buf]);
    };
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 2) zs[threadIdx.x * kStride + Z] = 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
        if (d0 < d1) issue_z(d0);
        if (d0 + 1 < d1) issue_z(d0 + 1);
    }
    const int64_t t0 = tbase[b * 32 + w], t1 = tbase[b * 32 + w + 1];
    int64_t t = t0;
    uint2 m_cur = t0 < t1 ? tiles[t0] : make_uint2(0, 0);
    uint2 m_nxt = t0 + 1 < t1 ? tiles[t0 + 1] : make_uint2(0, 0);
    const uint4 zero4 = make_uint4(0, 0, 0, 0);
    uint4 a_cur = zero4, b_cur = zero4;
    if (t0 < t1) {
        const uint4 *src = ent16 + (int64_t)m_cur.x * 32 + lane;
        a_cur = __ldcs(src);
        const int wd = m_cur.y & 0xffff, per = (m_cur.y >> 16) ? 8 : 4;
        if (wd > per) b_cur = __ldcs(src + 32);
    }
    double p[MAXS];
#pragma unroll
    for (int j = 0; j < MAXS; ++j) p[j] = 0.0;
    int d = d0;
    for (int g = g0; g < g1; ++g) {
        const bool dense = grp_panel[g] >= 0;
        const double *zb = zs + ((d - d0) & 1) * kStride;
        if (dense) mbar_wait(&full[(d - d0) & 1], ((d - d0) >> 1) & 1);
#pragma unroll
        for (int j = 0; j < MAXS; ++j) {
            if (w + 32 * j < spb) {
                // prefetch next tile's entries and the meta two ahead
                uint4 a_n = zero4, b_n = zero4;
                uint2 m_n2 = make_uint2(0, 0);
                if (t + 1 < t1) {
                    const uint4 *src = ent16 + (int64_t)m_nxt.x * 32 + lane;
                    a_n = __ldcs(src);
                    const int wd = m_nxt.y & 0xffff, per = (m_nxt.y >> 16) ? 8 : 4;
                    if (wd > per) b_n = __ldcs(src + 32);
                }
                if (t + 2 < t1) m_n2 = tiles[t + 2];
                const int wd = m_cur.y & 0xffff;
                double acc = p[j];
                if (dense) {
#pragma unroll
                    for (int k = 0; k < 16; k += 4) {
                        if (k < wd) {
                            const double v0 = zb[ent<true>(a_cur, b_cur, k)], v1 = zb[ent<true>(a_cur, b_cur, k + 1)],
                                         v2 = zb[ent<true>(a_cur, b_cur, k + 2)], v3 = zb[ent<true>(a_cur, b_cur, k + 3)];
                            acc = __dadd_rn(acc, v0);
                            acc = __dadd_rn(acc, v1);
                            acc = __dadd_rn(acc, v2);
                            acc = __dadd_rn(acc, v3);
                        }
                    }
                    for (int k = 16; k < wd; k += 8) {  // rare long tiles
                        const uint4 x = __ldcs(ent16 + (int64_t)m_cur.x * 32 + (k >> 3) * 32 + lane);
#pragma unroll
                        for (int e = 0; e < 8; ++e) acc = __dadd_rn(acc, zb[ent<true>(x, x, e)]);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 8; k += 4) {
                        if (k < wd) {
                            const double v0 = __ldg(z + ent<false>(a_cur, b_cur, k)),
                                         v1 = __ldg(z + ent<false>(a_cur, b_cur, k + 1)),
                                         v2 = __ldg(z + ent<false>(a_cur, b_cur, k + 2)),
                                         v3 = __ldg(z + ent<false>(a_cur, b_cur, k + 3));
                            acc = __dadd_rn(acc, v0);
                            acc = __dadd_rn(acc, v1);
                            acc = __dadd_rn(acc, v2);
                            acc = __dadd_rn(acc, v3);
                        }
                    }
                    for (int k = 8; k < wd; k += 4) {
                        const uint4 x = __ldcs(ent16 + (int64_t)m_cur.x * 32 + (k >> 2) * 32 + lane);
#pragma unroll
                        for (int e = 0; e < 4; ++e) acc = __dadd_rn(acc, __ldg(z + ent<false>(x, x, e)));
                    }
                }
                p[j] = acc;
                a_cur = a_n;
                b_cur = b_n;
                m_cur = m_nxt;
                m_nxt = m_n2;
                ++t;
            }
        }
        if (dense) {
            __syncthreads();
            if (threadIdx.x == 0 && d + 2 < d1) issue_z(d + 2);
            ++d;
        }
    }
#pragma unroll
    for (int j = 0; j < MAXS; ++j) {
        const int i = w + 32 * j;
        const int64_t r = (int64_t)b * spb * 32 + i * 32 + lane;
        if (i < spb && r < n) out[r] = p[j];
    }
}

template <int Z, int MAXS>
__global__ void __launch_bounds__(1024, 1)
    k_panel8(const int *blk_g, const int *grp_panel, const int *blk_dense, const int *dense_panel,
             const int64_t *tbase, const uint2 *tiles, const uint4 *ent16, const double *z, int spb,
             int64_t n, double *out) {
    extern __shared__ __align__(128) double zs[];
    __shared__ uint64_t full[2];
    const int b = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    constexpr int kStride = Z + 16;
    const int g0 = blk_g[b], g1 = blk_g[b + 1];
    const int d0 = blk_dense[b], d1 = blk_dense[b + 1];
    constexpr uint32_t kChunk = 16384;
    auto issue_z = [&](int d) {
        const int buf = (d - d0) & 1;
        const double *src = z + (int64_t)dense_panel[d] * Z;
        mbar_expect(&full[buf], Z * 8);
        for (uint32_t o = 0; o < Z * 8u; o += kChunk)
            bulk_g2s((char *)(zs + buf * kStride) + o, (const char *)src + o, min(kChunk, Z * 8u - o),
                     &full[buf]);
    };
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 2) zs[threadIdx.x * kStride + Z] = 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
        if (d0 < d1) issue_z(d0);
        if (d0 + 1 < d1) issue_z(d0 + 1);
    }
    const int64_t t0 = tbase[b * 32 + w], t1 = tbase[b * 32 + w + 1];
    const int nsl = (spb - w + 31) / 32;  // slices of this warp (same in every group)
    int64_t tg = t0;                      // first tile of the current group
    uint2 mg = lane < nsl && tg + lane < t1 ? tiles[tg + lane] : make_uint2(0, 0);
    uint2 mgn = lane < nsl && tg + nsl + lane < t1 ? tiles[tg + nsl + lane] : make_uint2(0, 0);
    uint2 m_cur = make_uint2(__shfl_sync(0xffffffffu, mg.x, 0), __shfl_sync(0xffffffffu, mg.y, 0));
    const uint4 zero4 = make_uint4(0, 0, 0, 0);
    uint4 a_cur = zero4, b_cur = zero4;
    if (t0 < t1) {
        const uint4 *src = ent16 + (int64_t)m_cur.x * 32 + lane;
        a_cur = __ldcs(src);
        const int wd = m_cur.y & 0xffff, per = (m_cur.y >> 16) ? 8 : 4;
        if (wd > per) b_cur = __ldcs(src + 32);
    }
    double p[MAXS];
#pragma unroll
    for (int j = 0; j < MAXS; ++j) p[j] = 0.0;
    int d = d0;
    for (int g = g0; g < g1; ++g) {
        const bool dense = grp_panel[g] >= 0;
        const double *zb = zs + ((d - d0) & 1) * kStride;
        if (dense) mbar_wait(&full[(d - d0) & 1], ((d - d0) >> 1) & 1);
#pragma unroll
        for (int j = 0; j < MAXS; ++j) {
            if (w + 32 * j < spb) {
                // prefetch next tile's entries and the meta two ahead
                uint4 a_n = zero4, b_n = zero4;
                const bool lastj = j + 1 >= nsl;
                const uint2 m_nxt = make_uint2(__shfl_sync(0xffffffffu, lastj ? mgn.x : mg.x, lastj ? 0 : j + 1),
                                               __shfl_sync(0xffffffffu, lastj ? mgn.y : mg.y, lastj ? 0 : j + 1));
                const int64_t t = tg + j;
                if (t + 1 < t1) {
                    const uint4 *src = ent16 + (int64_t)m_nxt.x * 32 + lane;
                    a_n = __ldcs(src);
                    const int wd = m_nxt.y & 0xffff, per = (m_nxt.y >> 16) ? 8 : 4;
                    if (wd > per) b_n = __ldcs(src + 32);
                }
                const int wd = m_cur.y & 0xffff;
                double acc = p[j];
                if (dense) {
#pragma unroll
                    for (int k = 0; k < 16; k += 4) {
                        if (k < wd) {
                            const double v0 = zb[ent<true>(a_cur, b_cur, k)], v1 = zb[ent<true>(a_cur, b_cur, k + 1)],
                                         v2 = zb[ent<true>(a_cur, b_cur, k + 2)], v3 = zb[ent<true>(a_cur, b_cur, k + 3)];
                            acc = __dadd_rn(acc, v0);
                            acc = __dadd_rn(acc, v1);
                            acc = __dadd_rn(acc, v2);
                            acc = __dadd_rn(acc, v3);
                        }
                    }
                    for (int k = 16; k < wd; k += 8) {  // rare long tiles
                        const uint4 x = __ldcs(ent16 + (int64_t)m_cur.x * 32 + (k >> 3) * 32 + lane);
#pragma unroll
                        for (int e = 0; e < 8; ++e) acc = __dadd_rn(acc, zb[ent<true>(x, x, e)]);
                    }
                } else {
                    if (wd > 4) {
                        double v[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) v[e] = __ldg(z + ent<false>(a_cur, b_cur, e));
#pragma unroll
                        for (int e = 0; e < 8; ++e) acc = __dadd_rn(acc, v[e]);
                    } else if (wd > 0) {
                        double v[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) v[e] = __ldg(z + ent<false>(a_cur, a_cur, e));
#pragma unroll
                        for (int e = 0; e < 4; ++e) acc = __dadd_rn(acc, v[e]);
                    }
                    for (int k = 8; k < wd; k += 4) {
                        const uint4 x = __ldcs(ent16 + (int64_t)m_cur.x * 32 + (k >> 2) * 32 + lane);
#pragma unroll
                        for (int e = 0; e < 4; ++e) acc = __dadd_rn(acc, __ldg(z + ent<false>(x, x, e)));
                    }
                }
                p[j] = acc;
                a_cur = a_n;
                b_cur = b_n;
                m_cur = m_nxt;
            }
        }
        tg += nsl;
        mg = mgn;
        mgn = lane < nsl && tg + nsl + lane < t1 ? tiles[tg + nsl + lane] : make_uint2(0, 0);
        if (dense) {
            __syncthreads();
            if (threadIdx.x == 0 && d + 2 < d1) issue_z(d + 2);
            ++d;
        }
    }
#pragma unroll
    for (int j = 0; j < MAXS; ++j) {
        const int i = w + 32 * j;
        const int64_t r = (int64_t)b * spb * 32 + i * 32 + lane;
        if (i < spb && r < n) out[r] = p[j];
    }
}

static Layout3 build3(const std::vector<int64_t> &rp, const std::vector<int> &col, int64_t n, int spb,
                      int Z, int thresh) {
    Layout3 L;
    L.spb = spb;
    L.Z = Z;
    const int64_t R = (int64_t)spb * 32;
    L.G = (int)((n + R - 1) / R);
    L.S = (int)((n + Z - 1) / Z);
    L.blk_g.push_back(0);
    L.blk_dense.push_back(0);
    std::vector<int64_t> cnt(L.S);
    L.tbase.assign((size_t)L.G * 32 + 1, 0);
    std::vector<std::vector<uint2>> wt(32);
    for (int b = 0; b < L.G; ++b) {
        const int64_t r0 = b * R, r1 = std::min(n, r0 + R);
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t j = rp[r0]; j < rp[r1]; ++j) cnt[col[j] / Z]++;
        std::vector<std::array<int, 3>> groups;
        for (int s = 0; s < L.S; ++s) {
            if (cnt[s] >= thresh) groups.push_back({s, s + 1, 1});
            else if (cnt[s] > 0) {
                if (!groups.empty() && !groups.back()[2]) groups.back()[1] = s + 1;
                else groups.push_back({s, s + 1, 0});
            }
        }
        std::vector<int64_t> cur(R);
        for (int64_t r = r0; r < r0 + R; ++r) cur[r - r0] = r < n ? rp[r] : 0;
        for (auto &v : wt) v.clear();
        for (auto &gr : groups) {
            const int64_t clo = (int64_t)gr[0] * Z, chi = (int64_t)gr[1] * Z;
            const bool dn = gr[2];
            L.grp_off.push_back((uint32_t)(L.bytes.size() / 512));
            L.grp_panel.push_back(dn ? gr[0] : -1);
            L.grp_off.push_back((uint32_t)(L.bytes.size() / 512));
            if (dn) L.dense_panel.push_back(gr[0]);
            for (int i = 0; i < spb; ++i) {
                int wmax = 0, c[32];
                for (int l = 0; l < 32; ++l) {
                    const int64_t r = r0 + i * 32 + l;
                    int k = 0;
                    if (r < n)
                        while (cur[r - r0] + k < rp[r + 1] && col[cur[r - r0] + k] < chi) ++k;
                    c[l] = k;
                    wmax = std::max(wmax, k);
                }
                const int esz = dn ? 2 : 4, per = 16 / esz;  // entries per lane per 16-B chunk
                const int nch = (wmax + per - 1) / per;
                const size_t tile0 = L.bytes.size();
                L.bytes.resize(tile0 + (size_t)nch * 512);
                for (int q = 0; q < nch * per; ++q)
                    for (int l = 0; l < 32; ++l) {
                        const int64_t r = r0 + i * 32 + l;
                        uint8_t *dst = &L.bytes[tile0 + ((size_t)(q / per) * 32 + l) * 16 + (q % per) * esz];
                        if (dn) {
                            uint16_t v = q < c[l] ? (uint16_t)(col[cur[r - r0] + q] - clo) : (uint16_t)Z;
                            memcpy(dst, &v, 2);
                        } else {
                            int32_t v = q < c[l] ? col[cur[r - r0] + q] : (int32_t)n;
                            memcpy(dst, &v, 4);
                        }
                    }
                wt[i % 32].push_back(make_uint2((uint32_t)(tile0 / 512), (uint32_t)wmax | (dn << 16)));
                for (int l = 0; l < 32; ++l) {
                    const int64_t r = r0 + i * 32 + l;
                    if (r < n) cur[r - r0] += c[l];
                }
            }
        }
        for (int w = 0; w < 32; ++w) {
            L.tbase[(size_t)b * 32 + w] = (int64_t)L.tiles.size();
            L.tiles.insert(L.tiles.end(), wt[w].begin(), wt[w].end());
        }
        L.blk_g.push_back((int)L.grp_panel.size());
        L.blk_dense.push_back((int)L.dense_panel.size());
    }
    L.tbase[(size_t)L.G * 32] = (int64_t)L.tiles.size();
    L.grp_off.push_back((uint32_t)(L.bytes.size() / 512));
    L.bytes.resize(L.bytes.size() + 4096);
    return L;
}

template <int Z, int MAXS>
static void run3(const std::vector<int64_t> &rp, const std::vector<int> &col, int64_t n, int spb,
                 int thresh, const double *dz, const std::vector<double> &ref, double *dout) {
    Layout3 L = build3(rp, col, n, spb, Z, thresh);
    int *bg = up(L.blk_g), *gp = up(L.grp_panel), *bd = up(L.blk_dense), *dp = up(L.dense_panel);
    int64_t *tb = up(L.tbase);
    uint2 *ti = up(L.tiles);
    uint8_t *en = up(L.bytes);
    const size_t smem = 2 * (Z + 16) * 8;
    CK(cudaFuncSetAttribute(k_panel3<Z, MAXS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    auto launch = [&] {
        k_panel3<Z, MAXS><<<L.G, 1024, smem>>>(bg, gp, bd, dp, tb, ti, (const uint4 *)en, dz, spb, n, dout);
    };
    CK(cudaMemset(dout, 0, n * 8));
    launch();
    CK(cudaDeviceSynchronize());
    std::vector<double> got(n);
    CK(cudaMemcpy(got.data(), dout, n * 8, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) bad += memcmp(&got[i], &ref[i], 8) != 0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int r = 0; r < 3; ++r) launch();
    const int reps = 20;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("v3 Z %5d thresh %5d | tiles %zu bytes %.1f MB | %8.1f us  %6.1f GNNZ/s | bad %lld\n", Z, thresh,
           L.tiles.size(), L.bytes.size() / 1e6, ms * 1e3, col.size() / ms / 1e6, (long long)bad);
    cudaFree(bg), cudaFree(gp), cudaFree(bd), cudaFree(dp), cudaFree(tb), cudaFree(ti), cudaFree(en);
}

template <int Z, int MAXS>
static void run8(const std::vector<int64_t> &rp, const std::vector<int> &col, int64_t n, int spb,
                 int thresh, const double *dz, const std::vector<double> &ref, double *dout) {
    Layout3 L = build3(rp, col, n, spb, Z, thresh);
    int *bg = up(L.blk_g), *gp = up(L.grp_panel), *bd = up(L.blk_dense), *dp = up(L.dense_panel);
    int64_t *tb = up(L.tbase);
    uint2 *ti = up(L.tiles);
    uint8_t *en = up(L.bytes);
    const size_t smem = 2 * (Z + 16) * 8;
    CK(cudaFuncSetAttribute(k_panel8<Z, MAXS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    auto launch = [&] {
        k_panel8<Z, MAXS><<<L.G, 1024, smem>>>(bg, gp, bd, dp, tb, ti, (const uint4 *)en, dz, spb, n, dout);
    };
    CK(cudaMemset(dout, 0, n * 8));
    launch();
    CK(cudaDeviceSynchronize());
    std::vector<double> got(n);
    CK(cudaMemcpy(got.data(), dout, n * 8, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) bad += memcmp(&got[i], &ref[i], 8) != 0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int r = 0; r < 3; ++r) launch();
    const int reps = 20;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("v8 Z %5d thresh %5d | tiles %zu bytes %.1f MB | %8.1f us  %6.1f GNNZ/s | bad %lld\n", Z, thresh,
           L.tiles.size(), L.bytes.size() / 1e6, ms * 1e3, col.size() / ms / 1e6, (long long)bad);
    cudaFree(bg), cudaFree(gp), cudaFree(bd), cudaFree(dp), cudaFree(tb), cudaFree(ti), cudaFree(en);
}

// plain lane-per-row CSR (ground truth on device too)

// ---- version 9: producer warp streams (group, round) stages into a smem ring by bulk copies ----
constexpr int kNC = 31;  // consumer warps; warp 31 is the producer
struct Layout9 {
    int spb, G, S, Z, nr;
    std::vector<int> blk_g, grp_panel;
    std::vector<int> blk_s;      // per block + 1: stage range
    std::vector<uint2> stg;      // (offset16, bytes)
    std::vector<uint8_t> bytes, sbytes;
    size_t max_stage = 0;
};

static Layout9 build9(const std::vector<int64_t> &rp, const std::vector<int> &col, int64_t n, int spb,
                      int Z, int thresh) {
    Layout9 L;
    L.spb = spb;
    L.Z = Z;
    L.nr = (spb + kNC - 1) / kNC;
    const int64_t R = (int64_t)spb * 32;
    L.G = (int)((n + R - 1) / R);
    L.S = (int)((n + Z - 1) / Z);
    L.blk_g.push_back(0);
    L.blk_s.push_back(0);
    std::vector<int64_t> cnt(L.S);
    for (int b = 0; b < L.G; ++b) {
        const int64_t r0 = b * R, r1 = std::min(n, r0 + R);
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t j = rp[r0]; j < rp[r1]; ++j) cnt[col[j] / Z]++;
        std::vector<std::array<int, 3>> groups;
        for (int s = 0; s < L.S; ++s) {
            if (cnt[s] >= thresh) groups.push_back({s, s + 1, 1});
            else if (cnt[s] > 0) {
                if (!groups.empty() && !groups.back()[2]) groups.back()[1] = s + 1;
                else groups.push_back({s, s + 1, 0});
            }
        }
        std::vector<int64_t> cur(R);
        for (int64_t r = r0; r < r0 + R; ++r) cur[r - r0] = r < n ? rp[r] : 0;
        for (auto &gr : groups) {
            const int64_t clo = (int64_t)gr[0] * Z, chi = (int64_t)gr[1] * Z;
            const bool dn = gr[2];
            L.grp_panel.push_back(dn ? gr[0] : -1);
            const int esz = dn ? 2 : 4, per = 16 / esz;
            for (int j = 0; j < L.nr; ++j) {
                const size_t st0 = L.bytes.size();
                L.bytes.resize(st0 + 256);  // header: per consumer warp (off16, nch)
                uint2 hdr[32] = {};
                for (int w = 0; w < kNC; ++w) {
                    const int i = w + kNC * j;
                    if (i >= spb) continue;
                    int wmax = 0, c[32];
                    for (int l = 0; l < 32; ++l) {
                        const int64_t r = r0 + i * 32 + l;
                        int k = 0;
                        if (r < n)
                            while (cur[r - r0] + k < rp[r + 1] && col[cur[r - r0] + k] < chi) ++k;
                        c[l] = k;
                        wmax = std::max(wmax, k);
                    }
                    const int nch = (wmax + per - 1) / per;
                    std::vector<uint8_t> &tb = dn ? L.bytes : L.sbytes;
                    const size_t tile0 = tb.size();
                    hdr[w] = make_uint2(dn ? (uint32_t)((tile0 - st0) / 16) : (uint32_t)(tile0 / 16), (uint32_t)nch);
                    tb.resize(tile0 + (size_t)nch * 512);
                    for (int q = 0; q < nch * per; ++q)
                        for (int l = 0; l < 32; ++l) {
                            const int64_t r = r0 + i * 32 + l;
                            uint8_t *dst = &tb[tile0 + ((size_t)(q / per) * 32 + l) * 16 + (q % per) * esz];
                            if (dn) {
                                uint16_t v = q < c[l] ? (uint16_t)(col[cur[r - r0] + q] - clo) : (uint16_t)Z;
                                memcpy(dst, &v, 2);
                            } else {
                                int32_t v = q < c[l] ? col[cur[r - r0] + q] : (int32_t)n;
                                memcpy(dst, &v, 4);
                            }
                        }
                    for (int l = 0; l < 32; ++l) {
                        const int64_t r = r0 + i * 32 + l;
                        if (r < n) cur[r - r0] += c[l];
                    }
                }
                memcpy(&L.bytes[st0], hdr, 256);
                const size_t sz = L.bytes.size() - st0;
                L.max_stage = std::max(L.max_stage, sz);
                L.stg.push_back(make_uint2((uint32_t)(st0 / 16), (uint32_t)sz));
            }
        }
        L.blk_g.push_back((int)L.grp_panel.size());
        L.blk_s.push_back((int)L.stg.size());
    }
    L.bytes.resize(L.bytes.size() + 4096);
    L.sbytes.resize(L.sbytes.size() + 4096);
    return L;
}

__device__ __forceinline__ void mbar_arrive(uint64_t *m) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(m)) : "memory");
}

template <int Z, int MAXS, int NS, int SLOT>
__global__ void __launch_bounds__(1024, 1)
    k_panel9(const int *blk_g, const int *grp_panel, const int *blk_s, const uint2 *stg,
             const uint8_t *bytes, const uint4 *sent, const double *z, int spb, int nr, int64_t n, double *out) {
    extern __shared__ __align__(128) double zs[];  // 2 x (Z + 16) doubles | NS x SLOT stage ring
    __shared__ uint64_t full[NS], empty[NS], zfull[2], zempty[2];
    __shared__ int sgp[512];
    constexpr int kStride = Z + 16;
    uint8_t *ring = (uint8_t *)(zs + 2 * kStride);
    const int b = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g0 = blk_g[b], g1 = blk_g[b + 1];
    const int s0 = blk_s[b], s1 = blk_s[b + 1];
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kNC);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&zfull[i], 1);
            mbar_init(&zempty[i], kNC);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int g = g0 + threadIdx.x; g < g1; g += blockDim.x) sgp[g - g0] = grp_panel[g];
    if (threadIdx.x < 2) zs[threadIdx.x * kStride + Z] = 0.0;
    __syncthreads();
    if (w == kNC) {  // producer
        if (lane == 0) {
            int s = s0, d = 0;
            for (int g = g0; g < g1; ++g) {
                const int pan = sgp[g - g0];
                if (pan >= 0) {
                    const int buf = d & 1;
                    if (d >= 2) mbar_wait(&zempty[buf], ((d - 2) >> 1) & 1);
                    mbar_expect(&zfull[buf], Z * 8);
                    const char *src = (const char *)(z + (int64_t)pan * Z);
                    for (uint32_t o = 0; o < Z * 8u; o += 16384)
                        bulk_g2s((char *)(zs + buf * kStride) + o, src + o, min(16384u, Z * 8u - o), &zfull[buf]);
                    ++d;
                }
                for (int j = 0; j < nr; ++j, ++s) {
                    const int k = s - s0, slot = k % NS;
                    if (k >= NS) mbar_wait(&empty[slot], ((k / NS) - 1) & 1);
                    const uint2 sd = stg[s];
                    mbar_expect(&full[slot], sd.y);
                    const uint8_t *src = bytes + (int64_t)sd.x * 16;
                    for (uint32_t o = 0; o < sd.y; o += 16384)
                        bulk_g2s(ring + slot * SLOT + o, src + o, min(16384u, sd.y - o), &full[slot]);
                }
            }
        }
        return;
    }
    double p[MAXS];
#pragma unroll
    for (int j = 0; j < MAXS; ++j) p[j] = 0.0;
    int k = 0, d = 0;
    for (int g = g0; g < g1; ++g) {
        const bool dense = sgp[g - g0] >= 0;
        const double *zb = zs + (d & 1) * kStride;
        if (dense) mbar_wait(&zfull[d & 1], (d >> 1) & 1);
#pragma unroll
        for (int j = 0; j < MAXS; ++j) {
            if (j < nr) {
                const int slot = k % NS;
                mbar_wait(&full[slot], (k / NS) & 1);
                const uint8_t *st = ring + slot * SLOT;
                if (w + kNC * j < spb) {
                    const uint2 h = ((const uint2 *)st)[w];
                    const uint4 *e = dense ? (const uint4 *)(st + h.x * 16) + lane : sent + (int64_t)h.x + lane;
                    const int nch = h.y;
                    double acc = p[j];
                    for (int c = 0; c < nch; ++c) {
                        const uint4 x = dense ? e[32 * c] : __ldcs(e + 32 * c);
                        if (dense) {
                            const double v0 = zb[x.x & 0xffff], v1 = zb[x.x >> 16], v2 = zb[x.y & 0xffff],
                                         v3 = zb[x.y >> 16], v4 = zb[x.z & 0xffff], v5 = zb[x.z >> 16],
                                         v6 = zb[x.w & 0xffff], v7 = zb[x.w >> 16];
                            acc = __dadd_rn(acc, v0);
                            acc = __dadd_rn(acc, v1);
                            acc = __dadd_rn(acc, v2);
                            acc = __dadd_rn(acc, v3);
                            acc = __dadd_rn(acc, v4);
                            acc = __dadd_rn(acc, v5);
                            acc = __dadd_rn(acc, v6);
                            acc = __dadd_rn(acc, v7);
                        } else {
                            const double v0 = __ldg(z + (int)x.x), v1 = __ldg(z + (int)x.y),
                                         v2 = __ldg(z + (int)x.z), v3 = __ldg(z + (int)x.w);
                            acc = __dadd_rn(acc, v0);
                            acc = __dadd_rn(acc, v1);
                            acc = __dadd_rn(acc, v2);
                            acc = __dadd_rn(acc, v3);
                        }
                    }
                    p[j] = acc;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[slot]);
                ++k;
            }
        }
        if (dense) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&zempty[d & 1]);
            ++d;
        }
    }
#pragma unroll
    for (int j = 0; j < MAXS; ++j) {
        const int i = w + kNC * j;
        const int64_t r = (int64_t)b * spb * 32 + i * 32 + lane;
        if (i < spb && r < n) out[r] = p[j];
    }
}

template <int Z, int MAXS, int NS, int SLOT>
static void run9(const std::vector<int64_t> &rp, const std::vector<int> &col, int64_t n, int spb,
                 int thresh, const double *dz, const std::vector<double> &ref, double *dout) {
    Layout9 L = build9(rp, col, n, spb, Z, thresh);
    if (L.max_stage > SLOT) {
        printf("v9 Z %d: max stage %zu > slot %d\n", Z, L.max_stage, SLOT);
        return;
    }
    int *bg = up(L.blk_g), *gp = up(L.grp_panel), *bs = up(L.blk_s);
    uint2 *st = up(L.stg);
    uint8_t *by = up(L.bytes), *sb = up(L.sbytes);
    const size_t smem = 2 * (Z + 16) * 8 + (size_t)NS * SLOT;
    CK(cudaFuncSetAttribute(k_panel9<Z, MAXS, NS, SLOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    auto launch = [&] {
        k_panel9<Z, MAXS, NS, SLOT><<<L.G, 1024, smem>>>(bg, gp, bs, st, by, (const uint4 *)sb, dz, spb, L.nr, n, dout);
    };
    CK(cudaMemset(dout, 0, n * 8));
    launch();
    CK(cudaDeviceSynchronize());
    std::vector<double> got(n);
    CK(cudaMemcpy(got.data(), dout, n * 8, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) bad += memcmp(&got[i], &ref[i], 8) != 0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int r = 0; r < 3; ++r) launch();
    const int reps = 20;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("v9 Z %5d NS %d SLOT %d | stages %zu max %zu bytes %.1f MB | %8.1f us  %6.1f GNNZ/s | bad %lld\n", Z, NS,
           SLOT, L.stg.size(), L.max_stage, L.bytes.size() / 1e6, ms * 1e3, col.size() / ms / 1e6, (long long)bad);
    cudaFree(bg), cudaFree(gp), cudaFree(bs), cudaFree(st), cudaFree(by), cudaFree(sb);
}

__global__ void k_csr(const int64_t *rp, const int *col, const double *z, int64_t n, double *out) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    double acc = 0.0;
    for (int64_t j = rp[r]; j < rp[r + 1]; ++j) acc = __dadd_rn(acc, z[col[j]]);
    out[r] = acc;
}

int main(int argc, char **argv) {
    const int64_t n = 1000000, blk = 100000;
    std::vector<int> col;
    std::vector<int64_t> rp(1, 0);
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
        rp.push_back((int64_t)col.size());
    }
    const int64_t nnz = (int64_t)col.size();
    std::vector<double> z(n + 65536, 0.0);
    for (int64_t i = 0; i < n; ++i) z[i] = (double)(rnd() >> 11) * 0x1.0p-53 - 0.25;
    std::vector<double> ref(n);
    for (int64_t i = 0; i < n; ++i) {
        double a = 0.0;
        for (int64_t j = rp[i]; j < rp[i + 1]; ++j) a += z[col[j]];
        ref[i] = a;
    }
    double *dz, *dout;
    CK(cudaMalloc(&dz, z.size() * 8));
    CK(cudaMemcpy(dz, z.data(), z.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dout, n * 8));
    // baseline csr
    {
        int64_t *drp = up(rp);
        int *dcol = up(col);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int r = 0; r < 3; ++r) k_csr<<<(n + 255) / 256, 256>>>(drp, dcol, dz, n, dout);
        cudaEventRecord(e0);
        for (int r = 0; r < 20; ++r) k_csr<<<(n + 255) / 256, 256>>>(drp, dcol, dz, n, dout);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        std::vector<double> got(n);
        CK(cudaMemcpy(got.data(), dout, n * 8, cudaMemcpyDeviceToHost));
        int64_t bad = 0;
        for (int64_t i = 0; i < n; ++i) bad += memcmp(&got[i], &ref[i], 8) != 0;
        printf("csr lane-per-row: %.1f us (bad %lld) nnz %lld\n", ms / 20 * 1e3, (long long)bad,
               (long long)nnz);
        cudaFree(drp), cudaFree(dcol);
    }
    const int spb = (int)((n / 148 + 32) / 32 + 0);  // slices per block for ~148 blocks
    run8<12288, 7>(rp, col, n, 212, 2048, dz, ref, dout);
    run9<8192, 7, 4, 24576>(rp, col, n, 212, 2048, dz, ref, dout);
    run9<8192, 7, 3, 32768>(rp, col, n, 212, 2048, dz, ref, dout);
    run9<10240, 7, 2, 32768>(rp, col, n, 212, 2048, dz, ref, dout);
    run9<10240, 7, 3, 21504>(rp, col, n, 212, 2048, dz, ref, dout);
    (void)spb;
    (void)argc;
    (void)argv;
    return 0;
}
