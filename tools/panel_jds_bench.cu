// panel_jds_bench.cu -- column-panel SpMV with an UNPADDED index stream (probe, config-2 pattern).
//
// Follow-up to panel_bench.cu, whose ELL tiles were 2-3x padded. Same panel idea (dense column
// panels of z staged in shared memory by TMA, sparse remainder gathered from L2, lane = row for
// the whole step so every row is summed in stored column order), but each (group, 32-row slice)
// tile is stored jagged-diagonal style: diagonal k holds the k-th entry of every lane whose count
// in this group exceeds k, packed in lane order. A lane finds its entry with one ballot:
// pos = D_k + popc(ballot(c > k) & lanemask_lt). Per tile only the 32 one-byte counts are stored.
// All of a CTA's tiles of one group form one "stage" that a single thread bulk-copies into a
// shared-memory ring (TMA, mbarrier completion), so the index stream moves in large transfers.
//
// Stage layout (16-byte aligned): u32 woff[32] (byte offset of warp w's entries) | u8 cnt[spb][32]
// | entries, warp-major (warp w's tiles j = 0.. in order, u16 panel-local or u32 global indices).
// Usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o panel_jds_bench panel_jds_bench.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
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
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes)
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
__device__ __forceinline__ void bulk_issue(void *dst, const void *src, uint32_t bytes, uint64_t *m) {
    mbar_expect(m, bytes);
    for (uint32_t o = 0; o < bytes; o += 32768)
        bulk_g2s((char *)dst + o, (const char *)src + o, min(32768u, bytes - o), m);
}

template <typename T>
static T *up(const std::vector<T> &v) {
    T *d;
    CK(cudaMalloc(&d, v.size() * sizeof(T) + 64));
    CK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}

struct LayoutJ {
    int spb = 0, G = 0, Z = 0;
    std::vector<int> blk_g;      // per CTA + 1: group range
    std::vector<int> grp_panel;  // dense: panel id, sparse: -1
    std::vector<uint2> stg;      // per group: (byte offset / 16, bytes)
    std::vector<uint8_t> bytes;
    size_t max_stage = 0;
    size_t entry_bytes = 0, header_bytes = 0;
};

// Groups of one CTA: panels with >= thresh entries are dense; runs of the others form sparse
// groups, cut so that a sparse stage stays below `budget` bytes.
static LayoutJ buildJ(const std::vector<int64_t> &rp, const std::vector<int> &col, int64_t n, int spb, int Z,
                      int thresh, size_t budget) {
    LayoutJ L;
    L.spb = spb;
    L.Z = Z;
    const int64_t R = (int64_t)spb * 32;
    L.G = (int)((n + R - 1) / R);
    const int S = (int)((n + Z - 1) / Z);
    L.blk_g.push_back(0);
    std::vector<int64_t> cnt(S);
    const size_t hdr = 128 + (size_t)spb * 32;
    for (int b = 0; b < L.G; ++b) {
        const int64_t r0 = b * R, r1 = std::min(n, r0 + R);
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t j = rp[r0]; j < rp[r1]; ++j) cnt[col[j] / Z]++;
        std::vector<std::array<int, 3>> groups;  // (panel lo, panel hi, dense)
        size_t run = 0;
        for (int s = 0; s < S; ++s) {
            if (cnt[s] >= thresh) {
                groups.push_back({s, s + 1, 1});
            } else if (cnt[s] > 0) {
                const size_t add = (size_t)cnt[s] * 4 + 64;
                if (!groups.empty() && !groups.back()[2] && groups.back()[1] == s && run + add + hdr <= budget) {
                    groups.back()[1] = s + 1;
                    run += add;
                } else {
                    groups.push_back({s, s + 1, 0});
                    run = add;
                }
            }
        }
        std::vector<int64_t> cur(R);
        for (int64_t r = r0; r < r0 + R; ++r) cur[r - r0] = r < n ? rp[r] : 0;
        for (auto &gr : groups) {
            const int64_t clo = (int64_t)gr[0] * Z, chi = std::min<int64_t>((int64_t)gr[1] * Z, n);
            const bool dn = gr[2];
            const int esz = dn ? 2 : 4;
            L.grp_panel.push_back(dn ? gr[0] : -1);
            std::vector<uint8_t> st(hdr, 0);
            uint32_t woff[32];
            for (int w = 0; w < 32; ++w) {
                while (st.size() % 4) st.push_back(0);
                woff[w] = (uint32_t)st.size();
                for (int i = w; i < spb; i += 32) {
                    int c[32], mx = 0;
                    for (int l = 0; l < 32; ++l) {
                        const int64_t r = r0 + (int64_t)i * 32 + l;
                        int k = 0;
                        if (r < n)
                            while (cur[r - r0] + k < rp[r + 1] && col[cur[r - r0] + k] < chi) ++k;
                        if (k > 255) {
                            printf("count > 255\n");
                            exit(1);
                        }
                        c[l] = k;
                        mx = std::max(mx, k);
                        st[128 + (size_t)i * 32 + l] = (uint8_t)k;
                    }
                    for (int k = 0; k < mx; ++k)
                        for (int l = 0; l < 32; ++l)
                            if (c[l] > k) {
                                const int64_t r = r0 + (int64_t)i * 32 + l;
                                const int v = col[cur[r - r0] + k];
                                if (dn) {
                                    const uint16_t u = (uint16_t)(v - clo);
                                    st.insert(st.end(), (uint8_t *)&u, (uint8_t *)&u + 2);
                                } else {
                                    st.insert(st.end(), (uint8_t *)&v, (uint8_t *)&v + 4);
                                }
                                L.entry_bytes += esz;
                            }
                    for (int l = 0; l < 32; ++l) {
                        const int64_t r = r0 + (int64_t)i * 32 + l;
                        if (r < n) cur[r - r0] += c[l];
                    }
                }
            }
            memcpy(st.data(), woff, 128);
            while (st.size() % 16) st.push_back(0);
            L.header_bytes += hdr;
            L.max_stage = std::max(L.max_stage, st.size());
            L.stg.push_back(make_uint2((uint32_t)(L.bytes.size() / 16), (uint32_t)st.size()));
            L.bytes.insert(L.bytes.end(), st.begin(), st.end());
        }
        L.blk_g.push_back((int)L.grp_panel.size());
    }
    L.bytes.resize(L.bytes.size() + 4096);
    return L;
}

template <int Z, int MAXS, int NS, bool COMPUTE = true>
__global__ void __launch_bounds__(1024, 1)
    k_pj(const int *__restrict__ blk_g, const int *__restrict__ grp_panel, const uint2 *__restrict__ stg,
         const uint8_t *__restrict__ bytes, const double *__restrict__ z, int spb, int slot_bytes, int64_t n,
         double *__restrict__ out) {
    extern __shared__ __align__(128) double zs[];  // 2 x (Z + 16) doubles | NS x slot ring
    __shared__ uint64_t sfull[NS], zfull[2];
    constexpr int kStride = Z + 16;
    uint8_t *ring = (uint8_t *)(zs + 2 * kStride);
    const int b = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g0 = blk_g[b], g1 = blk_g[b + 1];
    const uint32_t lt = (1u << lane) - 1u;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) mbar_init(&sfull[i], 1);
        for (int i = 0; i < 2; ++i) mbar_init(&zfull[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // prologue: first NS stages, first two dense panels
        for (int g = g0; g < g1 && g < g0 + NS; ++g) {
            const uint2 sd = stg[g];
            bulk_issue(ring + (g - g0) * slot_bytes, bytes + (int64_t)sd.x * 16, sd.y, &sfull[g - g0]);
        }
        int d = 0;
        for (int g = g0; g < g1 && d < 2; ++g)
            if (grp_panel[g] >= 0) {
                bulk_issue(zs + d * kStride, z + (int64_t)grp_panel[g] * Z, Z * 8, &zfull[d]);
                ++d;
            }
    }
    __syncthreads();
    double p[MAXS];
#pragma unroll
    for (int j = 0; j < MAXS; ++j) p[j] = 0.0;
    int d = 0;
    int next_dense = g0;  // scan position for the dense panel two ahead
    {
        int seen = 0;
        while (next_dense < g1 && seen < 2) {
            if (grp_panel[next_dense] >= 0) ++seen;
            ++next_dense;
        }
    }
    for (int g = g0; g < g1; ++g) {
        const int k = g - g0, slot = k % NS;
        const bool dense = grp_panel[g] >= 0;
        const double *zb = zs + (d & 1) * kStride;
        const uint8_t *st = ring + slot * slot_bytes;
        mbar_wait(&sfull[slot], (k / NS) & 1);
        if (dense) mbar_wait(&zfull[d & 1], (d >> 1) & 1);
        uint32_t off = ((const uint32_t *)st)[w];
#pragma unroll
        for (int j = 0; j < MAXS; ++j) {
            const int i = w + 32 * j;
            if (i < spb) {
                const int c = st[128 + i * 32 + lane];
                const int mx = __reduce_max_sync(0xffffffffu, c);
                double acc = p[j];
                if (dense) {
                    const uint16_t *e = (const uint16_t *)(st + off);
                    int D = 0;
                    for (int kk = 0; kk < mx; kk += 4) {
                        double v[4];
                        bool on[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint32_t B = __ballot_sync(0xffffffffu, c > kk + u);
                            on[u] = c > kk + u;
                            const int pos = D + __popc(B & lt);
                            D += __popc(B);
                            v[u] = on[u] ? zb[e[pos]] : 0.0;
                        }
                        if (COMPUTE) {
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                if (on[u]) acc = __dadd_rn(acc, v[u]);
                        } else {
                            acc += v[0];
                        }
                    }
                    off += D * 2;
                } else {
                    off = (off + 3) & ~3u;
                    const uint32_t *e = (const uint32_t *)(st + off);
                    int D = 0;
                    for (int kk = 0; kk < mx; kk += 4) {
                        double v[4];
                        bool on[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint32_t B = __ballot_sync(0xffffffffu, c > kk + u);
                            on[u] = c > kk + u;
                            const int pos = D + __popc(B & lt);
                            D += __popc(B);
                            v[u] = on[u] ? __ldg(z + e[pos]) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (on[u]) acc = __dadd_rn(acc, v[u]);
                    }
                    off += D * 4;
                }
                p[j] = acc;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (g + NS < g1) {
                const uint2 sd = stg[g + NS];
                bulk_issue(ring + slot * slot_bytes, bytes + (int64_t)sd.x * 16, sd.y, &sfull[slot]);
            }
            if (dense) {
                while (next_dense < g1 && grp_panel[next_dense] < 0) ++next_dense;
                if (next_dense < g1) {
                    bulk_issue(zs + (d & 1) * kStride, z + (int64_t)grp_panel[next_dense] * Z, Z * 8, &zfull[d & 1]);
                    ++next_dense;
                }
            }
        }
        if (dense) ++d;
    }
#pragma unroll
    for (int j = 0; j < MAXS; ++j) {
        const int i = w + 32 * j;
        const int64_t r = (int64_t)b * spb * 32 + i * 32 + lane;
        if (i < spb && r < n) out[r] = p[j];
    }
}

template <int Z, int MAXS, int NS, bool COMPUTE = true>
static void runJ(const std::vector<int64_t> &rp, const std::vector<int> &col, int64_t n, int spb, int thresh,
                 const double *dz, const std::vector<double> &ref, double *dout) {
    const size_t zbytes = 2 * (size_t)(Z + 16) * 8;
    const size_t avail = 232448 - 256 - zbytes;
    const size_t slot_cap = (avail / NS) & ~(size_t)127;
    LayoutJ L = buildJ(rp, col, n, spb, Z, thresh, slot_cap);
    if (L.max_stage > slot_cap) {
        printf("J Z %d NS %d: max stage %zu > slot %zu\n", Z, NS, L.max_stage, slot_cap);
        return;
    }
    const int slot = (int)((L.max_stage + 127) & ~(size_t)127);
    int *bg = up(L.blk_g), *gp = up(L.grp_panel);
    uint2 *st = up(L.stg);
    uint8_t *by = up(L.bytes);
    const size_t smem = zbytes + (size_t)NS * slot;
    CK(cudaFuncSetAttribute(k_pj<Z, MAXS, NS, COMPUTE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    auto launch = [&] { k_pj<Z, MAXS, NS, COMPUTE><<<L.G, 1024, smem>>>(bg, gp, st, by, dz, spb, slot, n, dout); };
    CK(cudaMemset(dout, 0, n * 8));
    launch();
    CK(cudaGetLastError());
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
    int ndense = 0;
    for (int x : L.grp_panel) ndense += x >= 0;
    printf("J%s Z %5d NS %d thr %4d | groups %zu (dense %d) slot %d stream %.1f MB (entries %.1f hdr %.1f) | %7.1f us "
           "%6.1f GNNZ/s | bad %lld\n",
           COMPUTE ? "" : "(nocompute)", Z, NS, thresh, L.grp_panel.size(), ndense, slot, L.bytes.size() / 1e6,
           L.entry_bytes / 1e6, L.header_bytes / 1e6, ms * 1e3, col.size() / ms / 1e6, (long long)bad);
    cudaFree(bg), cudaFree(gp), cudaFree(st), cudaFree(by);
}


// ---- v11: segment-sorted stages, partial sums in shared memory ----
// A (CTA, group) stage lists the "segments" (row, entries of that row in the group's column
// range) sorted by entry count, descending, padded to warp-iterations of 32 segments with one
// count each: u32 hdr[nq] (entry base | count << 24) | u16 row[32 nq] | entries, per
// warp-iteration diagonal-major (entry k of segment s at base + 32 k + s). Every lane adds its
// segment's entries to partial[row] in order; rows appear once per stage, stages are ordered by
// column, so each row is still summed in stored column order.
struct LayoutS {
    int R = 0, G = 0, Z = 0;
    std::vector<int> blk_g, grp_panel;
    std::vector<uint2> stg;   // (byte offset / 16, bytes)
    std::vector<uint32_t> nq; // per group: warp-iterations
    std::vector<uint32_t> roff;  // per group: byte offset of the row ids in the stage
    std::vector<uint32_t> eoff;  // per group: byte offset of the entries
    std::vector<uint8_t> bytes;
    size_t max_stage = 0, pad_entries = 0, entries = 0, segs = 0;
};

static LayoutS buildS(const std::vector<int64_t> &rp, const std::vector<int> &col, int64_t n, int R, int Z,
                      int thresh, size_t budget, int nw = 0) {
    LayoutS L;
    L.R = R;
    L.Z = Z;
    L.G = (int)((n + R - 1) / R);
    const int S = (int)((n + Z - 1) / Z);
    L.blk_g.push_back(0);
    std::vector<int64_t> cnt(S);
    for (int b = 0; b < L.G; ++b) {
        const int64_t r0 = (int64_t)b * R, r1 = std::min(n, r0 + R);
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t j = rp[r0]; j < rp[r1]; ++j) cnt[col[j] / Z]++;
        std::vector<std::array<int, 3>> groups;
        size_t run = 0;
        for (int s = 0; s < S; ++s) {
            if (cnt[s] >= thresh) {
                groups.push_back({s, s + 1, 1});
            } else if (cnt[s] > 0) {
                const size_t add = (size_t)cnt[s] * 7 + 256;
                if (!groups.empty() && !groups.back()[2] && groups.back()[1] == s && run + add <= budget) {
                    groups.back()[1] = s + 1;
                    run += add;
                } else {
                    groups.push_back({s, s + 1, 0});
                    run = add;
                }
            }
        }
        std::vector<int64_t> cur(r1 - r0);
        for (int64_t r = r0; r < r1; ++r) cur[r - r0] = rp[r];
        for (auto &gr : groups) {
            const int64_t clo = (int64_t)gr[0] * Z, chi = std::min<int64_t>((int64_t)gr[1] * Z, n);
            const bool dn = gr[2];
            L.grp_panel.push_back(dn ? gr[0] : -1);
            std::vector<std::pair<int, int>> seg;  // (count, local row)
            for (int64_t r = r0; r < r1; ++r) {
                int k = 0;
                while (cur[r - r0] + k < rp[r + 1] && col[cur[r - r0] + k] < chi) ++k;
                if (k) seg.push_back({k, (int)(r - r0)});
            }
            std::vector<uint32_t> wq(33, 0);
            if (nw) {  // per-warp row ranges, each padded to whole iterations
                const int rw = (R + nw - 1) / nw;
                std::vector<std::pair<int, int>> out;
                size_t a = 0;
                for (int w = 0; w < 32; ++w) {
                    wq[w] = (uint32_t)(out.size() / 32);
                    size_t e = a;
                    while (e < seg.size() && seg[e].second < (w + 1) * rw) ++e;
                    std::vector<std::pair<int, int>> part(seg.begin() + a, seg.begin() + e);
                    std::stable_sort(part.begin(), part.end(), [](auto &x, auto &y) { return x.first > y.first; });
                    out.insert(out.end(), part.begin(), part.end());
                    while (out.size() % 32) out.push_back({0, R});
                    a = e;
                }
                wq[32] = (uint32_t)(out.size() / 32);
                seg.swap(out);
            } else {
                std::stable_sort(seg.begin(), seg.end(), [](auto &a, auto &b) { return a.first > b.first; });
            }
            const int nq = (int)((seg.size() + 31) / 32);
            std::vector<uint32_t> hdr(nq);
            std::vector<uint16_t> rows((size_t)nq * 32, (uint16_t)R);
            std::vector<uint8_t> ent;
            uint32_t base = 0;
            for (int q = 0; q < nq; ++q) {
                const int c = seg[(size_t)q * 32].first;
                hdr[q] = base | ((uint32_t)c << 24);
                for (int k = 0; k < c; ++k)
                    for (int l = 0; l < 32; ++l) {
                        const size_t si = (size_t)q * 32 + l;
                        int64_t v;
                        if (si < seg.size() && seg[si].first > k && seg[si].second < R) {
                            const int lr = seg[si].second;
                            v = col[cur[lr] + k];
                            if (dn) v -= clo;
                            ++L.entries;
                        } else {
                            v = dn ? Z : n;
                            ++L.pad_entries;
                        }
                        if (dn) {
                            const uint16_t u = (uint16_t)v;
                            ent.insert(ent.end(), (uint8_t *)&u, (uint8_t *)&u + 2);
                        } else {
                            const uint32_t u = (uint32_t)v;
                            ent.insert(ent.end(), (uint8_t *)&u, (uint8_t *)&u + 4);
                        }
                    }
                for (int l = 0; l < 32; ++l) {
                    const size_t si = (size_t)q * 32 + l;
                    if (si < seg.size() && seg[si].second < R) rows[si] = (uint16_t)seg[si].second;
                }
                base += (uint32_t)c * 32;
            }
            for (auto &sg : seg)
                if (sg.second < R) cur[sg.second] += sg.first, ++L.segs;
            std::vector<uint8_t> st;
            if (nw) st.insert(st.end(), (uint8_t *)wq.data(), (uint8_t *)wq.data() + 128);
            st.insert(st.end(), (uint8_t *)hdr.data(), (uint8_t *)hdr.data() + hdr.size() * 4);
            while (st.size() % 16) st.push_back(0);
            L.roff.push_back((uint32_t)st.size());
            st.insert(st.end(), (uint8_t *)rows.data(), (uint8_t *)rows.data() + rows.size() * 2);
            while (st.size() % 16) st.push_back(0);
            L.eoff.push_back((uint32_t)st.size());
            st.insert(st.end(), ent.begin(), ent.end());
            while (st.size() % 16) st.push_back(0);
            L.nq.push_back((uint32_t)nq);
            L.max_stage = std::max(L.max_stage, st.size());
            L.stg.push_back(make_uint2((uint32_t)(L.bytes.size() / 16), (uint32_t)st.size()));
            L.bytes.insert(L.bytes.end(), st.begin(), st.end());
        }
        L.blk_g.push_back((int)L.grp_panel.size());
    }
    L.bytes.resize(L.bytes.size() + 4096);
    return L;
}

struct GrpMeta {
    int panel;
    uint32_t nq, roff, eoff;
};

template <int Z, int NS>
__global__ void __launch_bounds__(1024, 1)
    k_ps(const int *__restrict__ blk_g, const GrpMeta *__restrict__ meta, const uint2 *__restrict__ stg,
         const uint8_t *__restrict__ bytes, const double *__restrict__ z, int R, int slot_bytes, int64_t n,
         double *__restrict__ out) {
    extern __shared__ __align__(128) double zs[];  // 2 x (Z + 16) | partial[R + 16] | NS x slot
    __shared__ uint64_t sfull[NS], zfull[2];
    constexpr int kStride = Z + 16;
    double *part = zs + 2 * kStride;
    uint8_t *ring = (uint8_t *)(part + ((R + 16 + 15) & ~15));
    const int b = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g0 = blk_g[b], g1 = blk_g[b + 1];
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) mbar_init(&sfull[i], 1);
        for (int i = 0; i < 2; ++i) mbar_init(&zfull[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int g = g0; g < g1 && g < g0 + NS; ++g) {
            const uint2 sd = stg[g];
            bulk_issue(ring + (g - g0) * slot_bytes, bytes + (int64_t)sd.x * 16, sd.y, &sfull[g - g0]);
        }
        int d = 0;
        for (int g = g0; g < g1 && d < 2; ++g)
            if (meta[g].panel >= 0) {
                bulk_issue(zs + d * kStride, z + (int64_t)meta[g].panel * Z, Z * 8, &zfull[d]);
                ++d;
            }
    }
    for (int i = threadIdx.x; i < R + 16; i += blockDim.x) part[i] = 0.0;
    if (threadIdx.x < 2) zs[threadIdx.x * kStride + Z] = 0.0;
    int next_dense = g0;
    {
        int seen = 0;
        while (next_dense < g1 && seen < 2) {
            if (meta[next_dense].panel >= 0) ++seen;
            ++next_dense;
        }
    }
    __syncthreads();
    int d = 0;
    for (int g = g0; g < g1; ++g) {
        const int k = g - g0, slot = k % NS;
        const GrpMeta m = meta[g];
        const bool dense = m.panel >= 0;
        const double *zb = zs + (d & 1) * kStride;
        const uint8_t *st = ring + slot * slot_bytes;
        mbar_wait(&sfull[slot], (k / NS) & 1);
        if (dense) mbar_wait(&zfull[d & 1], (d >> 1) & 1);
        const uint32_t *hdr = (const uint32_t *)st;
        const uint16_t *rows = (const uint16_t *)(st + m.roff);
        if (dense) {
            const uint16_t *ent = (const uint16_t *)(st + m.eoff);
            for (uint32_t q = w; q < m.nq; q += 32) {
                const uint32_t h = hdr[q];
                const int c = h >> 24;
                const uint16_t *e = ent + (h & 0xffffff) + lane;
                const int row = rows[q * 32 + lane];
                double acc = part[row];
                int kk = 0;
                for (; kk + 4 <= c; kk += 4) {
                    const int i0 = e[32 * kk], i1 = e[32 * kk + 32], i2 = e[32 * kk + 64], i3 = e[32 * kk + 96];
                    const double v0 = zb[i0], v1 = zb[i1], v2 = zb[i2], v3 = zb[i3];
                    acc = __dadd_rn(acc, v0);
                    acc = __dadd_rn(acc, v1);
                    acc = __dadd_rn(acc, v2);
                    acc = __dadd_rn(acc, v3);
                }
                for (; kk < c; ++kk) acc = __dadd_rn(acc, zb[e[32 * kk]]);
                part[row] = acc;
            }
        } else {
            const uint32_t *ent = (const uint32_t *)(st + m.eoff);
            for (uint32_t q = w; q < m.nq; q += 32) {
                const uint32_t h = hdr[q];
                const int c = h >> 24;
                const uint32_t *e = ent + (h & 0xffffff) + lane;
                const int row = rows[q * 32 + lane];
                double acc = part[row];
                int kk = 0;
                for (; kk + 4 <= c; kk += 4) {
                    const uint32_t i0 = e[32 * kk], i1 = e[32 * kk + 32], i2 = e[32 * kk + 64], i3 = e[32 * kk + 96];
                    const double v0 = __ldg(z + i0), v1 = __ldg(z + i1), v2 = __ldg(z + i2), v3 = __ldg(z + i3);
                    acc = __dadd_rn(acc, v0);
                    acc = __dadd_rn(acc, v1);
                    acc = __dadd_rn(acc, v2);
                    acc = __dadd_rn(acc, v3);
                }
                for (; kk < c; ++kk) acc = __dadd_rn(acc, __ldg(z + e[32 * kk]));
                part[row] = acc;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (g + NS < g1) {
                const uint2 sd = stg[g + NS];
                bulk_issue(ring + slot * slot_bytes, bytes + (int64_t)sd.x * 16, sd.y, &sfull[slot]);
            }
            if (dense) {
                while (next_dense < g1 && meta[next_dense].panel < 0) ++next_dense;
                if (next_dense < g1) {
                    bulk_issue(zs + (d & 1) * kStride, z + (int64_t)meta[next_dense].panel * Z, Z * 8, &zfull[d & 1]);
                    ++next_dense;
                }
            }
        }
        if (dense) ++d;
    }
    const int64_t r0 = (int64_t)b * R;
    for (int i = threadIdx.x; i < R; i += blockDim.x)
        if (r0 + i < n) out[r0 + i] = part[i];
}


// ---- v12: warps own row ranges (no CTA barrier per group), producer warp, empty barriers ----
__device__ __forceinline__ void mbar_arrive(uint64_t *m) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(m)) : "memory");
}
constexpr int kCW = 31;  // consumer warps

template <int Z, int NS>
__global__ void __launch_bounds__(1024, 1)
    k_pw(const int *__restrict__ blk_g, const GrpMeta *__restrict__ meta, const uint2 *__restrict__ stg,
         const uint8_t *__restrict__ bytes, const double *__restrict__ z, int R, int slot_bytes, int64_t n,
         double *__restrict__ out) {
    extern __shared__ __align__(128) double zs[];
    __shared__ uint64_t sfull[NS], sempty[NS], zfull[2], zempty[2];
    constexpr int kStride = Z + 16;
    double *part = zs + 2 * kStride;
    uint8_t *ring = (uint8_t *)(part + ((R + 16 + 15) & ~15));
    const int b = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g0 = blk_g[b], g1 = blk_g[b + 1];
    const int rw = (R + kCW - 1) / kCW;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) mbar_init(&sfull[i], 1), mbar_init(&sempty[i], kCW);
        for (int i = 0; i < 2; ++i) mbar_init(&zfull[i], 1), mbar_init(&zempty[i], kCW);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 2) zs[threadIdx.x * kStride + Z] = 0.0;
    if (threadIdx.x == 32) part[R] = 0.0;
    __syncthreads();
    if (w == kCW) {
        if (lane == 0) {
            int d = 0;
            for (int g = g0; g < g1; ++g) {
                const int k = g - g0, slot = k % NS;
                if (k >= NS) mbar_wait(&sempty[slot], ((k / NS) - 1) & 1);
                const uint2 sd = stg[g];
                bulk_issue(ring + slot * slot_bytes, bytes + (int64_t)sd.x * 16, sd.y, &sfull[slot]);
                const int pan = meta[g].panel;
                if (pan >= 0) {
                    if (d >= 2) mbar_wait(&zempty[d & 1], ((d >> 1) - 1) & 1);
                    bulk_issue(zs + (d & 1) * kStride, z + (int64_t)pan * Z, Z * 8, &zfull[d & 1]);
                    ++d;
                }
            }
        }
        return;
    }
    const int lo = w * rw, hi = min(R, lo + rw);
    for (int i = lo + lane; i < hi; i += 32) part[i] = 0.0;
    __syncwarp();
    int d = 0;
    for (int g = g0; g < g1; ++g) {
        const int k = g - g0, slot = k % NS;
        const GrpMeta m = meta[g];
        const bool dense = m.panel >= 0;
        const double *zb = zs + (d & 1) * kStride;
        const uint8_t *st = ring + slot * slot_bytes;
        mbar_wait(&sfull[slot], (k / NS) & 1);
        if (dense) mbar_wait(&zfull[d & 1], (d >> 1) & 1);
        const uint32_t q0 = ((const uint32_t *)st)[w], q1 = ((const uint32_t *)st)[w + 1];
        const uint32_t *hdr = (const uint32_t *)st + 32;
        const uint16_t *rows = (const uint16_t *)(st + m.roff);
        if (dense) {
            const uint16_t *ent = (const uint16_t *)(st + m.eoff);
            for (uint32_t q = q0; q < q1; ++q) {
                const uint32_t h = hdr[q];
                const int c = h >> 24;
                const uint16_t *e = ent + (h & 0xffffff) + lane;
                const int row = rows[q * 32 + lane];
                double acc = part[row];
                int kk = 0;
                for (; kk + 4 <= c; kk += 4) {
                    const int i0 = e[32 * kk], i1 = e[32 * kk + 32], i2 = e[32 * kk + 64], i3 = e[32 * kk + 96];
                    const double v0 = zb[i0], v1 = zb[i1], v2 = zb[i2], v3 = zb[i3];
                    acc = __dadd_rn(acc, v0);
                    acc = __dadd_rn(acc, v1);
                    acc = __dadd_rn(acc, v2);
                    acc = __dadd_rn(acc, v3);
                }
                for (; kk < c; ++kk) acc = __dadd_rn(acc, zb[e[32 * kk]]);
                part[row] = acc;
            }
        } else {
            const uint32_t *ent = (const uint32_t *)(st + m.eoff);
            for (uint32_t q = q0; q < q1; ++q) {
                const uint32_t h = hdr[q];
                const int c = h >> 24;
                const uint32_t *e = ent + (h & 0xffffff) + lane;
                const int row = rows[q * 32 + lane];
                double acc = part[row];
                int kk = 0;
                for (; kk + 4 <= c; kk += 4) {
                    const uint32_t i0 = e[32 * kk], i1 = e[32 * kk + 32], i2 = e[32 * kk + 64], i3 = e[32 * kk + 96];
                    const double v0 = __ldg(z + i0), v1 = __ldg(z + i1), v2 = __ldg(z + i2), v3 = __ldg(z + i3);
                    acc = __dadd_rn(acc, v0);
                    acc = __dadd_rn(acc, v1);
                    acc = __dadd_rn(acc, v2);
                    acc = __dadd_rn(acc, v3);
                }
                for (; kk < c; ++kk) acc = __dadd_rn(acc, __ldg(z + e[32 * kk]));
                part[row] = acc;
            }
        }
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&sempty[slot]);
            if (dense) mbar_arrive(&zempty[d & 1]);
        }
        if (dense) ++d;
    }
    __syncwarp();
    const int64_t r0 = (int64_t)b * R;
    for (int i = lo + lane; i < hi; i += 32)
        if (r0 + i < n) out[r0 + i] = part[i];
}

template <int Z, int NS>
static void runW(const std::vector<int64_t> &rp, const std::vector<int> &col, int64_t n, int R, int thresh,
                 const double *dz, const std::vector<double> &ref, double *dout) {
    const size_t zbytes = 2 * (size_t)(Z + 16) * 8 + (size_t)((R + 16 + 15) & ~15) * 8;
    const size_t avail = 232448 - 256 - zbytes;
    const size_t slot_cap = (avail / NS) & ~(size_t)127;
    LayoutS L = buildS(rp, col, n, R, Z, thresh, slot_cap, kCW);
    if (L.max_stage > slot_cap) {
        printf("W Z %d R %d NS %d: max stage %zu > slot %zu\n", Z, R, NS, L.max_stage, slot_cap);
        return;
    }
    const int slot = (int)((L.max_stage + 127) & ~(size_t)127);
    std::vector<GrpMeta> meta(L.grp_panel.size());
    for (size_t g = 0; g < meta.size(); ++g) meta[g] = {L.grp_panel[g], L.nq[g], L.roff[g], L.eoff[g]};
    int *bg = up(L.blk_g);
    GrpMeta *dm = up(meta);
    uint2 *st = up(L.stg);
    uint8_t *by = up(L.bytes);
    const size_t smem = zbytes + (size_t)NS * slot;
    CK(cudaFuncSetAttribute(k_pw<Z, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    auto launch = [&] { k_pw<Z, NS><<<L.G, 1024, smem>>>(bg, dm, st, by, dz, R, slot, n, dout); };
    CK(cudaMemset(dout, 0, n * 8));
    launch();
    CK(cudaGetLastError());
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
    printf("W Z %5d R %5d NS %d thr %4d | CTAs %d groups %zu slot %d stream %.1f MB segs %.1fM pad %.2fM | "
           "%7.1f us %6.1f GNNZ/s | bad %lld\n",
           Z, R, NS, thresh, L.G, L.grp_panel.size(), slot, L.bytes.size() / 1e6, L.segs / 1e6,
           L.pad_entries / 1e6, ms * 1e3, col.size() / ms / 1e6, (long long)bad);
    cudaFree(bg), cudaFree(dm), cudaFree(st), cudaFree(by);
}

template <int Z, int NS>
static void runS(const std::vector<int64_t> &rp, const std::vector<int> &col, int64_t n, int R, int thresh,
                 const double *dz, const std::vector<double> &ref, double *dout) {
    const size_t zbytes = 2 * (size_t)(Z + 16) * 8 + (size_t)((R + 16 + 15) & ~15) * 8;
    if (zbytes + 256 > 232448) {
        printf("S Z %d R %d: no room\n", Z, R);
        return;
    }
    const size_t avail = 232448 - 256 - zbytes;
    const size_t slot_cap = (avail / NS) & ~(size_t)127;
    LayoutS L = buildS(rp, col, n, R, Z, thresh, slot_cap);
    if (L.max_stage > slot_cap) {
        printf("S Z %d R %d NS %d: max stage %zu > slot %zu\n", Z, R, NS, L.max_stage, slot_cap);
        return;
    }
    const int slot = (int)((L.max_stage + 127) & ~(size_t)127);
    std::vector<GrpMeta> meta(L.grp_panel.size());
    for (size_t g = 0; g < meta.size(); ++g) meta[g] = {L.grp_panel[g], L.nq[g], L.roff[g], L.eoff[g]};
    int *bg = up(L.blk_g);
    GrpMeta *dm = up(meta);
    uint2 *st = up(L.stg);
    uint8_t *by = up(L.bytes);
    const size_t smem = zbytes + (size_t)NS * slot;
    CK(cudaFuncSetAttribute(k_ps<Z, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    auto launch = [&] { k_ps<Z, NS><<<L.G, 1024, smem>>>(bg, dm, st, by, dz, R, slot, n, dout); };
    CK(cudaMemset(dout, 0, n * 8));
    launch();
    CK(cudaGetLastError());
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
    int ndense = 0;
    for (int x : L.grp_panel) ndense += x >= 0;
    printf("S Z %5d R %5d NS %d thr %4d | CTAs %d groups %zu (dense %d) slot %d stream %.1f MB segs %.1fM pad %.2fM | "
           "%7.1f us %6.1f GNNZ/s | bad %lld\n",
           Z, R, NS, thresh, L.G, L.grp_panel.size(), ndense, slot, L.bytes.size() / 1e6, L.segs / 1e6,
           L.pad_entries / 1e6, ms * 1e3, col.size() / ms / 1e6, (long long)bad);
    cudaFree(bg), cudaFree(dm), cudaFree(st), cudaFree(by);
}


// ---- v13: NW warps per CTA, ZB panel buffers (several CTAs per SM hide each other's
// barrier and panel-load waits) ----
template <int Z, int NS, int NW, int ZB>
__global__ void __launch_bounds__(NW * 32)
    k_ps2(const int *__restrict__ blk_g, const GrpMeta *__restrict__ meta, const uint2 *__restrict__ stg,
          const uint8_t *__restrict__ bytes, const double *__restrict__ z, int R, int slot_bytes, int64_t n,
          double *__restrict__ out) {
    extern __shared__ __align__(128) double zs[];  // ZB x (Z + 16) | partial[R + 16] | NS x slot
    __shared__ uint64_t sfull[NS], zfull[ZB];
    constexpr int kStride = Z + 16;
    double *part = zs + ZB * kStride;
    uint8_t *ring = (uint8_t *)(part + ((R + 16 + 15) & ~15));
    const int b = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g0 = blk_g[b], g1 = blk_g[b + 1];
    int next_dense = g0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) mbar_init(&sfull[i], 1);
        for (int i = 0; i < ZB; ++i) mbar_init(&zfull[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int g = g0; g < g1 && g < g0 + NS; ++g) {
            const uint2 sd = stg[g];
            bulk_issue(ring + (g - g0) * slot_bytes, bytes + (int64_t)sd.x * 16, sd.y, &sfull[g - g0]);
        }
        int d = 0;
        for (; next_dense < g1 && d < ZB; ++next_dense)
            if (meta[next_dense].panel >= 0) {
                bulk_issue(zs + d * kStride, z + (int64_t)meta[next_dense].panel * Z, Z * 8, &zfull[d]);
                ++d;
            }
    }
    for (int i = threadIdx.x; i < R + 16; i += blockDim.x) part[i] = 0.0;
    if (threadIdx.x < ZB) zs[threadIdx.x * kStride + Z] = 0.0;
    __syncthreads();
    int d = 0;
    for (int g = g0; g < g1; ++g) {
        const int k = g - g0, slot = k % NS;
        const GrpMeta m = meta[g];
        const bool dense = m.panel >= 0;
        const double *zb = zs + (d % ZB) * kStride;
        const uint8_t *st = ring + slot * slot_bytes;
        mbar_wait(&sfull[slot], (k / NS) & 1);
        if (dense) mbar_wait(&zfull[d % ZB], (d / ZB) & 1);
        const uint32_t *hdr = (const uint32_t *)st;
        const uint16_t *rows = (const uint16_t *)(st + m.roff);
        if (dense) {
            const uint16_t *ent = (const uint16_t *)(st + m.eoff);
            for (uint32_t q = w; q < m.nq; q += NW) {
                const uint32_t h = hdr[q];
                const int c = h >> 24;
                const uint16_t *e = ent + (h & 0xffffff) + lane;
                const int row = rows[q * 32 + lane];
                double acc = part[row];
                int kk = 0;
                for (; kk + 4 <= c; kk += 4) {
                    const int i0 = e[32 * kk], i1 = e[32 * kk + 32], i2 = e[32 * kk + 64], i3 = e[32 * kk + 96];
                    const double v0 = zb[i0], v1 = zb[i1], v2 = zb[i2], v3 = zb[i3];
                    acc = __dadd_rn(acc, v0);
                    acc = __dadd_rn(acc, v1);
                    acc = __dadd_rn(acc, v2);
                    acc = __dadd_rn(acc, v3);
                }
                for (; kk < c; ++kk) acc = __dadd_rn(acc, zb[e[32 * kk]]);
                part[row] = acc;
            }
        } else {
            const uint32_t *ent = (const uint32_t *)(st + m.eoff);
            for (uint32_t q = w; q < m.nq; q += NW) {
                const uint32_t h = hdr[q];
                const int c = h >> 24;
                const uint32_t *e = ent + (h & 0xffffff) + lane;
                const int row = rows[q * 32 + lane];
                double acc = part[row];
                int kk = 0;
                for (; kk + 4 <= c; kk += 4) {
                    const uint32_t i0 = e[32 * kk], i1 = e[32 * kk + 32], i2 = e[32 * kk + 64], i3 = e[32 * kk + 96];
                    const double v0 = __ldg(z + i0), v1 = __ldg(z + i1), v2 = __ldg(z + i2), v3 = __ldg(z + i3);
                    acc = __dadd_rn(acc, v0);
                    acc = __dadd_rn(acc, v1);
                    acc = __dadd_rn(acc, v2);
                    acc = __dadd_rn(acc, v3);
                }
                for (; kk < c; ++kk) acc = __dadd_rn(acc, __ldg(z + e[32 * kk]));
                part[row] = acc;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (g + NS < g1) {
                const uint2 sd = stg[g + NS];
                bulk_issue(ring + slot * slot_bytes, bytes + (int64_t)sd.x * 16, sd.y, &sfull[slot]);
            }
            if (dense) {
                while (next_dense < g1 && meta[next_dense].panel < 0) ++next_dense;
                if (next_dense < g1) {
                    bulk_issue(zs + (d % ZB) * kStride, z + (int64_t)meta[next_dense].panel * Z, Z * 8,
                               &zfull[d % ZB]);
                    ++next_dense;
                }
            }
        }
        if (dense) ++d;
    }
    const int64_t r0 = (int64_t)b * R;
    for (int i = threadIdx.x; i < R; i += blockDim.x)
        if (r0 + i < n) out[r0 + i] = part[i];
}

template <int Z, int NS, int NW, int ZB>
static void runS2(const std::vector<int64_t> &rp, const std::vector<int> &col, int64_t n, int R, int thresh,
                  int ctas_per_sm, const double *dz, const std::vector<double> &ref, double *dout) {
    const size_t fixed = ZB * (size_t)(Z + 16) * 8 + (size_t)((R + 16 + 15) & ~15) * 8;
    const size_t per_cta = (228 * 1024) / ctas_per_sm - 1024 - 256;
    if (fixed + 4096 > per_cta) {
        printf("S2: no room\\n");
        return;
    }
    const size_t slot_cap = ((per_cta - fixed) / NS) & ~(size_t)127;
    LayoutS L = buildS(rp, col, n, R, Z, thresh, slot_cap);
    if (L.max_stage > slot_cap) {
        printf("S2 Z %d R %d NS %d NW %d ZB %d: max stage %zu > slot %zu\\n", Z, R, NS, NW, ZB, L.max_stage, slot_cap);
        return;
    }
    const int slot = (int)((L.max_stage + 127) & ~(size_t)127);
    std::vector<GrpMeta> meta(L.grp_panel.size());
    for (size_t g = 0; g < meta.size(); ++g) meta[g] = {L.grp_panel[g], L.nq[g], L.roff[g], L.eoff[g]};
    int *bg = up(L.blk_g);
    GrpMeta *dm = up(meta);
    uint2 *st = up(L.stg);
    uint8_t *by = up(L.bytes);
    const size_t smem = fixed + (size_t)NS * slot;
    CK(cudaFuncSetAttribute(k_ps2<Z, NS, NW, ZB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ps2<Z, NS, NW, ZB>, NW * 32, smem));
    auto launch = [&] { k_ps2<Z, NS, NW, ZB><<<L.G, NW * 32, smem>>>(bg, dm, st, by, dz, R, slot, n, dout); };
    CK(cudaMemset(dout, 0, n * 8));
    launch();
    CK(cudaGetLastError());
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
    printf("S2 Z %5d R %5d NS %d NW %2d ZB %d occ %d | CTAs %d groups %zu smem %zu | %7.1f us %6.1f GNNZ/s | bad %lld\\n",
           Z, R, NS, NW, ZB, occ, L.G, L.grp_panel.size(), smem, ms * 1e3, col.size() / ms / 1e6, (long long)bad);
    cudaFree(bg), cudaFree(dm), cudaFree(st), cudaFree(by);
}

int main(int argc, char **argv) {
    int64_t n = 1000000;
    const int64_t blk = 100000;
    std::vector<int> col;
    std::vector<int64_t> rp(1, 0);
    if (argc > 2) {  // load a CSR: argv[2] = prefix of <prefix>.rp (int64) / <prefix>.col (int32)
        FILE *f = fopen((std::string(argv[2]) + ".rp").c_str(), "rb");
        fseek(f, 0, SEEK_END);
        n = ftell(f) / 8 - 1;
        fseek(f, 0, SEEK_SET);
        rp.resize(n + 1);
        fread(rp.data(), 8, n + 1, f);
        fclose(f);
        col.resize(rp[n]);
        f = fopen((std::string(argv[2]) + ".col").c_str(), "rb");
        fread(col.data(), 4, rp[n], f);
        fclose(f);
    }
    col.reserve(n * 44);
    uint64_t s = 0x9E3779B97F4A7C15ULL;
    auto rnd = [&]() {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        return s;
    };
    std::vector<int> row;
    for (int64_t i = 0; i < n && argc <= 2; ++i) {
        row.clear();
        const int64_t b = i / blk;
        for (int t = 0; t < 40; ++t) row.push_back((int)(b * blk + rnd() % blk));
        for (int t = 0; t < 4; ++t) row.push_back((int)(rnd() % n));
        std::sort(row.begin(), row.end());
        col.insert(col.end(), row.begin(), row.end());
        rp.push_back((int64_t)col.size());
    }
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
    printf("nnz %zu\n", col.size());
    if (argc > 1) {
        runS<8192, 2>(rp, col, n, 3392, 1024, dz, ref, dout);
        runS2<8192, 2, 32, 2>(rp, col, n, 3392, 1024, 1, dz, ref, dout);
        runS2<8192, 2, 16, 1>(rp, col, n, 1696, 512, 2, dz, ref, dout);
        runS2<8192, 2, 16, 1>(rp, col, n, 1696, 1024, 2, dz, ref, dout);
        runS2<4096, 2, 16, 2>(rp, col, n, 1696, 512, 2, dz, ref, dout);
        runS2<8192, 3, 16, 1>(rp, col, n, 1696, 512, 2, dz, ref, dout);
        runS2<4096, 2, 8, 2>(rp, col, n, 1696, 512, 3, dz, ref, dout);
        runS2<4096, 2, 10, 1>(rp, col, n, 1184, 256, 3, dz, ref, dout);
        return 0;
    }
    return 0;
}
