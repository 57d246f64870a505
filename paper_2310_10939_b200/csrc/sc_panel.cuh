// sc_panel.cuh -- column-panel layout and SpMV step for graphs whose vertex ids carry locality
// (included by sc_graph.cu after the handle and the SELL layout are defined).
//
// Why: the SELL kernel gathers every z value from L2 and runs at the L1->L2 random-request
// limit (one 8-byte gather per SM-cycle).  When a block of rows references a
// few contiguous column ranges heavily (planted-partition graphs numbered by block), those
// ranges ("panels" of kPanZ doubles) can be staged in shared memory by TMA and gathered there
// at many per cycle; the thin remainder is gathered from L2.
//
// Exactness: a lane adds its row's entries strictly in stored column order.  Rows are split
// into "segments" (row, entries of the row inside one group of columns); groups of a CTA are
// disjoint column ranges processed in increasing column order with a CTA barrier between
// them, and a row's running sum lives in shared memory (part[row]) between its segments, so
// every row sum is the same left-to-right chain as scipy's csr_matvec.  Padding entries add
// +0.0, an exact no-op (a running sum that starts at +0.0 is never -0.0).
//
// Layout (built on the device from the SELL arrays, so it works on renumbered ids):
//   CTA b owns renumbered rows [b*rpc, (b+1)*rpc), rpc = kPanR unless stages would overflow
//   the ring (then halved until they fit).  Its columns are cut into groups:
//   a panel (kPanZ columns) with >= kPanThresh of the CTA's entries is a dense group (z panel
//   staged in shared memory, 16-bit panel-local indices); runs of the other panels form sparse
//   groups (32-bit indices, z gathered from global memory).  One group's data is a "stage":
//     u32 hdr[nq]      iteration q: entry base | count << 24
//     u16 row[32 nq]   local row of each segment (kPanR = dummy)
//     entries          iteration q, entry k of lane l at base + 32 k + l
//   Segments are sorted by decreasing count, so the 32 segments of an iteration have (nearly)
//   the same count and the warp runs without divergence (k_pan_balance then places them in
//   lanes bank-aware for part[]); one thread streams the stages into
//   a shared-memory ring with bulk copies (cp.async.bulk + mbarrier).  Sparse padding entries
//   index z[ncols], a zero slot kept past the vector (sc_graph::zstride > ncols for whole
//   graphs; shard callers pass z buffers with the same padding, see sc_graph_build_panels).
// This header is included inside namespace sc.

constexpr int kPanZ = 8192;        // panel width in doubles (64 KB)
constexpr int kPanR = 3392;        // rows per CTA (106 slices)
constexpr int kPanNS = 2;          // stage ring depth
constexpr int kPanGMax = 48;       // groups per CTA
constexpr int kPanCMax = 128;      // entries per segment (exclusive bound)
constexpr int kPanThresh = 1024;   // entries of a CTA in a panel that make it dense
constexpr double kPanMinCover = 0.5;  // fraction of entries in dense panels the layout needs
constexpr double kPanMinSegment = 2.5;  // mean entries per dense segment it needs
constexpr int kPanSMax = 16384;    // panels (n <= 134M)
constexpr int kPanTPB = 1024;
constexpr int kPanZBytes = 2 * (kPanZ + 16) * 8;
constexpr int kPanPartLen = (kPanR + 32);  // + dummy row slot, padded
constexpr int kPanFixedSmem = kPanZBytes + kPanPartLen * 8;
constexpr int kPanSmemMax = 232448 - 256;

struct PanGroup {
    int32_t panel;   // dense: panel id; sparse: -1
    uint32_t nq;     // warp-iterations
    uint32_t roff;   // byte offset of the row ids in the stage
    uint32_t eoff;   // byte offset of the entries
    uint64_t off;    // byte offset of the stage in the stream
    uint32_t bytes;  // stage bytes (multiple of 16)
    uint32_t unused;
};

__device__ __forceinline__ uint32_t pan_smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void pan_mbar_init(uint64_t *m, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(pan_smem_u32(m)), "r"(count));
}
__device__ __forceinline__ void pan_mbar_wait(uint64_t *m, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n PW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra PW;\n}\n" ::"r"(pan_smem_u32(m)),
        "r"(phase)
        : "memory");
}
// bulk copy global -> shared of `bytes` (multiple of 16, both addresses 16-byte aligned),
// completing on mbarrier m
__device__ __forceinline__ void pan_bulk(void *dst, const void *src, uint32_t bytes, uint64_t *m) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(pan_smem_u32(m)),
                 "r"(bytes)
                 : "memory");
    for (uint32_t o = 0; o < bytes; o += 32768)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(pan_smem_u32((char *)dst + o)),
            "l"((const char *)src + o), "r"(min(32768u, bytes - o)), "r"(pan_smem_u32(m))
            : "memory");
}

struct PanArgs {
    const int32_t *blk;      // per CTA + 1: group range
    const PanGroup *grp;
    const uint8_t *stream;   // stages
    int64_t n;               // rows
    int64_t ncols;           // z space length; z[ncols] is a zero slot (padding target)
    int slot;                // ring slot bytes
    int rpc;                 // rows per CTA (<= kPanR, multiple of 32)
};

// Walks the entries of local row i of CTA b in the SELL layout (stored order).
template <typename F>
__device__ __forceinline__ void pan_row_walk(const int64_t *slice_ptr, const uint32_t *col, int64_t r,
                                             F &&f) {
    const int64_t sl = r >> 5;
    const int lane = (int)(r & 31);
    const int64_t base = slice_ptr[sl];
    const int width = (int)((slice_ptr[sl + 1] - base) >> 5);
    for (int t = 0; t < width; ++t) {
        const uint32_t c = __ldg(col + base + 32 * (int64_t)t + lane);
        if (c == kPad) break;
        f(c);
    }
}

// ---- the step kernel ----
template <bool SYM>
__global__ void __launch_bounds__(kPanTPB, 1) k_rw_panel(StepArgs a, PanArgs p) {
    extern __shared__ __align__(128) double zs[];  // 2 x (Z + 16) | part | ring
    __shared__ uint64_t sfull[kPanNS], zfull[2], efull;
    __shared__ int s_epi;  // panel buffer holding the epilogue's x_in / scale rows (-1: none)
    constexpr int kStride = kPanZ + 16;
    double *part = zs + 2 * kStride;
    uint8_t *ring = (uint8_t *)(part + kPanPartLen);
    const int b = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g0 = p.blk[b], g1 = p.blk[b + 1];
    const double *z = a.z_in;
    const int64_t r0 = (int64_t)b * p.rpc;
    const int rows_here = (int)((p.n - r0) < p.rpc ? (p.n - r0) : p.rpc);
    auto panel_bytes = [&](int pan) {
        const int64_t left = p.ncols - (int64_t)pan * kPanZ;
        return (uint32_t)(((left < kPanZ ? left : kPanZ) * 8 + 15) & ~15);
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < kPanNS; ++i) pan_mbar_init(&sfull[i], 1);
        for (int i = 0; i < 2; ++i) pan_mbar_init(&zfull[i], 1);
        pan_mbar_init(&efull, 1);
        s_epi = -1;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int g = g0; g < g1 && g < g0 + kPanNS; ++g) {
            const PanGroup m = p.grp[g];
            pan_bulk(ring + (g - g0) * p.slot, p.stream + m.off, m.bytes, &sfull[g - g0]);
        }
        int d = 0;
        for (int g = g0; g < g1 && d < 2; ++g) {
            const int pan = p.grp[g].panel;
            if (pan >= 0) {
                pan_bulk(zs + d * kStride, z + (int64_t)pan * kPanZ, panel_bytes(pan), &zfull[d]);
                ++d;
            }
        }
    }
    for (int i = threadIdx.x; i < kPanPartLen; i += kPanTPB) part[i] = 0.0;
    if (threadIdx.x < 2) zs[threadIdx.x * kStride + kPanZ] = 0.0;  // dense padding slot
    int next_dense = g0;  // thread 0: the dense group whose panel is fetched next
    if (threadIdx.x == 0) {
        int seen = 0;
        while (next_dense < g1 && seen < 2) seen += p.grp[next_dense++].panel >= 0;
    }
    __syncthreads();
    int d = 0;
    for (int g = g0; g < g1; ++g) {
        const int k = g - g0, slot = k % kPanNS;
        const PanGroup m = p.grp[g];
        const bool dense = m.panel >= 0;
        const double *zb = zs + (d & 1) * kStride;
        const uint8_t *st = ring + slot * p.slot;
        pan_mbar_wait(&sfull[slot], (k / kPanNS) & 1);
        if (dense) pan_mbar_wait(&zfull[d & 1], (d >> 1) & 1);
        const uint32_t *hdr = (const uint32_t *)st;
        const uint16_t *rows = (const uint16_t *)(st + m.roff);
        if (dense) {
            const uint16_t *ent = (const uint16_t *)(st + m.eoff);
            for (uint32_t q = w; q < m.nq; q += kPanTPB / 32) {
                const uint32_t h = hdr[q];
                const int c = h >> 24;
                const uint16_t *e = ent + (h & 0xffffff) + lane;
                const int row = rows[q * 32 + lane];
                double acc = part[row];
                int kk = 0;
                for (; kk + 4 <= c; kk += 4) {
                    const int i0 = e[32 * kk], i1 = e[32 * kk + 32], i2 = e[32 * kk + 64],
                              i3 = e[32 * kk + 96];
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
            // sparse groups gather from global memory; padding entries point at z[n], a zero
            // slot past the vector (sc_graph zstride)
            const uint32_t *ent = (const uint32_t *)(st + m.eoff);
            for (uint32_t q = w; q < m.nq; q += kPanTPB / 32) {
                const uint32_t h = hdr[q];
                const int c = h >> 24;
                const uint32_t *e = ent + (h & 0xffffff) + lane;
                const int row = rows[q * 32 + lane];
                double acc = part[row];
                int kk = 0;
                for (; kk + 4 <= c; kk += 4) {
                    const uint32_t i0 = e[32 * kk], i1 = e[32 * kk + 32], i2 = e[32 * kk + 64],
                                   i3 = e[32 * kk + 96];
                    const double v0 = __ldg(z + i0), v1 = __ldg(z + i1), v2 = __ldg(z + i2),
                                 v3 = __ldg(z + i3);
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
            if (g + kPanNS < g1) {
                const PanGroup mn = p.grp[g + kPanNS];
                pan_bulk(ring + slot * p.slot, p.stream + mn.off, mn.bytes, &sfull[slot]);
            }
            if (dense) {
                while (next_dense < g1 && p.grp[next_dense].panel < 0) ++next_dense;
                if (next_dense < g1) {
                    const int pan = p.grp[next_dense].panel;
                    pan_bulk(zs + (d & 1) * kStride, z + (int64_t)pan * kPanZ, panel_bytes(pan),
                             &zfull[d & 1]);
                    ++next_dense;
                } else if (s_epi < 0 && !(rows_here & 1)) {
                    // no dense panel left: this buffer is free for the rest of the kernel, so the
                    // epilogue's x_in and scale rows are prefetched into it
                    s_epi = d & 1;
                    double *eb = zs + (d & 1) * kStride;
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                                     pan_smem_u32(&efull)),
                                 "r"((uint32_t)rows_here * 16u)
                                 : "memory");
                    for (int h = 0; h < 2; ++h) {
                        const double *src = (h ? a.scale : a.x_in) + r0;
                        for (uint32_t o = 0; o < (uint32_t)rows_here * 8u; o += 32768)
                            asm volatile(
                                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
                                "[%1], %2, [%3];" ::"r"(pan_smem_u32((char *)(eb + h * rows_here) + o)),
                                "l"((const char *)src + o), "r"(min(32768u, (uint32_t)rows_here * 8u - o)),
                                "r"(pan_smem_u32(&efull))
                                : "memory");
                    }
                }
            }
        }
        if (dense) ++d;
    }
    __syncthreads();  // s_epi
    const int epi = s_epi;
    if (epi >= 0) pan_mbar_wait(&efull, 0);
    const double *eb = zs + epi * kStride;
    // epilogue: all loads of this thread's (<= 4) rows first, so the CTA pays one memory
    // latency here, not one per row (the stores below could alias the loads for the compiler)
    static_assert(kPanR <= 4 * kPanTPB, "epilogue handles at most 4 rows per thread");
    double xr[4], sv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int i = threadIdx.x + j * kPanTPB;
        const bool ld = i < rows_here;
        if (epi >= 0) {
            xr[j] = ld ? eb[i] : 0.0;
            sv[j] = ld ? eb[rows_here + i] : 1.0;
        } else {
            xr[j] = ld ? __ldcs(a.x_in + r0 + i) : 0.0;
            sv[j] = ld ? __ldcs(a.scale + r0 + i) : 1.0;
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int i = threadIdx.x + j * kPanTPB;
        if (i < rows_here) row_epilogue<SYM>(a, r0 + i, part[i], xr[j], sv[j]);
    }
}

// ---- layout construction (device) ----
struct PanPlan {
    int32_t lo, hi, dense, bytes;  // panel range, dense flag, stage bytes
};
struct PanPlanQ {
    uint32_t nq, roff, eoff, ent;  // iterations, offsets, entries incl. padding
};

// Per CTA: panel histogram -> groups -> segment histogram per (group, count) -> stage sizes.
// flag[0] |= 1 (too many groups), 2 (segment longer than kPanCMax - 1), 4 (stage > slot cap),
// 8 (a row's stored order goes back to an earlier group);
// flag[1] = max stage bytes; cover[0] / cover[1] / cover[2] += entries in dense panels / all
// entries / dense segments.
__global__ void __launch_bounds__(kPanTPB) k_pan_plan(const int64_t *slice_ptr, const uint32_t *col,
                                                      int64_t n, int S, int rpc, uint32_t slot_cap,
                                                      int32_t *cta_ng, PanPlan *plan, PanPlanQ *planq,
                                                      int32_t *flag, unsigned long long *cover) {
    extern __shared__ uint32_t psm[];
    uint32_t *hist = psm;                  // S: entries per panel, then panel -> group
    uint32_t *h2 = psm + S;                // kPanGMax x kPanCMax segment counts
    __shared__ PanPlan gt[kPanGMax];
    __shared__ int ng_s, bad_s;
    const int b = blockIdx.x;
    const int64_t r0 = (int64_t)b * rpc;
    const int rows = (int)((n - r0) < rpc ? (n - r0) : rpc);
    for (int i = threadIdx.x; i < S; i += kPanTPB) hist[i] = 0;
    for (int i = threadIdx.x; i < kPanGMax * kPanCMax; i += kPanTPB) h2[i] = 0;
    if (threadIdx.x == 0) bad_s = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < rows; i += kPanTPB)
        pan_row_walk(slice_ptr, col, r0 + i, [&](uint32_t c) { atomicAdd(&hist[c / kPanZ], 1u); });
    __syncthreads();
    if (threadIdx.x < 32) {  // warp 0: groups in column order
        const int lane = threadIdx.x;
        int ng = 0, last_sparse = 0;
        uint32_t run = 0;
        unsigned long long dense_e = 0, all_e = 0;
        const uint32_t budget = slot_cap - slot_cap / 10;
        for (int s0 = 0; s0 < S; s0 += 32) {
            const uint32_t c = s0 + lane < S ? hist[s0 + lane] : 0;
            uint32_t nz = __ballot_sync(0xffffffffu, c != 0);
            while (nz) {
                const int l = __ffs(nz) - 1;
                nz &= nz - 1;
                const uint32_t cs = __shfl_sync(0xffffffffu, c, l);
                const int s = s0 + l;
                const uint32_t est = cs * 13 / 2;  // ~ stage bytes per entry (idx + row + hdr)
                if (lane == 0) {
                    all_e += cs;
                    if (cs >= (uint32_t)kPanThresh) dense_e += cs;
                    if (cs >= (uint32_t)kPanThresh) {
                        if (ng < kPanGMax) gt[ng] = {s, s + 1, 1, 0};
                        ++ng;
                        last_sparse = 0;
                    } else if (last_sparse && run + est <= budget) {
                        gt[ng - 1].hi = s + 1;
                        run += est;
                    } else {
                        if (ng < kPanGMax) gt[ng] = {s, s + 1, 0, 0};
                        ++ng;
                        last_sparse = 1;
                        run = 1024 + est;
                    }
                }
                ng = __shfl_sync(0xffffffffu, ng, 0);
                last_sparse = __shfl_sync(0xffffffffu, last_sparse, 0);
                run = __shfl_sync(0xffffffffu, run, 0);
            }
        }
        if (lane == 0) {
            ng_s = ng;
            if (ng > kPanGMax) bad_s |= 1;
            atomicAdd(&cover[0], dense_e);
            atomicAdd(&cover[1], all_e);
        }
    }
    __syncthreads();
    const int ng = min(ng_s, kPanGMax);
    for (int g = 0; g < ng; ++g)
        for (int s = gt[g].lo + (int)threadIdx.x; s < gt[g].hi; s += kPanTPB) hist[s] = g;
    __syncthreads();
    if (!bad_s) {
        for (int i = threadIdx.x; i < rows; i += kPanTPB) {
            int cur = -1, cnt = 0;
            pan_row_walk(slice_ptr, col, r0 + i, [&](uint32_t c) {
                const int g = (int)hist[c / kPanZ];
                if (g != cur) {
                    // a row must visit its groups in increasing order (its stored column order
                    // must not go back to an earlier panel): renamed shard columns, BFS
                    // pre-orders or unsorted input rows can break that -> decline
                    if (g < cur) atomicOr(&bad_s, 8);
                    if (cnt) {
                        if (cnt >= kPanCMax) atomicOr(&bad_s, 2);
                        else atomicAdd(&h2[cur * kPanCMax + cnt], 1u);
                    }
                    cur = g;
                    cnt = 0;
                }
                ++cnt;
            });
            if (cnt) {
                if (cnt >= kPanCMax) atomicOr(&bad_s, 2);
                else atomicAdd(&h2[cur * kPanCMax + cnt], 1u);
            }
        }
    }
    __syncthreads();
    for (int g = threadIdx.x; g < ng; g += kPanTPB) {
        uint32_t pos = 0, ent = 0;
        for (int c = kPanCMax - 1; c >= 1; --c) {
            const uint32_t h = h2[g * kPanCMax + c];
            if (!h) continue;
            const uint32_t q0 = (pos + 31) / 32, q1 = (pos + h + 31) / 32;
            ent += (q1 - q0) * 32 * (uint32_t)c;
            pos += h;
        }
        const uint32_t nq = (pos + 31) / 32;
        if (gt[g].dense) atomicAdd(&cover[2], (unsigned long long)pos);
        const uint32_t esz = gt[g].dense ? 2 : 4;
        const uint32_t roff = (4 * nq + 15) & ~15u;
        const uint32_t eoff = roff + ((64 * nq + 15) & ~15u);
        const uint32_t bytes = eoff + ((ent * esz + 15) & ~15u);
        if (bytes > slot_cap) atomicOr(&bad_s, 4);
        atomicMax(&flag[1], (int32_t)bytes);
        PanPlan pl = gt[g];
        pl.bytes = (int32_t)bytes;
        plan[(int64_t)b * kPanGMax + g] = pl;
        planq[(int64_t)b * kPanGMax + g] = {nq, roff, eoff, ent};
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        cta_ng[b] = ng;
        if (bad_s) atomicOr(&flag[0], bad_s);
    }
}

// stage sizes in global group order (for the offset scan)
__global__ void k_pan_sizes(const int32_t *blk, const PanPlan *plan, int ncta, uint64_t *sizes) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= ncta) return;
    for (int g = 0; g < blk[b + 1] - blk[b]; ++g) sizes[blk[b] + g] = (uint64_t)plan[(int64_t)b * kPanGMax + g].bytes;
}

// Per CTA: writes the group descriptors, headers, padding and then scatters every segment
// (row id and entries) into its slot of the count-sorted order.
__global__ void __launch_bounds__(kPanTPB) k_pan_fill(const int64_t *slice_ptr, const uint32_t *col,
                                                      int64_t n, int64_t ncols, int S, int rpc,
                                                      const int32_t *blk,
                                                      const PanPlan *plan, const PanPlanQ *planq,
                                                      const uint64_t *offs, PanGroup *grp,
                                                      uint8_t *stream) {
    extern __shared__ uint32_t psm[];
    uint32_t *map = psm;               // S: panel -> group
    uint32_t *nxt = psm + S;           // kPanGMax x kPanCMax: next slot of each count bucket
    const int b = blockIdx.x;
    const int64_t r0 = (int64_t)b * rpc;
    const int rows = (int)((n - r0) < rpc ? (n - r0) : rpc);
    const int gb = blk[b], ng = blk[b + 1] - gb;
    for (int i = threadIdx.x; i < S; i += kPanTPB) map[i] = 0xffffffffu;
    for (int i = threadIdx.x; i < kPanGMax * kPanCMax; i += kPanTPB) nxt[i] = 0;
    __syncthreads();
    for (int g = 0; g < ng; ++g) {
        const PanPlan pl = plan[(int64_t)b * kPanGMax + g];
        for (int s = pl.lo + (int)threadIdx.x; s < pl.hi; s += kPanTPB) map[s] = g;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < rows; i += kPanTPB) {  // segment histogram again
        int cur = -1, cnt = 0;
        pan_row_walk(slice_ptr, col, r0 + i, [&](uint32_t c) {
            const int g = (int)map[c / kPanZ];
            if (g != cur) {
                if (cnt) atomicAdd(&nxt[cur * kPanCMax + cnt], 1u);
                cur = g;
                cnt = 0;
            }
            ++cnt;
        });
        if (cnt) atomicAdd(&nxt[cur * kPanCMax + cnt], 1u);
    }
    __syncthreads();
    // descriptors, bucket starts and iteration headers: one thread per group
    for (int g = threadIdx.x; g < ng; g += kPanTPB) {
        const PanPlan pl = plan[(int64_t)b * kPanGMax + g];
        const PanPlanQ pq = planq[(int64_t)b * kPanGMax + g];
        const uint64_t off = offs[gb + g];
        grp[gb + g] = {pl.dense ? pl.lo : -1, pq.nq, pq.roff, pq.eoff, off, (uint32_t)pl.bytes, 0u};
        uint32_t *hdr = (uint32_t *)(stream + off);
        uint32_t pos = 0, base = 0;
        for (int c = kPanCMax - 1; c >= 1; --c) {
            const uint32_t h = nxt[g * kPanCMax + c];
            nxt[g * kPanCMax + c] = pos;
            if (!h) continue;
            for (uint32_t q = (pos + 31) / 32; q < (pos + h + 31) / 32; ++q) {
                hdr[q] = base | ((uint32_t)c << 24);
                base += 32 * (uint32_t)c;
            }
            pos += h;
        }
    }
    // padding: dummy rows, zero-slot / sentinel entries
    for (int g = 0; g < ng; ++g) {
        const PanPlan pl = plan[(int64_t)b * kPanGMax + g];
        const PanPlanQ pq = planq[(int64_t)b * kPanGMax + g];
        uint8_t *st = stream + offs[gb + g];
        uint16_t *rw = (uint16_t *)(st + pq.roff);
        for (uint32_t i = threadIdx.x; i < 32 * pq.nq; i += kPanTPB) rw[i] = (uint16_t)kPanR;
        if (pl.dense) {
            uint16_t *e = (uint16_t *)(st + pq.eoff);
            for (uint32_t i = threadIdx.x; i < pq.ent; i += kPanTPB) e[i] = (uint16_t)kPanZ;
        } else {
            uint32_t *e = (uint32_t *)(st + pq.eoff);
            for (uint32_t i = threadIdx.x; i < pq.ent; i += kPanTPB) e[i] = (uint32_t)ncols;  // z[ncols] = 0
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < rows; i += kPanTPB) {
        int cur = -1, cnt = 0;
        // a segment is flushed when the row leaves its group: its count is known then, and its
        // entries are re-read from the SELL layout into their diagonal-major positions
        auto flush = [&](int g, int count, int first_t) {
            const PanPlan pl = plan[(int64_t)b * kPanGMax + g];
            const PanPlanQ pq = planq[(int64_t)b * kPanGMax + g];
            uint8_t *st = stream + offs[gb + g];
            const uint32_t slot = atomicAdd(&nxt[g * kPanCMax + count], 1u);
            const uint32_t q = slot >> 5, l = slot & 31;
            ((uint16_t *)(st + pq.roff))[slot] = (uint16_t)i;
            const uint32_t base = ((const uint32_t *)st)[q] & 0xffffffu;
            const int64_t r = r0 + i;
            const int64_t sl = r >> 5;
            const int lane = (int)(r & 31);
            const int64_t sb = slice_ptr[sl];
            for (int k = 0; k < count; ++k) {
                const uint32_t c = __ldg(col + sb + 32 * (int64_t)(first_t + k) + lane);
                if (pl.dense)
                    ((uint16_t *)(st + pq.eoff))[base + 32 * k + l] = (uint16_t)(c - (uint32_t)pl.lo * kPanZ);
                else
                    ((uint32_t *)(st + pq.eoff))[base + 32 * k + l] = c;
            }
        };
        int t = 0, first = 0;
        pan_row_walk(slice_ptr, col, r0 + i, [&](uint32_t c) {
            const int g = (int)map[c / kPanZ];
            if (g != cur) {
                if (cnt) flush(cur, cnt, first);
                cur = g;
                cnt = 0;
                first = t;
            }
            ++cnt;
            ++t;
        });
        if (cnt) flush(cur, cnt, first);
    }
}

// Bank-aware lane assignment: the 32 segments of an iteration may sit in any lanes (a segment
// moves with its entries, so every row keeps its order).  part[row] is a double, so rows r
// and r' collide in a half-warp access when r == r' (mod 16); this places the segments so
// that each half-warp sees each residue at most about half as often (one match_any + two
// ballots per iteration), cutting the replayed wavefronts of the part[] loads and stores.
__global__ void __launch_bounds__(256) k_pan_balance(const PanGroup *__restrict__ grp,
                                                     uint8_t *__restrict__ stream) {
    const PanGroup m = grp[blockIdx.x];
    uint8_t *st = stream + m.off;
    const uint32_t *hdr = (const uint32_t *)st;
    uint16_t *rows = (uint16_t *)(st + m.roff);
    const int lane = threadIdx.x & 31;
    for (uint32_t q = threadIdx.x >> 5; q < m.nq; q += blockDim.x >> 5) {
        const uint32_t h = hdr[q];
        const int c = (int)(h >> 24);
        const uint32_t base = h & 0xffffffu;
        const uint16_t row = rows[q * 32 + lane];
        const bool dummy = row >= kPanR;
        // the k-th segment (in lane order) of each residue goes to half k & 1; dummy rows share
        // one address and are spread the same way; overflow of a half spills into the other
        const int bank = dummy ? 16 : (row & 15);
        const uint32_t lt = (1u << lane) - 1u;
        const unsigned same = __match_any_sync(0xffffffffu, bank);
        const int half = __popc(same & lt) & 1;
        const unsigned inA = __ballot_sync(0xffffffffu, half == 0);
        const int nA = __popc(inA);
        const int pos = __popc((half == 0 ? inA : ~inA) & lt);
        int mine;
        if (half == 0) mine = pos < 16 ? pos : 16 + (32 - nA) + (pos - 16);
        else mine = pos < 16 ? 16 + pos : nA + (pos - 16);
        __syncwarp();
        rows[q * 32 + mine] = row;
        if (m.panel >= 0) {
            uint16_t *e = (uint16_t *)(st + m.eoff) + base;
            for (int k = 0; k < c; ++k) {
                const uint16_t v = e[32 * k + lane];
                __syncwarp();
                e[32 * k + mine] = v;
                __syncwarp();
            }
        } else {
            uint32_t *e = (uint32_t *)(st + m.eoff) + base;
            for (int k = 0; k < c; ++k) {
                const uint32_t v = e[32 * k + lane];
                __syncwarp();
                e[32 * k + mine] = v;
                __syncwarp();
            }
        }
    }
}

static int32_t build_panels_rpc(sc_graph *g, bool prof, int rpc, int32_t *declined);

// Builds g's panel layout from its SELL arrays.  Returns SC_OK with g->pan_ctas == 0 when the
// graph does not qualify (weighted, wide rows, too many panels/groups, long segments, rows
// that revisit a panel, too little dense coverage or too short dense segments); a stage
// larger than the ring slot is retried with half the rows per CTA.  CUDA errors are returned.
static int32_t build_panels(sc_graph *g, bool prof) {
    g->pan_ctas = 0;
    const int64_t n = g->n;
    if (!g->unit || g->n_wide || n < kPanR) return SC_OK;
    if ((g->ncols + kPanZ - 1) / kPanZ > kPanSMax) return SC_OK;
    for (int rpc = kPanR; rpc >= 256; rpc = (rpc / 2) & ~31) {
        int32_t declined = 0;
        const int32_t st = build_panels_rpc(g, prof, rpc, &declined);
        if (st || g->pan_ctas) return st;
        if (declined != 4) break;  // only oversized stages improve with fewer rows
    }
    return SC_OK;
}

static int32_t build_panels_rpc(sc_graph *g, bool prof, int rpc, int32_t *declined) {
    const int64_t n = g->n;
    const int S = (int)((g->ncols + kPanZ - 1) / kPanZ);
    cudaStream_t s = g->stream;
    const int ncta = (int)((n + rpc - 1) / rpc);
    const uint32_t slot_cap = (uint32_t)(((kPanSmemMax - kPanFixedSmem) / kPanNS) & ~127);
    int32_t *cta_ng = nullptr, *flag = nullptr, *blk = nullptr;
    PanPlan *plan = nullptr;
    PanPlanQ *planq = nullptr;
    uint64_t *sizes = nullptr, *offs = nullptr;
    void *tmp = nullptr;
    auto cleanup = [&]() {
        for (void *p_ : {(void *)cta_ng, (void *)flag, (void *)plan, (void *)planq, (void *)sizes,
                         (void *)offs, tmp})
            if (p_) cudaFreeAsync(p_, s);
    };
    cudaError_t e = cudaSuccess;
    const size_t smem_plan = ((size_t)S + kPanGMax * kPanCMax) * 4;
    e = cudaFuncSetAttribute(k_pan_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_plan);
    if (!e) e = cudaFuncSetAttribute(k_pan_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_plan);
    if (!e) e = cudaMallocAsync((void **)&cta_ng, (size_t)(ncta + 1) * 4, s);
    if (!e) e = cudaMallocAsync((void **)&flag, 64, s);
    if (!e) e = cudaMallocAsync((void **)&plan, (size_t)ncta * kPanGMax * sizeof(PanPlan), s);
    if (!e) e = cudaMallocAsync((void **)&planq, (size_t)ncta * kPanGMax * sizeof(PanPlanQ), s);
    if (!e) e = cudaMemsetAsync(flag, 0, 64, s);
    if (!e) e = cudaMemsetAsync(cta_ng + ncta, 0, 4, s);
    if (!e) {
        k_pan_plan<<<ncta, kPanTPB, smem_plan, s>>>(g->d_slice_ptr, g->d_col, n, S, rpc, slot_cap, cta_ng,
                                                    plan, planq, flag, (unsigned long long *)(flag + 8));
        e = cudaGetLastError();
    }
    int32_t hflag[16] = {0};
    if (!e) e = cudaMemcpyAsync(hflag, flag, 64, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) {
        cleanup();
        return fail(SC_E_CUDA, "panel plan: %s", cudaGetErrorString(e));
    }
    // the layout pays off only when most entries fall into dense panels (graphs whose ids
    // carry no locality stay on SELL) and dense segments are long enough to amortise the
    // partial-sum round trip through shared memory (config 5: 1.3 entries -> SELL is faster)
    unsigned long long cover[3];
    memcpy(cover, hflag + 8, 24);
    if (!hflag[0] && cover[0] < kPanMinCover * cover[1]) hflag[0] = 16;
    if (!hflag[0] && cover[0] < kPanMinSegment * cover[2]) hflag[0] = 32;
    if (hflag[0]) {
        *declined = hflag[0];
        if (prof)
            fprintf(stderr, "[sc_graph_create] panel layout declined at %d rows/CTA (flags %d)\n", rpc,
                    hflag[0]);
        cleanup();
        return SC_OK;
    }
    int32_t st;
    if ((st = dmalloc(g, (void **)&g->d_pan_blk, (size_t)(ncta + 1) * 4))) {
        cleanup();
        return st;
    }
    size_t tb = 0, tb2 = 0;
    e = cub::DeviceScan::ExclusiveSum(nullptr, tb, cta_ng, g->d_pan_blk, ncta + 1, s);
    int32_t ngroups = 0;
    if (!e) e = cudaMallocAsync(&tmp, tb + 16, s);
    if (!e) e = cub::DeviceScan::ExclusiveSum(tmp, tb, cta_ng, g->d_pan_blk, ncta + 1, s);
    if (!e) e = cudaMemcpyAsync(&ngroups, g->d_pan_blk + ncta, 4, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (!e) e = cudaMallocAsync((void **)&sizes, (size_t)(ngroups + 1) * 8, s);
    if (!e) e = cudaMallocAsync((void **)&offs, (size_t)(ngroups + 1) * 8, s);
    if (!e) e = cudaMemsetAsync(sizes + ngroups, 0, 8, s);
    if (!e) {
        k_pan_sizes<<<(ncta + 255) / 256, 256, 0, s>>>(g->d_pan_blk, plan, ncta, sizes);
        e = cudaGetLastError();
    }
    if (!e) e = cub::DeviceScan::ExclusiveSum(nullptr, tb2, sizes, offs, ngroups + 1, s);
    if (!e && tb2 > tb) {
        cudaFreeAsync(tmp, s);
        e = cudaMallocAsync(&tmp, tb2 + 16, s);
    }
    if (!e) e = cub::DeviceScan::ExclusiveSum(tmp, tb2, sizes, offs, ngroups + 1, s);
    uint64_t total = 0;
    if (!e) e = cudaMemcpyAsync(&total, offs + ngroups, 8, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) {
        cleanup();
        return fail(SC_E_CUDA, "panel offsets: %s", cudaGetErrorString(e));
    }
    if ((st = dmalloc(g, (void **)&g->d_pan_grp, (size_t)std::max(ngroups, 1) * sizeof(PanGroup))) ||
        (st = dmalloc(g, (void **)&g->d_pan_stream, (size_t)total + 64))) {
        cleanup();
        return st;
    }
    k_pan_fill<<<ncta, kPanTPB, smem_plan, s>>>(g->d_slice_ptr, g->d_col, n, g->ncols, S, rpc, g->d_pan_blk, plan, planq,
                                                offs, g->d_pan_grp, g->d_pan_stream);
    e = cudaGetLastError();
    if (!e && ngroups) {
        k_pan_balance<<<ngroups, 256, 0, s>>>(g->d_pan_grp, g->d_pan_stream);
        e = cudaGetLastError();
    }
    if (!e) e = cudaStreamSynchronize(s);
    cleanup();
    if (e) return fail(SC_E_CUDA, "panel fill: %s", cudaGetErrorString(e));
    g->pan_slot = (hflag[1] + 127) & ~127;
    // the attribute is per function, shared by all handles: allow the largest ring any handle
    // can have (a handle's launch asks for its own, smaller or equal, amount)
    const int smem = kPanFixedSmem + kPanNS * (int)slot_cap;
    SC_CUDA(cudaFuncSetAttribute(k_rw_panel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    SC_CUDA(cudaFuncSetAttribute(k_rw_panel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    g->pan_ctas = ncta;
    g->pan_rpc = rpc;
    g->pan_groups = ngroups;
    g->pan_bytes = (int64_t)total;
    if (prof)
        fprintf(stderr, "[sc_graph_create] panels: %d CTAs x %d rows, %d groups, %.1f MB stream, slot %d\n",
                ncta, rpc, ngroups, total / 1e6, g->pan_slot);
    return SC_OK;
}

static cudaError_t launch_panel_step(const sc_graph *g, const StepArgs &a, bool sym, cudaStream_t s) {
    PanArgs p;
    p.blk = g->d_pan_blk;
    p.grp = g->d_pan_grp;
    p.stream = g->d_pan_stream;
    p.n = g->n;
    p.ncols = g->ncols;
    p.slot = g->pan_slot;
    p.rpc = g->pan_rpc;
    const int smem = kPanFixedSmem + kPanNS * g->pan_slot;
    if (sym) k_rw_panel<true><<<g->pan_ctas, kPanTPB, smem, s>>>(a, p);
    else k_rw_panel<false><<<g->pan_ctas, kPanTPB, smem, s>>>(a, p);
    return cudaGetLastError();
}
