// sc_window.cuh -- row-window layout and SpMV step for graphs whose renumbered rows reference
// mostly their own neighbourhood (k-NN / geometric / mesh graphs after the BFS pre-order;
// included by sc_graph.cu after sc_panel.cuh, inside namespace sc).
//
// Why: after the BFS pre-order ~80 % of a 4096-row region's entries point into the region
// itself (config 4: 0.796, tools/window_probe.py).  The SELL kernel still gathers every one of
// them through the L1/L2 request path and streams a 4-byte column per entry.  Here a CTA owns
// a run of slices inside one 4096-row panel and stages, once,
//   * the panel's 4096 z values by one bulk copy (TMA, 32 KB), and
//   * the z values of its "far" entries (columns outside the panel), gathered from L2 by all
//     threads at full memory-level parallelism -- outside every row's dependent add chain,
// into shared memory; every stored entry then is a 16-bit shared-memory index (2 bytes streamed
// instead of 4) and the in-order row sums read shared memory only.
//
// Exactness: the SELL slices, their stored order and the per-lane left-to-right __dadd_rn chain
// are unchanged (same products, same order as k_rw_step); padding entries read a zero slot with
// weight 0 and add +0.0, an exact no-op (a sum that starts at +0.0 is never -0.0).  Only where
// a z value is read from changes.
//
// Layout (built on the device from the SELL arrays):
//   Entries are stored in PAIRS so one 32-bit load brings two indices and one 128-bit load two
//   weights (the kernel is bound by instruction issue, not bytes: ~25 instructions per
//   entry-step with scalar loads, profiles/r02_spmv_c4_win_ncu_full.txt).  Slice sl holds
//   ceil(width / 2) pair-steps; pair p of lane l sits at ptr[sl] + 32 p + l.
//   widx[]    2 x u16 per pair: panel-local index (< 4096), 4096 = zero slot (padding),
//             4097 + s = far slot s of the item
//   wval[]    the pair's two weights (double2; float2 for the fp32-value variant; none for unit)
//   far[]     u32 z-space column of every far entry, item after item, in (slice, position) order
//   items[]   slice range [slice_lo, slice_hi) inside one panel, far list range; a panel's 128
//             slices are cut greedily so an item has <= kWinSlicesMax slices and <= kWinFarMax
//             far entries (a single slice always fits: 32 rows x 256 entries)

constexpr int kWinZ = 4096;          // panel width = the SELL sorting window
constexpr int kWinFarMax = 8192;     // far slots per item (64 KB)
constexpr int kWinTPB = 512;         // 2 CTAs/SM: 64 registers per thread
constexpr int kWinSlicesMax = 4 * (kWinTPB / 32);  // slices per item: four per warp
constexpr int kWinFar0 = kWinZ + 1;  // first far slot; kWinZ is the zero slot
constexpr double kWinMinCover = 0.6; // fraction of entries inside the own panel the layout needs
static_assert(kWinZ == kSigma, "panels are the SELL sorting windows");

static_assert(kWinFar0 + kWinFarMax <= 65536, "16-bit indices");
static_assert(kWinSlicesMax / (kWinTPB / 32) <= 32, "a lane per slice of the warp");

struct WinItem {
    int32_t slice_lo, slice_hi;
    int64_t far_base;
    int32_t nfar, unused;
};

struct WinArgs {
    const WinItem *items;
    const int64_t *ptr;     // nslices + 1: first pair of each slice (multiples of 32)
    const uint32_t *idx;    // index pairs
    const double2 *val;     // weight pairs (fp64) or null
    const float2 *val32;    // weight pairs (fp32 variant) or null
    const uint32_t *far;
    int64_t ncols;
};

#ifndef SC_WIN_UNROLL
#define SC_WIN_UNROLL 2
#endif
constexpr int kWinUnroll = SC_WIN_UNROLL;  // pair-steps per batch; two batches in flight per lane
constexpr int kWinFarPT = (kWinFarMax + kWinTPB - 1) / kWinTPB;  // far slots per thread
constexpr uint32_t kWinPadPair = (uint32_t)kWinZ | ((uint32_t)kWinZ << 16);

// one slice (32 rows, a lane each) folded in stored order from the staged window wz
template <bool UNIT, bool SYM, bool F32>
__device__ __forceinline__ void win_fold_slice(const StepArgs &a, const WinArgs &w,
                                               const double *wz, int sl, int lane) {
    const int64_t r = (int64_t)sl * kSlice + lane;
    const bool live = r < a.n_sell;
    double xr = 0.0, sc = 1.0;
    if (live) {
        xr = __ldcs(a.x_in + r);
        sc = __ldcs(a.scale + r);
    }
    const int64_t base = w.ptr[sl];
    const int np = (int)((w.ptr[sl + 1] - base) >> 5);
    const uint32_t *ip = w.idx + base + lane;
    const double2 *vp = (UNIT || F32) ? nullptr : w.val + base + lane;
    const float2 *vp32 = F32 ? w.val32 + base + lane : nullptr;
    // three register sets rotate by name: while one batch of kWinUnroll pair-steps is
    // gathered from shared memory and added in order, the next two batches' index and
    // weight pairs are in flight from global memory.  (Tried: one stream per warp across
    // its slices with two cursors -- 505 us vs 481 us at config 4, and any spilled load
    // target serialises the prefetch: 607 us.)
    auto load = [&](int p0, uint32_t (&ci)[kWinUnroll], double2 (&wv)[kWinUnroll]) {
#pragma unroll
        for (int q = 0; q < kWinUnroll; ++q) {
            const int p = p0 + q;
            const bool in = p < np;
            ci[q] = in ? __ldcs(ip + (int64_t)p * kSlice) : kWinPadPair;
            if (!UNIT) {
                wv[q] = make_double2(0.0, 0.0);
                if (in) {
                    if (F32) {
                        const float2 f = __ldcs(vp32 + (int64_t)p * kSlice);
                        wv[q] = make_double2((double)f.x, (double)f.y);
                    } else {
                        wv[q] = __ldcs(vp + (int64_t)p * kSlice);
                    }
                }
            }
        }
    };
    double s = 0.0;
    auto fold = [&](const uint32_t (&ci)[kWinUnroll], const double2 (&wv)[kWinUnroll]) {
        double z0[kWinUnroll], z1[kWinUnroll];
#pragma unroll
        for (int q = 0; q < kWinUnroll; ++q) {
            z0[q] = wz[ci[q] & 0xffffu];
            z1[q] = wz[ci[q] >> 16];
        }
#pragma unroll
        for (int q = 0; q < kWinUnroll; ++q) {
            s = __dadd_rn(s, UNIT ? z0[q] : __dmul_rn(wv[q].x, z0[q]));
            s = __dadd_rn(s, UNIT ? z1[q] : __dmul_rn(wv[q].y, z1[q]));
        }
    };
    uint32_t cA[kWinUnroll], cB[kWinUnroll], cC[kWinUnroll];
    double2 wA[kWinUnroll], wB[kWinUnroll], wC[kWinUnroll];
    load(0, cA, wA);
    load(kWinUnroll, cB, wB);
    for (int p0 = 0; p0 < np;) {
        load(p0 + 2 * kWinUnroll, cC, wC);
        fold(cA, wA);
        if ((p0 += kWinUnroll) >= np) break;
        load(p0 + 2 * kWinUnroll, cA, wA);
        fold(cB, wB);
        if ((p0 += kWinUnroll) >= np) break;
        load(p0 + 2 * kWinUnroll, cB, wB);
        fold(cC, wC);
        p0 += kWinUnroll;
    }
    if (live) row_epilogue<SYM>(a, r, s, xr, sc);
}

template <bool UNIT, bool SYM, bool F32>
__global__ void __launch_bounds__(kWinTPB, 2) k_rw_win(StepArgs a, WinArgs w) {
    extern __shared__ __align__(128) double wz[];  // panel (kWinZ) | zero slot | far slots
    __shared__ uint64_t zfull;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const WinItem it = w.items[blockIdx.x];
    const int64_t zb = a.col_offset + ((int64_t)it.slice_lo * kSlice / kWinZ) * kWinZ;
    if (threadIdx.x == 0) {
        pan_mbar_init(&zfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const int64_t left = w.ncols - zb;
        const uint32_t bytes = (uint32_t)(((left < kWinZ ? left : kWinZ) * 8 + 15) & ~15);
        pan_bulk(wz, a.z_in + zb, bytes, &zfull);
        wz[kWinZ] = 0.0;
    }
    // far z values: every thread loads its (<= kWinFarPT) far columns, then issues all its
    // gathers, then stores them -- two memory latencies per item, nothing on a row's add chain
    {
        double *fz = wz + kWinFar0;
        const uint32_t *fl = w.far + it.far_base;
        uint32_t c[kWinFarPT];
        double v[kWinFarPT];
#pragma unroll
        for (int u = 0; u < kWinFarPT; ++u) {
            const int i = u * kWinTPB + (int)threadIdx.x;
            c[u] = i < it.nfar ? __ldcs(fl + i) : kPad;
        }
#pragma unroll
        for (int u = 0; u < kWinFarPT; ++u) v[u] = c[u] != kPad ? __ldg(a.z_in + c[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < kWinFarPT; ++u) {
            const int i = u * kWinTPB + (int)threadIdx.x;
            if (i < it.nfar) fz[i] = v[u];
        }
    }
    __syncthreads();
    pan_mbar_wait(&zfull, 0);
    // slices are dealt round-robin to the warps (an item's slices are consecutive in the
    // length-sorted window, so every warp gets a similar mix)
    for (int sl = it.slice_lo + warp; sl < it.slice_hi; sl += kWinTPB / 32)
        win_fold_slice<UNIT, SYM, F32>(a, w, wz, sl, lane);
    peer_fence(a);
}

// ---- layout construction (device) ----

// per slice: far entries (stored, not padding, outside the slice's own panel); totals[0] +=
// entries inside the own panel, totals[1] += stored entries (padding excluded), totals[2] =
// max far entries of one slice (an item holds at least one slice, so it must fit the far slots)
__global__ void k_win_count(const int64_t *__restrict__ slice_ptr, const uint32_t *__restrict__ col,
                            int64_t nslices, int64_t col_offset, int32_t *__restrict__ far_cnt,
                            unsigned long long *__restrict__ totals) {
    const int lane = threadIdx.x & 31;
    const int64_t sl = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (sl >= nslices) return;
    const int64_t base = slice_ptr[sl];
    const int width = (int)((slice_ptr[sl + 1] - base) >> 5);
    const int64_t zb = col_offset + (sl * kSlice / kWinZ) * kWinZ;
    int nfar = 0, nin = 0;
    for (int t = 0; t < width; ++t) {
        const uint32_t c = __ldg(col + base + (int64_t)t * kSlice + lane);
        if (c == kPad) continue;
        const int64_t off = (int64_t)c - zb;
        if (off >= 0 && off < kWinZ) ++nin;
        else ++nfar;
    }
    for (int o = 16; o; o >>= 1) {
        nfar += __shfl_xor_sync(0xffffffffu, nfar, o);
        nin += __shfl_xor_sync(0xffffffffu, nin, o);
    }
    if (lane == 0) {
        far_cnt[sl] = nfar;
        atomicAdd(&totals[0], (unsigned long long)nin);
        atomicAdd(&totals[1], (unsigned long long)(nin + nfar));
        atomicMax(&totals[2], (unsigned long long)nfar);
    }
}

// one thread per panel: cuts the panel's slices into items.  Pass 1 (items == null) counts;
// pass 2 writes the items at item_off[panel] and each slice's first far slot inside its item.
__global__ void k_win_items(const int32_t *__restrict__ far_cnt, const int64_t *__restrict__ far_off,
                            int64_t nslices, int64_t npanels, int32_t *__restrict__ item_cnt,
                            const int32_t *__restrict__ item_off, WinItem *__restrict__ items,
                            int32_t *__restrict__ slot_base) {
    const int64_t pnl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (pnl >= npanels) return;
    constexpr int spp = kWinZ / kSlice;
    const int64_t s0 = pnl * spp, s1 = s0 + spp < nslices ? s0 + spp : nslices;
    int count = 0;
    int64_t lo = s0;
    int far = 0;
    for (int64_t sl = s0; sl < s1; ++sl) {
        const int f = far_cnt[sl];
        if (sl > lo && (far + f > kWinFarMax || sl - lo >= kWinSlicesMax)) {
            if (items) items[item_off[pnl] + count] = {(int32_t)lo, (int32_t)sl, far_off[lo], far, 0};
            ++count;
            lo = sl;
            far = 0;
        }
        if (items) slot_base[sl] = far;
        far += f;
    }
    if (s1 > lo) {
        if (items) items[item_off[pnl] + count] = {(int32_t)lo, (int32_t)s1, far_off[lo], far, 0};
        ++count;
    }
    if (!items) item_cnt[pnl] = count;
}

// pair-steps (x 32 lanes) of every slice, for the scan that gives WinArgs::ptr
__global__ void k_win_pairs(const int64_t *__restrict__ slice_ptr, int64_t nslices,
                            int64_t *__restrict__ npairs) {
    const int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (sl > nslices) return;
    if (sl == nslices) {
        npairs[sl] = 0;
        return;
    }
    const int64_t width = (slice_ptr[sl + 1] - slice_ptr[sl]) >> 5;
    npairs[sl] = ((width + 1) >> 1) * kSlice;
}

// warp per slice: the index pairs, weight pairs and the far column list.  Far slots are handed
// out in (slice, stored position, lane) order.
__global__ void k_win_fill(const int64_t *__restrict__ slice_ptr, const uint32_t *__restrict__ col,
                           const double *__restrict__ val, const float *__restrict__ val32,
                           int64_t nslices, int64_t col_offset, const int64_t *__restrict__ far_off,
                           const int32_t *__restrict__ slot_base, const int64_t *__restrict__ wptr,
                           uint32_t *__restrict__ widx, double2 *__restrict__ wval,
                           float2 *__restrict__ wval32, uint32_t *__restrict__ far) {
    const int lane = threadIdx.x & 31;
    const int64_t sl = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (sl >= nslices) return;
    const int64_t base = slice_ptr[sl];
    const int width = (int)((slice_ptr[sl + 1] - base) >> 5);
    const int64_t zb = col_offset + (sl * kSlice / kWinZ) * kWinZ;
    const int64_t fo = far_off[sl];
    const int sb = slot_base[sl];
    const int64_t pb = wptr[sl];
    int run = 0;
    for (int t0 = 0; t0 < width; t0 += 2) {
        uint32_t pair = 0;
        double wd[2] = {0.0, 0.0};
        float wf[2] = {0.f, 0.f};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int t = t0 + h;
            const int64_t j = base + (int64_t)t * kSlice + lane;
            const uint32_t c = t < width ? __ldg(col + j) : kPad;
            const int64_t off = (int64_t)c - zb;
            const bool pad = c == kPad, in = !pad && off >= 0 && off < kWinZ, isfar = !pad && !in;
            const uint32_t m = __ballot_sync(0xffffffffu, isfar);
            const int rank = run + __popc(m & ((1u << lane) - 1u));
            uint32_t v = (uint32_t)kWinZ;
            if (in) v = (uint32_t)off;
            if (isfar) {
                v = (uint32_t)(kWinFar0 + sb + rank);
                far[fo + rank] = c;
            }
            pair |= v << (16 * h);
            if (!pad && val) wd[h] = val[j];
            if (!pad && val32) wf[h] = val32[j];
            run += __popc(m);
        }
        const int64_t dst = pb + (int64_t)(t0 >> 1) * kSlice + lane;
        widx[dst] = pair;
        if (wval) wval[dst] = make_double2(wd[0], wd[1]);
        if (wval32) wval32[dst] = make_float2(wf[0], wf[1]);
    }
}

template <typename K>
static cudaError_t win_set_smem(K kern, int smem) {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

// Builds g's row-window layout from its SELL arrays.  Returns SC_OK with g->win_items == 0 when
// the graph does not qualify (fewer than kWinMinCover of the stored entries inside the rows' own
// panels, one slice with more far entries than an item's slots, a z space that is not 16-byte
// aligned at panel starts, more than 2^26 slices or 2^32 stored entries).
static int32_t build_windows(sc_graph *g, bool prof) {
    g->win_items = 0;
    if (!g->nslices || g->nslices >= (int64_t(1) << 26) || (g->col_offset & 1)) return SC_OK;
    if (g->sell_entries >= (int64_t(1) << 32)) return SC_OK;  // 32-bit pair offsets
    cudaStream_t s = g->stream;
    const int64_t ns = g->nslices;
    const int64_t npanels = (ns * kSlice + kWinZ - 1) / kWinZ;
    int32_t *far_cnt = nullptr, *item_cnt = nullptr, *item_off = nullptr, *slot_base = nullptr;
    int64_t *far_off = nullptr;
    unsigned long long *totals = nullptr;
    void *tmp = nullptr;
    auto cleanup = [&]() {
        for (void *p_ : {(void *)far_cnt, (void *)item_cnt, (void *)item_off, (void *)slot_base,
                         (void *)far_off, (void *)totals, tmp})
            if (p_) cudaFreeAsync(p_, s);
    };
    cudaError_t e = cudaMallocAsync((void **)&far_cnt, (size_t)(ns + 1) * 4, s);
    if (!e) e = cudaMallocAsync((void **)&far_off, (size_t)(ns + 1) * 8, s);
    if (!e) e = cudaMallocAsync((void **)&totals, 24, s);
    if (!e) e = cudaMemsetAsync(totals, 0, 24, s);
    if (!e) e = cudaMemsetAsync(far_cnt + ns, 0, 4, s);
    const unsigned wgrid = (unsigned)((ns * 32 + 255) / 256);
    if (!e) {
        k_win_count<<<wgrid, 256, 0, s>>>(g->d_slice_ptr, g->d_col, ns, g->col_offset, far_cnt, totals);
        e = cudaGetLastError();
    }
    unsigned long long htot[3] = {0, 0, 0};
    if (!e) e = cudaMemcpyAsync(htot, totals, 24, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) {
        cleanup();
        return fail(SC_E_CUDA, "window count: %s", cudaGetErrorString(e));
    }
    if (htot[1] == 0 || (double)htot[0] < kWinMinCover * (double)htot[1] || htot[2] > (unsigned long long)kWinFarMax) {
        if (prof)
            fprintf(stderr, "[sc_graph_create] window layout declined: %.3f of the entries in own panels\n",
                    htot[1] ? (double)htot[0] / (double)htot[1] : 0.0);
        cleanup();
        return SC_OK;
    }
    size_t tb = 0, tb2 = 0;
    e = cub::DeviceScan::ExclusiveSum(nullptr, tb, far_cnt, far_off, ns + 1, s);
    if (!e) e = cub::DeviceScan::ExclusiveSum(nullptr, tb2, item_cnt, item_off, npanels + 1, s);
    if (!e) e = cudaMallocAsync(&tmp, std::max(tb, tb2) + 16, s);
    if (!e) e = cub::DeviceScan::ExclusiveSum(tmp, tb, far_cnt, far_off, ns + 1, s);
    if (!e) e = cudaMallocAsync((void **)&item_cnt, (size_t)(npanels + 1) * 4, s);
    if (!e) e = cudaMallocAsync((void **)&item_off, (size_t)(npanels + 1) * 4, s);
    if (!e) e = cudaMallocAsync((void **)&slot_base, (size_t)ns * 4, s);
    if (!e) e = cudaMemsetAsync(item_cnt + npanels, 0, 4, s);
    const unsigned pgrid = (unsigned)((npanels + 127) / 128);
    if (!e) {
        k_win_items<<<pgrid, 128, 0, s>>>(far_cnt, far_off, ns, npanels, item_cnt, nullptr, nullptr, nullptr);
        e = cudaGetLastError();
    }
    if (!e) e = cub::DeviceScan::ExclusiveSum(tmp, tb2, item_cnt, item_off, npanels + 1, s);
    int32_t nitems = 0;
    int64_t nfar = 0;
    if (!e) e = cudaMemcpyAsync(&nitems, item_off + npanels, 4, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaMemcpyAsync(&nfar, far_off + ns, 8, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) {
        cleanup();
        return fail(SC_E_CUDA, "window items: %s", cudaGetErrorString(e));
    }
    // pair offsets of the slices
    int32_t st;
    int64_t npair = 0;
    int64_t *npairs = nullptr;
    if ((st = dmalloc(g, (void **)&g->d_win_ptr, (size_t)(ns + 1) * 8))) {
        cleanup();
        return st;
    }
    e = cudaMallocAsync((void **)&npairs, (size_t)(ns + 1) * 8, s);
    if (!e) {
        k_win_pairs<<<(unsigned)((ns + 256) / 256), 256, 0, s>>>(g->d_slice_ptr, ns, npairs);
        e = cudaGetLastError();
    }
    size_t tb3 = 0;
    if (!e) e = cub::DeviceScan::ExclusiveSum(nullptr, tb3, npairs, g->d_win_ptr, ns + 1, s);
    if (!e && tb3 > std::max(tb, tb2)) {
        cudaFreeAsync(tmp, s);
        e = cudaMallocAsync(&tmp, tb3 + 16, s);
    }
    if (!e) e = cub::DeviceScan::ExclusiveSum(tmp, tb3, npairs, g->d_win_ptr, ns + 1, s);
    if (!e) e = cudaMemcpyAsync(&npair, g->d_win_ptr + ns, 8, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (npairs) cudaFreeAsync(npairs, s);
    if (e) {
        cleanup();
        return fail(SC_E_CUDA, "window pair offsets: %s", cudaGetErrorString(e));
    }
    const bool w64 = !g->unit && !g->f32, w32 = !g->unit && g->f32;
    if ((st = dmalloc(g, (void **)&g->d_win_items, (size_t)std::max(nitems, 1) * sizeof(WinItem))) ||
        (st = dmalloc(g, (void **)&g->d_win_idx, (size_t)npair * 4 + 16)) ||
        (w64 && (st = dmalloc(g, (void **)&g->d_win_val, (size_t)npair * 16 + 16))) ||
        (w32 && (st = dmalloc(g, (void **)&g->d_win_val32, (size_t)npair * 8 + 16))) ||
        (st = dmalloc(g, (void **)&g->d_win_far, (size_t)nfar * 4 + 16))) {
        cleanup();
        return st;
    }
    k_win_items<<<pgrid, 128, 0, s>>>(far_cnt, far_off, ns, npanels, item_cnt, item_off, g->d_win_items,
                                      slot_base);
    e = cudaGetLastError();
    if (!e) {
        k_win_fill<<<wgrid, 256, 0, s>>>(g->d_slice_ptr, g->d_col, w64 ? g->d_val : nullptr,
                                         w32 ? g->d_val32 : nullptr, ns, g->col_offset, far_off,
                                         slot_base, g->d_win_ptr, g->d_win_idx, g->d_win_val,
                                         g->d_win_val32, g->d_win_far);
        e = cudaGetLastError();
    }
    if (!e) e = cudaStreamSynchronize(s);
    cleanup();
    if (e) return fail(SC_E_CUDA, "window fill: %s", cudaGetErrorString(e));
    // the attribute is per function and shared by all handles: allow the largest item
    const int smem = (kWinFar0 + kWinFarMax) * 8;
    e = win_set_smem(k_rw_win<true, false, false>, smem);
    if (!e) e = win_set_smem(k_rw_win<true, true, false>, smem);
    if (!e) e = win_set_smem(k_rw_win<false, false, false>, smem);
    if (!e) e = win_set_smem(k_rw_win<false, true, false>, smem);
    if (!e) e = win_set_smem(k_rw_win<false, false, true>, smem);
    if (!e) e = win_set_smem(k_rw_win<false, true, true>, smem);
    if (e) return fail(SC_E_CUDA, "window kernel attributes: %s", cudaGetErrorString(e));
    g->win_items = nitems;
    g->win_far = nfar;
    g->win_pairs = npair;
    g->win_cover = (double)htot[0] / (double)htot[1];
    if (prof)
        fprintf(stderr, "[sc_graph_create] windows: %d items, %.3f of the entries in own panels, %lld far\n",
                nitems, g->win_cover, (long long)nfar);
    return SC_OK;
}

// the SELL rows of a whole-handle step through the window layout (wide rows stay with
// k_rw_wide, launched by the caller)
static cudaError_t launch_window_step(const sc_graph *g, const StepArgs &a, bool sym, cudaStream_t s) {
    WinArgs w;
    w.items = g->d_win_items;
    w.ptr = g->d_win_ptr;
    w.idx = g->d_win_idx;
    w.val = g->d_win_val;
    w.val32 = g->d_win_val32;
    w.far = g->d_win_far;
    w.ncols = g->ncols;
    const int smem = (kWinFar0 + kWinFarMax) * 8;
    const dim3 grid((unsigned)g->win_items);
    if (g->unit) {
        if (sym) k_rw_win<true, true, false><<<grid, kWinTPB, smem, s>>>(a, w);
        else k_rw_win<true, false, false><<<grid, kWinTPB, smem, s>>>(a, w);
    } else if (g->f32) {
        if (sym) k_rw_win<false, true, true><<<grid, kWinTPB, smem, s>>>(a, w);
        else k_rw_win<false, false, true><<<grid, kWinTPB, smem, s>>>(a, w);
    } else {
        if (sym) k_rw_win<false, true, false><<<grid, kWinTPB, smem, s>>>(a, w);
        else k_rw_win<false, false, false><<<grid, kWinTPB, smem, s>>>(a, w);
    }
    return cudaGetLastError();
}
