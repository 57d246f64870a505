// sc_multi.cuh -- one graph handle over several GPUs in ONE process (SURVEY.md §8(b)'s
// `n_gpus` argument; the drop-in entry point fast_spectral_cluster(g, params) stays one call,
// ref: pipeline.py:127).  Included at the end of sc_graph.cu (uses its internals).
//
// Layout.  Rows are cut into W contiguous blocks balanced by stored entries (shard w owns
// global rows [row0_w, row0_w + n_w)).  Every shard keeps its own SELL renumbering
// (sell_order of its row offsets -- exactly what graph_init computes for a shard), and all
// shards share one z space in which shard w's renumbered rows live at [zoff_w, zoff_w + n_w),
// zoff_w aligned to 8192 slots so the column-panel layout's 4096-row renumbering windows
// never straddle a panel.  zidx[v] = zoff_w + iperm_w[v - row0_w] renames every global
// column once, on the host, before the shards are uploaded.
//
// Exchange.  Every device holds the whole z space (2 buffers).  A step's epilogue stores each
// z value it produces into its own buffer AND at the same offset of every peer's buffer
// (StepArgs.peer_base: coalesced 256-byte warp stores over NVLink, overlapped with the
// gathers of the same kernel -- the compute+collective fusion), then the shard records an
// event; step t+1 of every shard waits for the step-t events of all shards
// (cudaStreamWaitEvent across devices: kernel completion makes its peer stores visible, no
// spin barrier, so W shards may also share one GPU -- which is how the one-GPU tests run it).
// Hazard: shard w's step t writes buffer (t+1)&1 of every peer, which the peers last read in
// step t-1; step t of w starts after all step-(t-1) events, so those reads are done.
//
// Exactness.  Rows are never split and keep their stored column order; only where z values
// live changes, so x_T and f are bit-identical to the one-GPU handle (and the reference).
// The k-means replica then runs on the first device, on f gathered into vertex order there.
#pragma once

namespace sc {

struct MultiShard {
    sc_graph *g = nullptr;
    int device = 0;
    int64_t row0 = 0, n = 0, zoff = 0;
    cudaEvent_t ev[2] = {nullptr, nullptr};
};

struct Multi {
    std::vector<MultiShard> sh;
    int64_t ncols = 0;
    int32_t *d_zidx = nullptr;  // device of shard 0: global vertex -> z-space slot
    double *d_f = nullptr;      // device of shard 0: f in vertex order (k-means input)
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    int result = -1;
    bool have_x0 = false;
};

constexpr int64_t kMultiAlign = 8192;

static void multi_free(sc_graph *mg) {
    Multi *m = mg->multi;
    if (!m) return;
    for (auto &s : m->sh) {
        if (s.g) {
            cudaSetDevice(s.device);
            cudaStreamSynchronize(s.g->stream);
            for (auto &e : s.ev)
                if (e) cudaEventDestroy(e);
            sc_graph_destroy(s.g);
        }
    }
    if (!m->sh.empty()) cudaSetDevice(m->sh[0].device);
    if (m->d_zidx) cudaFree(m->d_zidx);
    if (m->d_f) cudaFree(m->d_f);
    if (m->t0) cudaEventDestroy(m->t0);
    if (m->t1) cudaEventDestroy(m->t1);
    delete m;
    mg->multi = nullptr;
}

// row blocks balanced by stored entries: shard w starts at the first row whose offset reaches
// w * nnz / W (every shard keeps >= 1 row)
static std::vector<int64_t> multi_partition(const int64_t *rp, int64_t n, int W) {
    const int64_t nnz = rp[n];
    std::vector<int64_t> b((size_t)W + 1);
    b[0] = 0;
    b[W] = n;
    for (int w = 1; w < W; ++w) {
        const int64_t target = (int64_t)((__int128)nnz * w / W);
        int64_t r = std::lower_bound(rp, rp + n + 1, target) - rp;
        r = std::max<int64_t>(r, b[w - 1] + 1);
        r = std::min<int64_t>(r, n - (W - w));
        b[w] = r;
    }
    return b;
}

static int32_t multi_create(const int64_t *rp, const int32_t *col, const double *val,
                            const double *deg, int64_t n, int64_t nnz, int W,
                            const int32_t *devices, uint32_t cflags, sc_graph **out) {
    SC_REQUIRE(out, SC_E_INVALID, "out is null");
    *out = nullptr;
    SC_REQUIRE(rp && deg && (col || nnz == 0), SC_E_INVALID, "null CSR array");
    SC_REQUIRE(W >= 1 && W <= kMaxWorld, SC_E_INVALID, "n_gpus=%d outside [1, %d]", W, kMaxWorld);
    SC_REQUIRE(n >= W && n < (int64_t(1) << 31) - 1, SC_E_INVALID,
               "n=%lld out of range for %d shards", (long long)n, W);
    SC_REQUIRE(rp[0] == 0 && rp[n] == nnz, SC_E_RANGE,
               "row_ptr[0] must be 0 and row_ptr[n] must equal nnz=%lld", (long long)nnz);
    SC_REQUIRE(!(cflags & SC_CREATE_REORDER_BFS), SC_E_INVALID,
               "the BFS pre-order applies to single-GPU handles");
    SC_REQUIRE(!(cflags & (SC_CREATE_KEEP_WEIGHTS | SC_CREATE_FP32_VALUES)) || val, SC_E_INVALID,
               "weight flags need a weight array");
    int ndev = 0;
    SC_CUDA(cudaGetDeviceCount(&ndev));
    std::vector<int> dev((size_t)W);
    for (int w = 0; w < W; ++w) {
        dev[w] = devices ? devices[w] : w;
        SC_REQUIRE(dev[w] >= 0 && dev[w] < ndev, SC_E_INVALID,
                   "device %d of shard %d: %d CUDA device(s) visible", dev[w], w, ndev);
    }
    // peer access between every pair of distinct devices (NVLink / NVSwitch on B200 nodes)
    for (int a = 0; a < W; ++a)
        for (int b = 0; b < W; ++b) {
            if (dev[a] == dev[b]) continue;
            int can = 0;
            SC_CUDA(cudaDeviceCanAccessPeer(&can, dev[a], dev[b]));
            SC_REQUIRE(can, SC_E_INVALID, "GPU %d cannot access GPU %d's memory (no P2P path)",
                       dev[a], dev[b]);
            SC_CUDA(cudaSetDevice(dev[a]));
            cudaError_t e = cudaDeviceEnablePeerAccess(dev[b], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else SC_CUDA(e);
        }

    auto *mg = new sc_graph();
    mg->multi = new Multi();
    Multi *m = mg->multi;
    auto fail_out = [&](int32_t st) {
        multi_free(mg);
        delete mg;
        return st;
    };
    const std::vector<int64_t> b = multi_partition(rp, n, W);
    m->sh.resize((size_t)W);
    // per-shard renumbering (identical to the one graph_init computes for the shard)
    std::vector<std::vector<int32_t>> perm((size_t)W);
    int64_t zo = 0;
    for (int w = 0; w < W; ++w) {
        MultiShard &s = m->sh[w];
        s.device = dev[w];
        s.row0 = b[w];
        s.n = b[w + 1] - b[w];
        s.zoff = zo;
        zo = (zo + s.n + kMultiAlign - 1) / kMultiAlign * kMultiAlign;
        std::vector<int64_t> lrp((size_t)s.n + 1);
        for (int64_t i = 0; i <= s.n; ++i) lrp[i] = rp[s.row0 + i] - rp[s.row0];
        sell_order(lrp.data(), s.n, perm[w]);
    }
    m->ncols = m->sh[W - 1].zoff + m->sh[W - 1].n;
    SC_REQUIRE(m->ncols < (int64_t(1) << 32) - 64, SC_E_INVALID, "z space too large");
    std::vector<int32_t> zidx((size_t)n);
    for (int w = 0; w < W; ++w) {
        const MultiShard &s = m->sh[w];
        for (int64_t p = 0; p < s.n; ++p) zidx[s.row0 + perm[w][p]] = (int32_t)(s.zoff + p);
    }
    // every shard's columns renamed into the z space (host threads), range-checked here
    std::vector<int32_t> rcol((size_t)nnz);
    {
        const int nt = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        std::vector<int64_t> badpos((size_t)nt, -1);
        const int64_t chunk = (nnz + nt - 1) / nt;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                const int64_t lo = t * chunk, hi = std::min(nnz, lo + chunk);
                for (int64_t i = lo; i < hi; ++i) {
                    const int32_t c = col[i];
                    if ((uint32_t)c >= (uint64_t)n) {
                        badpos[t] = i;
                        return;
                    }
                    rcol[i] = zidx[c];
                }
            });
        for (auto &x : th) x.join();
        for (int t = 0; t < nt; ++t)
            if (badpos[t] >= 0)
                return fail_out(fail(SC_E_RANGE, "column index %d at entry %lld outside [0, %lld)",
                                     col[badpos[t]], (long long)badpos[t], (long long)n));
    }
    int32_t st;
    for (int w = 0; w < W; ++w) {
        MultiShard &s = m->sh[w];
        std::vector<int64_t> lrp((size_t)s.n + 1);
        const int64_t e0 = rp[s.row0];
        for (int64_t i = 0; i <= s.n; ++i) lrp[i] = rp[s.row0 + i] - e0;
        st = graph_init(lrp.data(), rcol.data() + e0, val ? val + e0 : nullptr, deg + s.row0, s.n,
                        lrp[s.n], m->ncols, s.zoff, s.row0, 0,
                        cflags & (SC_CREATE_KEEP_WEIGHTS | SC_CREATE_FP32_VALUES), s.device, &s.g);
        if (st) return fail_out(st);
        SC_REQUIRE(s.g->n_sell + s.g->n_wide == s.n, SC_E_INTERNAL, "shard layout mismatch");
        s.g->peer_events = true;
        if ((cflags & SC_CREATE_PANELS) && (st = build_panels(s.g, false))) return fail_out(st);
        if ((cflags & SC_CREATE_WINDOWS) && !s.g->pan_ctas && (st = build_windows(s.g, false)))
            return fail_out(st);
        SC_CUDA(cudaSetDevice(s.device));
        for (auto &e : s.ev) SC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    // peers: every shard's epilogue mirrors its z values into all other shards' z buffers
    if (W > 1) {
        std::vector<void *> zb((size_t)W), fb((size_t)W);
        for (int w = 0; w < W; ++w) {
            double *z;
            uint32_t *f;
            if ((st = sc_shard_buffers(m->sh[w].g, &z, &f))) return fail_out(st);
            zb[w] = z;
            fb[w] = f;
        }
        for (int w = 0; w < W; ++w)
            if ((st = sc_shard_set_peers(m->sh[w].g, zb.data(), fb.data(), W, w))) return fail_out(st);
    }
    const MultiShard &s0 = m->sh[0];
    SC_CUDA(cudaSetDevice(s0.device));
    SC_CUDA(cudaEventCreate(&m->t0));
    SC_CUDA(cudaEventCreate(&m->t1));
    SC_CUDA(cudaMalloc((void **)&m->d_zidx, (size_t)n * 4));
    SC_CUDA(cudaMalloc((void **)&m->d_f, (size_t)n * 8));
    SC_CUDA(cudaMemcpy(m->d_zidx, zidx.data(), (size_t)n * 4, cudaMemcpyHostToDevice));
    mg->device = s0.device;
    mg->sm_count = s0.g->sm_count;
    mg->n = n;
    mg->nnz = nnz;
    mg->ncols = n;
    mg->unit = s0.g->unit;
    *out = mg;
    return SC_OK;
}

// x0 per shard (Irwin-Hall on global ids, or the caller's), x0_out / x0_in in vertex order
static int32_t multi_sample(sc_graph *mg, uint64_t key0, uint64_t key1, double *x0_out) {
    Multi *m = mg->multi;
    for (auto &s : m->sh) {
        int32_t st = sc_sample_irwin_hall(s.g, key0, key1, x0_out ? x0_out + s.row0 : nullptr);
        if (st) return st;
    }
    m->have_x0 = true;
    m->result = -1;
    return SC_OK;
}

static int32_t multi_set_x0(sc_graph *mg, const double *x0) {
    Multi *m = mg->multi;
    for (auto &s : m->sh) {
        int32_t st = sc_set_x0(s.g, x0 + s.row0);
        if (st) return st;
    }
    m->have_x0 = true;
    m->result = -1;
    return SC_OK;
}

// every shard waits for the events of parity `par` of all OTHER shards (same-stream order
// covers its own)
static int32_t multi_wait_all(Multi *m, int w, int par) {
    for (int v = 0; v < (int)m->sh.size(); ++v)
        if (v != w) SC_CUDA(cudaStreamWaitEvent(m->sh[w].g->stream, m->sh[v].ev[par], 0));
    return SC_OK;
}

static int32_t multi_power(sc_graph *mg, int32_t T, double sign, uint32_t flags, double *xT_out,
                           double *f_out, sc_timing *t_out) {
    Multi *m = mg->multi;
    SC_REQUIRE(m->have_x0, SC_E_STATE, "no start vector: call sc_sample_irwin_hall or sc_set_x0");
    const int W = (int)m->sh.size();
    const bool sym = flags & SC_SYM_VARIANT;
    const uint32_t sflags = flags & (SC_SYM_VARIANT | SC_FORCE_WEIGHTED | SC_FORCE_SELL);
    int32_t st;
    // the clock starts on shard 0's stream; every other stream joins behind it
    MultiShard &s0 = m->sh[0];
    SC_CUDA(cudaSetDevice(s0.device));
    SC_CUDA(cudaEventRecord(m->t0, s0.g->stream));
    SC_CUDA(cudaEventRecord(s0.ev[1], s0.g->stream));
    for (int w = 1; w < W; ++w) {
        SC_CUDA(cudaSetDevice(m->sh[w].device));
        SC_CUDA(cudaStreamWaitEvent(m->sh[w].g->stream, s0.ev[1], 0));
    }
    // z_0 = x0 / d (mirrored into every peer), then T steps
    for (int w = 0; w < W; ++w) {
        MultiShard &s = m->sh[w];
        SC_CUDA(cudaSetDevice(s.device));
        if (sym && (st = ensure_isd(s.g, s.g->stream))) return st;
        if ((st = sc_shard_scale(s.g, s.g->d_x0, s.g->d_z[0], sflags & SC_SYM_VARIANT, s.g->stream)))
            return st;
        SC_CUDA(cudaEventRecord(s.ev[1], s.g->stream));
    }
    for (int32_t t = 0; t < T; ++t) {
        const int in = t & 1, out = in ^ 1;
        for (int w = 0; w < W; ++w) {
            MultiShard &s = m->sh[w];
            SC_CUDA(cudaSetDevice(s.device));
            if ((st = multi_wait_all(m, w, out))) return st;  // previous phase's parity
            if ((st = launch_step(s.g, s.g->d_z[in], t == 0 ? s.g->d_x0 : s.g->d_x[in],
                                  s.g->d_x[out], s.g->d_z[out], sign, sflags, s.g->stream)))
                return st;
            SC_CUDA(cudaEventRecord(s.ev[in], s.g->stream));
        }
    }
    // join: shard 0 waits for the last phase of every shard, then stops the clock
    const int last = T == 0 ? 1 : ((T - 1) & 1);
    SC_CUDA(cudaSetDevice(s0.device));
    if ((st = multi_wait_all(m, 0, last))) return st;
    SC_CUDA(cudaEventRecord(m->t1, s0.g->stream));
    SC_CUDA(cudaEventSynchronize(m->t1));
    float ms = 0.f;
    SC_CUDA(cudaEventElapsedTime(&ms, m->t0, m->t1));
    m->result = T & 1;
    auto h0 = std::chrono::steady_clock::now();
    for (auto &s : m->sh) {
        SC_CUDA(cudaSetDevice(s.device));
        s.g->result = m->result;
        const double *xT = T == 0 ? s.g->d_x0 : s.g->d_x[m->result];
        if (xT_out && (st = to_host_original(s.g, xT, xT_out + s.row0))) return st;
        if (f_out && (st = to_host_original(s.g, s.g->d_z[m->result] + s.zoff, f_out + s.row0)))
            return st;
    }
    auto h1 = std::chrono::steady_clock::now();
    if (t_out) {
        t_out->power_ms = ms;
        t_out->kernel_ms = T ? ms / T : 0.0;
        t_out->d2h_ms = std::chrono::duration<double, std::milli>(h1 - h0).count();
    }
    return SC_OK;
}

static int32_t multi_download_f(sc_graph *mg, double *f_out) {
    Multi *m = mg->multi;
    SC_REQUIRE(m->result >= 0, SC_E_STATE, "no power iteration has run on this handle");
    for (auto &s : m->sh) {
        SC_CUDA(cudaSetDevice(s.device));
        int32_t st = to_host_original(s.g, s.g->d_z[m->result] + s.zoff, f_out + s.row0);
        if (st) return st;
    }
    return SC_OK;
}

// f in vertex order on the first device: every device holds the whole z space after the
// last step, so one gather through zidx assembles it there
static const double *multi_f_device(sc_graph *mg) {
    Multi *m = mg->multi;
    if (m->result < 0) return nullptr;
    const MultiShard &s0 = m->sh[0];
    if (cudaSetDevice(s0.device) != cudaSuccess) return nullptr;
    if (sc_gather_f64(s0.g->d_z[m->result], m->d_zidx, mg->n, m->d_f, s0.g->stream)) return nullptr;
    if (cudaStreamSynchronize(s0.g->stream) != cudaSuccess) return nullptr;
    return m->d_f;
}

static int32_t multi_info(const sc_graph *mg, sc_graph_info *o) {
    const Multi *m = mg->multi;
    std::memset(o, 0, sizeof *o);
    o->n = mg->n;
    o->nnz = mg->nnz;
    o->ncols = m->ncols;
    o->unit_weights = mg->unit;
    o->device = mg->device;
    o->sm_count = mg->sm_count;
    o->n_gpus = (int32_t)m->sh.size();
    o->window_items = 0;
    for (const MultiShard &s : m->sh) o->window_items += s.g->win_items;
    for (const auto &s : m->sh) {
        o->ntiles += s.g->nslices;
        o->long_rows += s.g->n_wide;
        o->device_bytes += s.g->bytes;
        o->stored_entries += s.g->sell_entries;
        o->panel_groups += s.g->pan_ctas ? s.g->pan_groups : 0;
        o->panel_bytes += s.g->pan_ctas ? s.g->pan_bytes : 0;
    }
    o->device_bytes += mg->n * 12;
    o->zstride = m->sh[0].g->zstride;
    return SC_OK;
}

}  // namespace sc

extern "C" int32_t sc_graph_create_multi(const int64_t *row_ptr, const int32_t *col,
                                         const double *val, const double *deg, int64_t n,
                                         int64_t nnz, int32_t n_gpus, const int32_t *devices,
                                         uint32_t create_flags, sc_graph **out) {
    return sc::multi_create(row_ptr, col, val, deg, n, nnz, n_gpus, devices, create_flags, out);
}

extern "C" int32_t sc_graph_shard_layout(const sc_graph *g, int32_t shard, int64_t *row0,
                                         int64_t *rows, int64_t *zoff, int32_t *device) {
    SC_REQUIRE(g && g->multi, SC_E_INVALID, "not a multi-GPU handle");
    SC_REQUIRE(shard >= 0 && shard < (int32_t)g->multi->sh.size(), SC_E_INVALID, "bad shard %d",
               shard);
    const sc::MultiShard &s = g->multi->sh[shard];
    if (row0) *row0 = s.row0;
    if (rows) *rows = s.n;
    if (zoff) *zoff = s.zoff;
    if (device) *device = s.device;
    return SC_OK;
}
