/*
 * sc_b200.h -- C-ABI of the B200-native one-vector clustering path.
 *
 * Plain pointers and sizes only (no torch / CUDA types), callable from ctypes, cgo, JNI
 * or C++.  Every entry point returns an int status: 0 = ok, -1..-99 = input error
 * (maps to specluster.errors.InputError, CLI exit 2), <= -100 = CUDA / internal error
 * (maps to SpeclusterError, CLI exit 1); see specluster/errors.py:8-29 and
 * specluster/cli.py:411-427.  The message of the last failure on the calling thread
 * is returned by sc_last_error().
 *
 * Which reference interface each entry point replaces (paths relative to
 * /root/reference/pkg/src/specluster):
 *
 *   sc_graph_create        Graph CSR arrays (graph.py:28-45) + SignlessLaplacianOp
 *                          .__init__ (spectral.py:46-50: caches the adjacency and
 *                          deg^{-1/2}); uploads once, builds the nnz-balanced tiling.
 *   sc_sample_irwin_hall   the start vector x0(u) ~ IW(deg u) of the one-vector method
 *                          (PAPER.md:20); stands where sample_gaussian_vectors
 *                          (spectral.py:183-195) stands for Algorithm 2.
 *   sc_set_x0              an x0 supplied by the caller (the reference's own vector).
 *   sc_power_iterate       power_method(op, x0, t) (spectral.py:87-102) with op the lazy
 *                          random walk x -> 0.5 x +/- 0.5 A D^-1 x (or, with
 *                          SC_SYM_VARIANT, SignlessLaplacianOp.matvec spectral.py:52-57),
 *                          followed by the degree normalisation (pipeline.py:157 analogue:
 *                          f = D^-1 x_T for rw, f = D^-1/2 x_T for sym).
 *   sc_kmeans_*            lloyd (kmeans.py:167-215) on the 1-D embedding, bit-exact
 *                          replica of its k-means++ seeding (kmeans.py:116-137) and Lloyd
 *                          iterations; the host replays the PCG64 draws
 *                          (rng_for(seed, r), spectral.py:32-36).
 *   sc_shard_*             row-block shard of the CSR for 1/2/4/8-GPU runs (no reference
 *                          counterpart).
 */
#ifndef SC_B200_H
#define SC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define SC_OK 0
#define SC_E_INVALID (-1)      /* bad argument (null pointer, size, dtype contract) */
#define SC_E_RANGE (-2)        /* index out of range / inconsistent CSR */
#define SC_E_STATE (-3)        /* call order violated (e.g. power_iterate before x0) */
#define SC_E_CUDA (-100)       /* CUDA runtime error */
#define SC_E_OOM (-101)        /* device allocation failed */
#define SC_E_INTERNAL (-102)

/* sc_power_iterate flags */
#define SC_SYM_VARIANT 0x1u    /* signless symmetric operator (reference Algorithm-2 op) */
#define SC_NO_CUDA_GRAPH 0x2u  /* launch T kernels instead of replaying a captured graph */
#define SC_L2_PERSIST 0x4u     /* pin the gathered z vector in L2 (access-policy window) */
#define SC_FORCE_WEIGHTED 0x8u /* use the weighted kernel even if all weights are 1.0 */
#define SC_FORCE_SELL 0x10u    /* use the SELL kernel even if the handle has a panel layout */

typedef struct sc_graph sc_graph;
typedef struct sc_kmeans sc_kmeans;

typedef struct sc_graph_info {
    int64_t n;            /* local rows */
    int64_t nnz;          /* local stored entries */
    int64_t ncols;        /* length of the gathered z space */
    int64_t col_offset;   /* where local row i's z lives in z space */
    int64_t ntiles;       /* SELL-32 slices (32 renumbered rows each) */
    int64_t long_rows;    /* wide rows (> 256 entries), one warp each */
    int32_t unit_weights; /* 1 if the val array was elided */
    int32_t rp64;         /* 1 if row offsets are kept as int64 on device */
    int64_t device_bytes; /* device memory owned by the handle */
    int32_t device;
    int32_t sm_count;
    int64_t stored_entries; /* SELL-32 entries incl. padding (+ wide-row entries excluded) */
    int64_t panel_groups;   /* column-panel layout: stages (0 = no panel layout) */
    int64_t panel_bytes;    /* column-panel layout: bytes streamed per step */
    int64_t zstride;        /* doubles between the handle's two z buffers (sc_shard_buffers) */
    int32_t n_gpus;         /* shards of a multi-GPU handle (sc_graph_create_multi), else 1 */
    int32_t window_items;   /* row-window layout: CTA work items per step (0 = no window layout) */
} sc_graph_info;

typedef struct sc_timing {
    double sample_ms;     /* Irwin-Hall / x0 upload + z0 */
    double power_ms;      /* T iterations, CUDA events on the handle's stream */
    double kernel_ms;     /* power_ms / T */
    double d2h_ms;
} sc_timing;

int32_t sc_version(void);
const char *sc_last_error(void);
int32_t sc_device_count(void);

/* ---- graph handle ------------------------------------------------------- */
/* row_ptr int64[n+1] (host), col int32[nnz] (host), val double[nnz] or NULL (unit),
 * deg double[n] (host, copied verbatim -- never recomputed).  The handle owns the
 * device copies and one CUDA stream on `device`. */
int32_t sc_graph_create(const int64_t *row_ptr, const int32_t *col, const double *val,
                        const double *deg, int64_t n, int64_t nnz, int32_t device,
                        sc_graph **out);
/* As sc_graph_create; create_flags: SC_CREATE_KEEP_WEIGHTS keeps an all-ones weight array on
 * the device (the weighted kernel then streams it) instead of eliding it. */
#define SC_CREATE_KEEP_WEIGHTS 0x1u
/* store the weights as fp32 (8 -> 4 bytes per entry; products still formed in fp64): the
 * optional fp32-value variant, agreeing with fp64 within 1e-5 relative (not bit-exact) */
#define SC_CREATE_FP32_VALUES 0x2u
/* locality pre-order: vertices renumbered by a multi-source BFS (regions of ~4096 vertices
 * around every 4096th vertex, by level) before the SELL layout, for graphs whose ids carry no
 * locality; exact (only where z values live changes), whole graphs only */
#define SC_CREATE_REORDER_BFS 0x4u
/* column-panel layout in addition to SELL (unit weights, no rows > 256 entries, whole graphs):
 * each 3392-row block's heavily referenced 8192-column ranges are staged in shared memory
 * and gathered there, the rest from L2; bit-identical results.  Declined silently when the
 * graph does not qualify (sc_graph_info.panel_groups == 0). */
#define SC_CREATE_PANELS 0x8u
/* row-window layout in addition to SELL (any weights; whole-handle steps): for graphs whose
 * renumbered rows reference mostly their own 4096-row neighbourhood (k-NN / geometric graphs,
 * typically after SC_CREATE_REORDER_BFS) each CTA stages its panel's 4096 z values (one bulk
 * copy) and the z values of its out-of-panel entries (gathered once, off the rows' add chains)
 * in shared memory and streams 16-bit shared-memory indices instead of 32-bit columns;
 * bit-identical results.  Declined silently when fewer than 60 % of the stored entries fall
 * into the rows' own panels (sc_graph_info.window_items == 0) or when the handle already has
 * a column-panel layout. */
#define SC_CREATE_WINDOWS 0x10u
int32_t sc_graph_create_ex(const int64_t *row_ptr, const int32_t *col, const double *val,
                           const double *deg, int64_t n, int64_t nnz, int32_t device,
                           uint32_t create_flags, sc_graph **out);
/* Row-block shard: rows are the local block, columns index a z space of length ncols in
 * which this shard's own rows live at [col_offset, col_offset + n).  Columns must already
 * be renamed into the renumbered z space (every shard's sc_sell_order permutation). */
int32_t sc_shard_create(const int64_t *row_ptr, const int32_t *col, const double *val,
                        const double *deg, int64_t n, int64_t nnz, int64_t ncols,
                        int64_t col_offset, int64_t global_row0, int32_t device,
                        sc_graph **out);
/* Multi-GPU handle in ONE process (SURVEY.md §8(b)'s n_gpus; replaces the single-GPU graph
 * behind fast_spectral_cluster, ref: pipeline.py:127 -- the call stays one call).  Rows are
 * cut into n_gpus blocks balanced by stored entries, one shard per entry of `devices`
 * (nullable = 0..n_gpus-1; a device may repeat: several shards share it).  Every device holds
 * the whole gathered vector; each step's epilogue stores its z values into all peers' copies
 * over peer memory (NVLink P2P) and the shards' streams are ordered by events.  The handle
 * works with sc_sample_irwin_hall, sc_set_x0, sc_power_iterate, sc_graph_download_f,
 * sc_graph_info_get and sc_kmeans_create_from_graph (f gathered to the first device); x_T
 * and f are bit-identical to the single-GPU handle's.  create_flags: SC_CREATE_PANELS,
 * SC_CREATE_WINDOWS, SC_CREATE_KEEP_WEIGHTS, SC_CREATE_FP32_VALUES (no BFS pre-order). */
int32_t sc_graph_create_multi(const int64_t *row_ptr, const int32_t *col, const double *val,
                              const double *deg, int64_t n, int64_t nnz, int32_t n_gpus,
                              const int32_t *devices, uint32_t create_flags, sc_graph **out);
/* where shard `shard` of a multi-GPU handle lives: its global rows [row0, row0 + rows), its
 * z-space block [zoff, zoff + rows) and its device (all outputs nullable) */
int32_t sc_graph_shard_layout(const sc_graph *g, int32_t shard, int64_t *row0, int64_t *rows,
                              int64_t *zoff, int32_t *device);
void sc_graph_destroy(sc_graph *g);
/* Destroyed handles return their device buffers to a process-wide cache (reused by the next
 * handle; capped by SC_BUFFER_CACHE_MB, default 16384).  This frees the cached buffers of
 * `device` (all devices if < 0) and returns the bytes released. */
int64_t sc_release_cached_memory(int32_t device);
int32_t sc_graph_info_get(const sc_graph *g, sc_graph_info *out);
/* Builds the column-panel layout (SC_CREATE_PANELS) on an existing handle -- whole graphs or
 * shards; declined silently when the graph does not qualify (panel_groups stays 0).  Steps
 * over a shard's full row range then use it: the caller's z buffers must be 16-byte aligned
 * and hold ncols + 16 doubles with z[ncols..] == 0 (the padding target; the handle's own
 * buffers already do). */
int32_t sc_graph_build_panels(sc_graph *g);
/* Builds the row-window layout (SC_CREATE_WINDOWS) on an existing single-GPU handle or shard;
 * declined silently when the graph does not qualify (window_items stays 0).  Whole-handle
 * steps then use it when the z buffer is 16-byte aligned and holds z[ncols] == 0. */
int32_t sc_graph_build_windows(sc_graph *g);
/* The device layout renumbers rows (SELL-32-sigma: length-sorted inside 4096-row windows,
 * rows longer than 256 last).  sc_sell_order returns that permutation for a row_ptr
 * (perm[p] = original row of renumbered row p) so a multi-GPU driver can rename columns
 * across shards; sc_graph_order returns a handle's permutation.  Host-facing vectors
 * (x0, x_T, f) are always in ORIGINAL order; shard device buffers are renumbered. */
int32_t sc_sell_order(const int64_t *row_ptr, int64_t n, int32_t *perm_out);
int32_t sc_graph_order(const sc_graph *g, int32_t *perm_out);

/* ---- start vector ------------------------------------------------------- */
/* x0(u) = sum of floor(deg u) uniforms (+ frac(deg u) * one more), uniform j of global
 * vertex u = word j%4 of Philox4x64-10(key, counter (j/4+1, u, 0, 0)) as
 * (raw >> 11) * 2^-53.  x0_out (host, nullable) receives the local x0. */
int32_t sc_sample_irwin_hall(sc_graph *g, uint64_t key0, uint64_t key1, double *x0_out);
int32_t sc_set_x0(sc_graph *g, const double *x0_host);

/* ---- power iteration ---------------------------------------------------- */
/* T steps of x <- 0.5 x + sign*0.5 A D^-1 x (sign = +1 or -1) from the current x0;
 * xT_out / f_out are host buffers (nullable).  After the call f stays resident on the
 * device for sc_kmeans_create_from_graph. */
int32_t sc_power_iterate(sc_graph *g, int32_t T, double sign, uint32_t flags, double *xT_out,
                         double *f_out, sc_timing *t_out);
/* f of the last sc_power_iterate (original order) into a host buffer: lets a caller fetch the
 * embedding while a k-means context built from the handle runs on another thread. */
int32_t sc_graph_download_f(sc_graph *g, double *f_out);

/* Block power method for the reference's pm_log_k mode (pipeline.py:144-147): T steps of
 * the signless operator M = (I + D^-1/2 A D^-1/2) / 2 on an (n, L) block x0 (host,
 * row-major, original vertex order, 1 <= L <= 16), every column bit-identical to
 * power_method(SignlessLaplacianOp(g), x0, T) (spectral.py:87-102).  raw_out = M^T x0,
 * scaled_out = raw * d^-1/2 per row (pipeline.py:157); both host (n, L), nullable. */
int32_t sc_power_iterate_block(sc_graph *g, int32_t T, int32_t L, const double *x0,
                               double *raw_out, double *scaled_out, sc_timing *t_out);

/* ---- device-pointer shard step (multi-GPU composition) ------------------ */
/* One iteration on a shard using caller-owned device buffers, launched on `stream` (a
 * cudaStream_t; 0 = the legacy default stream), all buffers in renumbered order:
 * reads z_in[ncols] (gathered), x_in[n]; writes x_out[n], z_out[col_offset + i]. */
int32_t sc_shard_step(sc_graph *g, const double *z_in, const double *x_in, double *x_out,
                      double *z_out, double sign, uint32_t flags, void *stream);
/* Only renumbered rows [row_lo, row_hi) (slice aligned: multiples of 32 below the wide
 * rows): the pieces of a pipelined multi-GPU step, each followed by its own all-gather. */
int32_t sc_shard_step_range(sc_graph *g, int64_t row_lo, int64_t row_hi, const double *z_in,
                            const double *x_in, double *x_out, double *z_out, double sign,
                            uint32_t flags, void *stream);
/* z_out[col_offset + i] = x[i] / deg[i] (or * deg^-1/2 with SC_SYM_VARIANT) */
int32_t sc_shard_scale_range(sc_graph *g, int64_t row_lo, int64_t row_hi, const double *x,
                             double *z_out, uint32_t flags, void *stream);
int32_t sc_shard_scale(sc_graph *g, const double *x, double *z_out, uint32_t flags,
                       void *stream);
/* ---- fused z exchange over peer memory (NVLink P2P), instead of an all-gather ------- */
/* sc_shard_buffers: the handle's own z allocation (z0 then z1 = z0 + zstride, zeroed; zstride
 * from sc_graph_info, >= ncols + 1 so z[ncols] stays a zero slot) and
 * its 64-word flag array.  Ranks export both with sc_ipc_export, import the peers' with
 * sc_ipc_import, and hand all world bases to sc_shard_set_peers (entries for `rank` ignored).
 * From then on every z value a step / scale writes into the handle's z allocation is also
 * stored at the same offset of every peer's allocation from the SpMV epilogue itself, and
 * sc_shard_barrier (one tiny kernel per step: release/acquire flags at system scope) replaces
 * the collective.  Results stay bit-identical: rows and their summation order are untouched. */
int32_t sc_shard_buffers(sc_graph *g, double **z_base, uint32_t **flags);
int32_t sc_shard_set_peers(sc_graph *g, void *const *z_bases, void *const *flag_bases,
                           int32_t world, int32_t rank);
int32_t sc_shard_barrier(sc_graph *g, void *stream);
int32_t sc_ipc_export(const void *dptr, void *handle_out /* 64 bytes */);
int32_t sc_ipc_import(const void *handle /* 64 bytes */, int32_t device, void **dptr_out);
int32_t sc_ipc_release(void *dptr);
/* ---- halo exchange (only the z entries a peer references) -------------------------- */
/* dst[i] = src[idx[i]] for i < count (device pointers, on `stream`): packs the own z
 * entries a peer's rows reference into a contiguous send buffer.  Paired with a shard whose
 * columns are renamed into [own rows | halo entries grouped by owner], the exchange moves
 * only those entries (ncclSend/ncclRecv) instead of all-gathering z; bit-exact, since no row
 * or summation order changes. */
int32_t sc_gather_f64(const double *src, const int32_t *idx, int64_t count, double *dst,
                      void *stream);
/* x0 for the shard rows (global ids global_row0..), device output */
int32_t sc_shard_irwin_hall(sc_graph *g, uint64_t key0, uint64_t key1, double *x_out,
                            void *stream);

/* ---- device graph generator (configs too large for the host) ------------ */
/* Planted-partition graph with the reference SBM's law (generate.py:112-149): k blocks of
 * n/k consecutive vertices, pairs u < v independent with prob p (same block) / q, isolated
 * vertices dropped and ids compacted.  Realised on the device with geometric skips over each
 * row's upper candidates; skip j of row u is word j%4 of Philox4x64-10(key, (j/4+1, u,
 * 0x5bd1e995, 0)), U = ((raw >> 11) + 1) 2^-53, G = 1 + floor(log(U) * inv_log1m_{p,q})
 * with inv_log1m_x = 1 / log1p(-x) supplied by the caller and log evaluated with basic
 * correctly rounded operations only (host oracles reproduce it bit for bit). */
typedef struct sc_csr sc_csr;
int32_t sc_generate_sbm(int64_t n, int32_t k, double p, double q, double inv_log1m_p,
                        double inv_log1m_q, uint64_t key0, uint64_t key1, int32_t device,
                        sc_csr **out);
int32_t sc_csr_info(const sc_csr *h, int64_t *n, int64_t *nnz, int64_t *n_generated);
/* host buffers, each nullable: row_ptr[n+1], col[nnz], deg[n], orig_ids[n] (generated id of
 * every kept vertex; block = orig_id / (n_generated / k)) */
int32_t sc_csr_download(const sc_csr *h, int64_t *row_ptr, int32_t *col, double *deg,
                        int32_t *orig_ids);
void sc_csr_destroy(sc_csr *h);
/* weights of a weighted device CSR (nnz doubles; SC_E_STATE for unit-weight CSRs) */
int32_t sc_csr_download_weights(const sc_csr *h, double *val);
/* config 4 (weighted random geometric cluster graph): k Gaussian-like
 * centres in [0,1]^3, n points, each joined to its knn (= 16) nearest by exact rounded d2,
 * union symmetrised, weight exp(-d2 / scale) (sc_generate_wt.cu states the law; replaces the
 * reference's brute-force unit-weight kNN builder, generate.py:176-220, which refuses
 * n > 50,000) */
int32_t sc_generate_knn3d(int64_t n, int32_t k, double sigma, int32_t knn, double scale,
                          uint64_t key0, uint64_t key1, int32_t device, sc_csr **out);
/* config 3 (degree-corrected SBM): block_offsets[nblocks + 1] from the
 * host (Dirichlet sizes), integer power-law expected degrees (A = dmin^a, B = dmax^a,
 * inv_a = 1/a, a = 1 - gamma), Chung-Lu stubs inside the block with probability 1 - mix,
 * weights Uniform(wlo, whi); isolated vertices dropped */
int32_t sc_generate_dcsbm(int64_t n, const int64_t *block_offsets, int32_t nblocks, double A,
                          double B, double inv_a, int32_t dmin, int32_t dmax, double mix,
                          double wlo, double whi, uint64_t key0, uint64_t key1, int32_t device,
                          sc_csr **out);
/* graph handle straight from a device-resident CSR (the column array is not copied to the
 * host; the handle does not keep a reference to h) */
int32_t sc_graph_create_from_csr(const sc_csr *h, uint32_t create_flags, sc_graph **out);
/* Row-block shard [row_lo, row_hi) straight from a device-resident CSR of the WHOLE graph on
 * this device (e.g. a device generator's output: every rank generates the graph and keeps its
 * rows, so no column ever visits the host); columns are renamed on the device through
 * d_slot_of (device, n int32: global vertex -> z slot of the shard plan).  ncols / col_offset
 * as sc_shard_create.  The CSR may be destroyed after the call. */
int32_t sc_shard_create_from_csr(const sc_csr *h, int64_t row_lo, int64_t row_hi,
                                 const int32_t *d_slot_of, int64_t ncols, int64_t col_offset,
                                 sc_graph **out);

/* ---- 1-D k-means replica ------------------------------------------------ */
/* points: host f (n doubles) or, with _from_graph, the f left on the device by the last
 * sc_power_iterate.  restarts batches independent restarts on the device. */
int32_t sc_kmeans_create(const double *points_host, int64_t n, int32_t device,
                         sc_kmeans **out);
int32_t sc_kmeans_create_from_graph(sc_graph *g, sc_kmeans **out);
/* points of dimension l (host, [n][l] row-major; 1 <= l <= 64).  Everything above applies;
 * distances are (sum x^2 - 2 sum x c) + sum c^2 with left-to-right sums (the reference uses
 * BLAS for the middle term, so for l > 1 labels match it up to exact distance ties), means
 * and cost keep the reference's np.add.at / einsum order per coordinate. */
int32_t sc_kmeans_create_nd(const double *points_host, int64_t n, int32_t l, int32_t device,
                            sc_kmeans **out);
void sc_kmeans_destroy(sc_kmeans *km);
/* k-means++ seeding for `restarts` restarts at once.  chosen[r*k + i] (in/out);
 * rounds start_round[r]..k-1 are run with uniforms[r*(k-1) + i-1] as round i's
 * rng.random() draw.  degenerate_out[r] = -1 if complete, else the first round at which
 * every D^2 weight was 0 (the caller replays rng.integers on the host and resumes). */
int32_t sc_kmeans_pp(sc_kmeans *km, int32_t k, int32_t restarts, const int32_t *start_round,
                     const double *uniforms, int64_t *chosen, int32_t *degenerate_out);
/* Lloyd from the points at chosen[r*k..], max_iters / tol as lloyd(); writes the final
 * cost and iteration count of every restart and the labels of the winning restart (first
 * restart with the strictly smallest cost). */
int32_t sc_kmeans_lloyd(sc_kmeans *km, int32_t k, int32_t restarts, const int64_t *chosen,
                        int32_t max_iters, double tol, int64_t *labels_out, double *costs_out,
                        int32_t *iters_out, int32_t *best_restart_out, double *ms_out);

/* Context options.  SC_KM_NO_COST_ASSERT: do not raise SC_E_INTERNAL when a restart's cost
 * goes up between iterations -- the reference's check is a Python `assert`
 * (kmeans.py:206) that `python -O` skips; with it skipped the increase simply stops that
 * restart (kmeans.py:207: prev - cost <= tol * prev holds for a negative gain).  The host
 * mirror sets the flag when Python runs without __debug__. */
#define SC_KM_NO_COST_ASSERT 0x1u
int32_t sc_kmeans_set_flags(sc_kmeans *km, uint32_t flags);

/* Fast mode (north star step 3): the same seeds, then Lloyd on the sorted values -- every
 * cluster is an interval of the sorted points, so an iteration is k binary searches plus
 * prefix-sum means and costs, all restarts' iterations in one kernel (one CTA per restart).
 * Tie rules, empty-cluster repair and stop rules follow the reference, but the sums are
 * prefix sums (not the reference's np.add.at / einsum order): not bit-exact, labels agree
 * with the replica except where a distance or stop decision sits within rounding.
 * 1-D points, k <= 2048. */
int32_t sc_kmeans_lloyd_sorted(sc_kmeans *km, int32_t k, int32_t restarts, const int64_t *chosen,
                               int32_t max_iters, double tol, int64_t *labels_out,
                               double *costs_out, int32_t *iters_out, int32_t *best_restart_out);

/* ---- exact sequential sums (the k-means replica's engine, exposed for testing) ---- */
/* totals[s] = ((vals[lo] + vals[lo+1]) + ...) left to right in double, lo..hi = segment s;
 * bit-identical to a scalar loop / np.cumsum(...)[-1].  chunk_starts (nullable) receives
 * the running value at every 256-element chunk start. */
int32_t sc_seqsum(const double *vals, int32_t nseg, const int64_t *seg_off, int32_t device,
                  double *totals, double *chunk_starts);

/* ---- evaluation metrics (metrics.py:36-201 of the reference) -------------------------- */
/* sums_out[q] = np.add.at(zeros(nkeys), keys, vals)[q] bit for bit (stable device sort by key,
 * then the exact sequential sums above); counts_out (nullable) = occurrences of every key.
 * Used for part volumes, the matched-volume intersections and the cut weights. */
int32_t sc_keyed_sums(const int32_t *keys, const double *vals, int64_t m, int32_t nkeys,
                      int32_t device, double *sums_out, int64_t *counts_out);
/* cut_out[c] = sum of the weights (1.0 if w is NULL) of the CSR entries (r, col) with
 * labels[r] = c != labels[col], added in CSR order (np.add.at, metrics.py:143-146) */
int32_t sc_cut_sums(const int64_t *row_ptr, const int32_t *col, const double *w,
                    const int64_t *labels, int64_t n, int64_t nnz, int32_t k, int32_t device,
                    double *cut_out);
/* counts_out[a * kb + b] = #{i : la[i] = a, lb[i] = b} (the contingency table) */
int32_t sc_contingency(const int64_t *la, const int64_t *lb, int64_t n, int32_t ka, int32_t kb,
                       int32_t device, int64_t *counts_out);

#ifdef __cplusplus
}
#endif
#endif /* SC_B200_H */
