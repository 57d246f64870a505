// sc_hostcopy.cuh -- host -> device uploads of large arrays that may live in ordinary
// (pageable) host memory, as a reference caller's numpy CSR does.
//
// A pageable cudaMemcpyAsync is staged by the driver through its own small pinned buffer, one
// chunk at a time on the calling thread (~11 GB/s on the B200 box: config 2's 192 MB CSR took
// ~17 ms against ~3.5 ms from pinned memory).  Here a process-wide pool of pinned slots is
// filled by several host threads in parallel (memcpy out of the caller's array) while the copy
// engine drains the slots already filled, so the upload runs near the PCIe rate from pageable
// arrays too.  Pinned (page-locked or registered) sources, and small arrays, go straight to
// cudaMemcpyAsync.
//
// Ordering contract (same as cudaMemcpyAsync from pageable memory): when h2d_upload returns,
// every byte of the source has been read (the caller may free or modify it); the device writes
// are ordered before any work enqueued on `s` afterwards.
// This header is included inside namespace sc.

constexpr size_t kStageChunk = size_t(4) << 20;   // bytes per slot
constexpr int kStageSlots = 2;                     // slots per thread
constexpr int kStageMaxThreads = 8;
constexpr size_t kStageMin = size_t(16) << 20;     // smaller (or pinned) sources: direct copy

struct StagePool {
    int device = -1;
    int nthr = 0;
    char *buf = nullptr;  // nthr * kStageSlots * kStageChunk pinned bytes
    cudaStream_t st[kStageMaxThreads] = {};
    cudaEvent_t ev[kStageMaxThreads][kStageSlots] = {};
    cudaEvent_t done[kStageMaxThreads] = {};
    std::mutex mu;  // one staged upload at a time per device
};

inline StagePool *stage_pool(int device) {
    static std::mutex mu;
    static StagePool pools[64];
    if (device < 0 || device >= 64) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    StagePool &p = pools[device];
    if (p.device == device) return &p;
    if (p.device == -2) return nullptr;  // creation failed before: direct copies only
    int nthr = (int)std::thread::hardware_concurrency() / 2;
    if (const char *e = std::getenv("SC_STAGE_THREADS")) nthr = std::atoi(e);
    nthr = std::max(1, std::min(kStageMaxThreads, nthr));
    if (nthr < 2) {
        p.device = -2;
        return nullptr;
    }
    bool ok = cudaHostAlloc((void **)&p.buf, (size_t)nthr * kStageSlots * kStageChunk,
                            cudaHostAllocPortable) == cudaSuccess;
    for (int t = 0; ok && t < nthr; ++t) {
        ok = cudaStreamCreateWithFlags(&p.st[t], cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&p.done[t], cudaEventDisableTiming) == cudaSuccess;
        for (int i = 0; ok && i < kStageSlots; ++i)
            ok = cudaEventCreateWithFlags(&p.ev[t][i], cudaEventDisableTiming) == cudaSuccess;
    }
    if (!ok) {
        cudaGetLastError();
        p.device = -2;
        return nullptr;
    }
    p.nthr = nthr;
    p.device = device;
    return &p;
}

inline bool host_is_pinned(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// true when h2d_upload would stage `src` (large and pageable), i.e. the call is host-bound
inline bool h2d_staged(const void *src, size_t bytes) {
    return bytes >= kStageMin && !host_is_pinned(src) && !std::getenv("SC_STAGE_OFF");
}

inline cudaError_t h2d_upload(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    if (!bytes) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e) return e;
    StagePool *P = h2d_staged(src, bytes) ? stage_pool(dev) : nullptr;
    if (!P) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
    std::lock_guard<std::mutex> lk(P->mu);
    // the pool's streams start after everything already enqueued on s (e.g. allocations)
    cudaEvent_t start;
    if ((e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming))) return e;
    cudaEventRecord(start, s);
    const size_t nchunk = (bytes + kStageChunk - 1) / kStageChunk;
    const int nthr = (int)std::min<size_t>((size_t)P->nthr, nchunk);
    std::vector<cudaError_t> err(nthr, cudaSuccess);
    auto work = [&](int t) {
        cudaError_t r = cudaSetDevice(dev);
        if (!r) r = cudaStreamWaitEvent(P->st[t], start, 0);
        int use = 0;
        for (size_t c = t; !r && c < nchunk; c += nthr, use ^= 1) {
            char *slot = P->buf + ((size_t)t * kStageSlots + use) * kStageChunk;
            r = cudaEventSynchronize(P->ev[t][use]);  // the slot's previous DMA has drained
            if (r) break;
            const size_t off = c * kStageChunk, len = std::min(kStageChunk, bytes - off);
            std::memcpy(slot, (const char *)src + off, len);
            r = cudaMemcpyAsync((char *)dst + off, slot, len, cudaMemcpyHostToDevice, P->st[t]);
            if (!r) r = cudaEventRecord(P->ev[t][use], P->st[t]);
        }
        if (!r) r = cudaEventRecord(P->done[t], P->st[t]);
        err[t] = r;
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nthr; ++t) th.emplace_back(work, t);
    work(0);
    for (auto &x : th) x.join();
    cudaEventDestroy(start);
    for (int t = 0; t < nthr; ++t) {
        if (err[t]) return err[t];
        if ((e = cudaStreamWaitEvent(s, P->done[t], 0))) return e;
    }
    // slots are reused by the next upload only after their DMA (ev) has completed, and the
    // caller's source was fully read above
    return cudaSuccess;
}
