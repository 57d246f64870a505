// sc_seqsum.cuh -- bit-exact, warp-parallel evaluation of a SEQUENTIAL floating-point sum
//
//     s_0 = 0,  s_{j+1} = fl(s_j + a_j)        (a_j >= 0, round-to-nearest-even)
//
// which is what numpy's cumsum / np.add.at and a scalar C loop compute, and which the
// reference's k-means depends on bit for bit (kmeans.py:89,117).
//
// Idea ("ulp-grid accumulation"): while the running sum stays inside one binade
// [2^e, 2^(e+1)], every representable value is a multiple of u = 2^(e-52), so
//     fl(s + a) = s + u * rne(a / u)
// where the rounding of a/u to an integer depends on s only through the parity of s/u
// (ties go to even).  An element therefore acts on S = s/u as a "parity map"
// (inc if S even, inc if S odd); parity maps compose associatively, so a run of elements
// inside one binade is summed exactly with integer prefix scans.  Where the running sum
// crosses into the next binade (at most ~60 times for a nonnegative sequence) the
// crossing element is added with one real fl() add and the grid is re-derived.
//
// Pipeline for a batch of segments (each summed independently from 0):
//   summarize  (one warp / chunk of kSeqChunk elements): approximate chunk sum and max
//   predict    (one warp / segment): approximate chunk starts -> expected binade per chunk
//   chunkmap   (one warp / chunk): parity map of the whole chunk on that binade's grid
//   compose    (one warp / segment): walks 32 chunks per step; chunks whose exact start
//              confirms the prediction advance in O(1), others are added sequentially by
//              one lane (warp_step_seq).  Emits the exact start of every chunk and the
//              exact segment total.
// Every decision is re-checked in compose against the exact running value, so the
// prediction only affects speed, never the result.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sc {

constexpr int kSeqChunk = 256;               // elements per chunk (8 per lane)
constexpr int kSeqPerLane = kSeqChunk / 32;
constexpr int kNoGrid = -2147483647 - 1;  // "no predicted grid" (grid exponents span [-971, 1074])

struct PMap {
    int64_t i0, i1;  // increment in ulp units when the incoming count is even / odd
};

__device__ __forceinline__ PMap pmap_id() { return PMap{0, 0}; }

// first A, then B
__device__ __forceinline__ PMap pmap_then(PMap A, PMap B) {
    const int64_t p0 = A.i0 & 1;        // parity after A from an even start
    const int64_t p1 = (1 + A.i1) & 1;  // parity after A from an odd start
    return PMap{A.i0 + (p0 ? B.i1 : B.i0), A.i1 + (p1 ? B.i1 : B.i0)};
}

__device__ __forceinline__ int64_t pmap_apply(PMap m, int64_t S) { return S + ((S & 1) ? m.i1 : m.i0); }

// element map of v = a/u (exact, v <= 2^53)
__device__ __forceinline__ PMap pmap_elem(double v) {
    if (!(v <= 9.0e15)) return PMap{int64_t(1) << 54, int64_t(1) << 54};  // beyond any grid
    const double fl = floor(v);
    const int64_t q = (int64_t)fl;
    const double f = v - fl;  // exact
    if (f > 0.5) return PMap{q + 1, q + 1};
    if (f < 0.5) return PMap{q, q};
    return PMap{q + (q & 1), q + ((q + 1) & 1)};  // tie: result even
}

// Binade of s >= 0: scale exponent k with u = 2^-k (so S = s * 2^k is an integer) and
// top = the count at which the grid changes (2^53, or 2^52 below the normal range).
struct Grid {
    int k;
    int64_t top;
};

__device__ __forceinline__ Grid grid_of(double s) {
    const uint64_t bits = (uint64_t)__double_as_longlong(s);
    const int eb = (int)((bits >> 52) & 0x7ff);
    if (eb == 0) return Grid{1074, int64_t(1) << 52};  // zero / subnormal: u = 2^-1074
    return Grid{1075 - eb, int64_t(1) << 53};          // e = eb-1023, u = 2^(e-52)
}

__device__ __forceinline__ double to_units(double a, int k) { return scalbn(a, k); }
__device__ __forceinline__ double from_units(int64_t S, int k) { return scalbn((double)S, -k); }

// ---------------------------------------------------------------------------
// warp helpers

__device__ __forceinline__ PMap shfl_pmap_up(PMap m, int d) {
    PMap r;
    r.i0 = __shfl_up_sync(0xffffffffu, m.i0, d);
    r.i1 = __shfl_up_sync(0xffffffffu, m.i1, d);
    return r;
}

// inclusive composition scan over lanes (lane order = sequence order)
__device__ __forceinline__ PMap warp_scan_pmap(PMap m) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const PMap o = shfl_pmap_up(m, d);
        if (lane >= d) m = pmap_then(o, m);
    }
    return m;
}

__device__ __forceinline__ PMap warp_exclusive(PMap incl) {
    const int lane = threadIdx.x & 31;
    PMap e = shfl_pmap_up(incl, 1);
    return lane == 0 ? pmap_id() : e;
}

// ---------------------------------------------------------------------------
// Exact stepping of up to 256 elements held 8 per lane (lane-contiguous), starting from
// the exact running value s: the chunk is staged in the warp's shared-memory slot `buf`
// (kSeqChunk doubles) and lane 0 adds it left to right -- the sequential sum itself, at the
// FP64 add latency (~2k cycles per chunk).  Used for the few chunks whose binade the
// prediction could not pin (grid crossings), where a warp-parallel walk would pay one full
// parity-map scan per crossing.  If `search`, stops at the first element whose running sum
// exceeds target and returns its index (else -1; s is then the chunk end).  Warp-uniform.
__device__ __forceinline__ int warp_step_seq(const double (&a)[kSeqPerLane], int n_valid,
                                             double &s, double target, bool search,
                                             double *buf) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
#pragma unroll
    for (int t = 0; t < kSeqPerLane; ++t) buf[lane * kSeqPerLane + t] = a[t];
    __syncwarp();
    double r = s;
    int hit = -1;
    if (lane == 0) {
#pragma unroll 8
        for (int j = 0; j < n_valid; ++j) {
            r = __dadd_rn(r, buf[j]);
            if (search && r > target) {
                hit = j;
                break;
            }
        }
    }
    s = __shfl_sync(0xffffffffu, r, 0);
    return __shfl_sync(0xffffffffu, hit, 0);
}

}  // namespace sc
