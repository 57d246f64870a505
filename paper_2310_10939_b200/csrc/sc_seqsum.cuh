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
//              confirms the prediction advance in O(1), others are stepped element by
//              element (still 256 elements per warp step).  Emits the exact start of
//              every chunk and the exact segment total.
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
// the exact running value s.  Advances s over all n_valid elements.  If `target` >= 0 is
// given (k-means++ search), stops at the first element whose running sum exceeds target
// and returns its index (else -1).  Uniform across the warp.
__device__ __forceinline__ int warp_step_elements(const double (&a)[kSeqPerLane], int n_valid,
                                                  double &s, double target, bool search) {
    const int lane = threadIdx.x & 31;
    int pos = 0;
    while (pos < n_valid) {
        const Grid g = grid_of(s);
        const int64_t S0 = (int64_t)to_units(s, g.k);
        // lane map over its elements >= pos
        PMap lm = pmap_id();
        double v[kSeqPerLane];
#pragma unroll
        for (int t = 0; t < kSeqPerLane; ++t) {
            const int j = lane * kSeqPerLane + t;
            v[t] = (j >= pos && j < n_valid) ? to_units(a[t], g.k) : 0.0;
            lm = pmap_then(lm, pmap_elem(v[t]));
        }
        const PMap excl = warp_exclusive(warp_scan_pmap(lm));
        int64_t S = pmap_apply(excl, S0);
        // walk this lane's elements: first invalid (grid change) or search hit
        int bad = 1 << 30, hit = 1 << 30;
#pragma unroll
        for (int t = 0; t < kSeqPerLane; ++t) {
            const int j = lane * kSeqPerLane + t;
            if (j >= pos && j < n_valid && bad == (1 << 30) && hit == (1 << 30)) {
                if ((double)(g.top - S) < v[t] || !(a[t] >= 0.0) || !isfinite(a[t])) {
                    bad = j;
                } else {
                    S = pmap_apply(pmap_elem(v[t]), S);
                    if (search && from_units(S, g.k) > target) hit = j;
                }
            }
        }
        int first_bad = bad, first_hit = hit;
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            first_bad = min(first_bad, __shfl_xor_sync(0xffffffffu, first_bad, d));
            first_hit = min(first_hit, __shfl_xor_sync(0xffffffffu, first_hit, d));
        }
        if (search && first_hit < first_bad) {
            // running value right after first_hit, computed by its lane
            return first_hit;
        }
        const int stop = min(first_bad, n_valid);
        // exact running value just before `stop`: owner lane of element stop-1 recomputes
        // (cheap: re-walk its elements)
        {
            const int64_t Sst = pmap_apply(excl, S0);
            int64_t Sw = Sst;
#pragma unroll
            for (int t = 0; t < kSeqPerLane; ++t) {
                const int j = lane * kSeqPerLane + t;
                if (j >= pos && j < stop) Sw = pmap_apply(pmap_elem(v[t]), Sw);
            }
            // lane owning element stop-1 (or the lane before the range if stop == pos)
            const int owner = stop > pos ? (stop - 1) / kSeqPerLane : -1;
            if (owner >= 0) {
                const int64_t Sfin = __shfl_sync(0xffffffffu, Sw, owner);
                s = from_units(Sfin, g.k);
            }
        }
        if (first_bad >= n_valid) return -1;
        // one real add for the grid-crossing element (owner lane broadcasts the addend)
        const int ol = first_bad / kSeqPerLane, ot = first_bad % kSeqPerLane;
        double ab = 0.0;
#pragma unroll
        for (int t = 0; t < kSeqPerLane; ++t)
            if (t == ot) ab = a[t];
        ab = __shfl_sync(0xffffffffu, ab, ol);
        s = __dadd_rn(s, ab);
        if (search && s > target) return first_bad;
        pos = first_bad + 1;
    }
    return -1;
}

}  // namespace sc
