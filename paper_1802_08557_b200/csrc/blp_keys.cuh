// blp_keys.cuh -- numpy-exact arg-reductions on order-preserving 64-bit keys.
//
// np.argmax / np.argmin (tableau.py:183, :212; simplex.py:124) return the
// first index of the extreme value, NaN counting as the extreme, and treat
// -0.0 == +0.0.  Mapping each double to an unsigned key whose integer order
// is that total order turns every arg-reduction into three warp-wide
// redux.sync instructions (max of the high word, max of the low word among
// the winners, min of the index among the full-key winners) instead of a
// five-level shuffle tree of double compares.
#pragma once

#include "blp_common.cuh"

namespace blp {

// Key whose unsigned order is numpy's max order: -inf < ... < -0 == +0 < ... < +inf < NaN.
// Branch-free (every lane computes the key, NaN selected last): C2 5.04 -> 4.97 ms, C3
// 72.8 -> 71.9 per 2e4 against the early-return form, which compiled to a divergent branch.
__device__ __forceinline__ unsigned long long key_max(double v) {
    const long long b = __double_as_longlong(v == 0.0 ? 0.0 : v);
    const unsigned long long k = b < 0 ? ~(unsigned long long)b : ((unsigned long long)b | 0x8000000000000000ull);
    return v != v ? ~0ull : k;
}

// Key whose unsigned order is numpy's min order: NaN < -inf < ... < +inf.
__device__ __forceinline__ unsigned long long key_min(double v) {
    const long long b = __double_as_longlong(v == 0.0 ? 0.0 : v);
    const unsigned long long k = b < 0 ? ~(unsigned long long)b : ((unsigned long long)b | 0x8000000000000000ull);
    return v != v ? 0ull : k;   // branch-free, as key_max
}

constexpr unsigned long long kKeyEmptyMax = 0ull;    // no candidate (max reductions)
constexpr unsigned long long kKeyEmptyMin = ~0ull;   // no candidate (min reductions)

__device__ __forceinline__ unsigned long long warp_max_key(unsigned long long k) {
    const unsigned hi = __reduce_max_sync(kFull, (unsigned)(k >> 32));
    const unsigned lo = __reduce_max_sync(kFull, (unsigned)(k >> 32) == hi ? (unsigned)k : 0u);
    return ((unsigned long long)hi << 32) | lo;
}

__device__ __forceinline__ unsigned long long warp_min_key(unsigned long long k) {
    const unsigned hi = __reduce_min_sync(kFull, (unsigned)(k >> 32));
    const unsigned lo = __reduce_min_sync(kFull, (unsigned)(k >> 32) == hi ? (unsigned)k : ~0u);
    return ((unsigned long long)hi << 32) | lo;
}

// Lowest index among the lanes holding the winning key (kNone if none).
__device__ __forceinline__ int warp_index_of(unsigned long long k, unsigned long long win, int idx) {
    return (int)__reduce_min_sync(kFull, k == win ? (unsigned)idx : (unsigned)kNone);
}

// Keys of the reference thresholds, for comparisons done on keys.
__device__ __forceinline__ unsigned long long key_of_tol() { return key_max(kTol); }

// a[i] for a warp-uniform runtime index: a uniform branch tree down to
// groups of 8, then 7 selp's.  Register arrays must only ever be indexed
// statically -- a computed index (or a switch the compiler turns into one)
// sends the whole row to local memory.
template <int LO, int N, int CPW>
struct RegPicker {
    static __device__ __forceinline__ double get(const double (&a)[CPW], int i) {
        if constexpr (N == 1) {
            return a[LO];
        } else if constexpr (N <= 8) {
            // a select tree on the index bits below the group (depth log2 N, not an N-1 chain)
            const double lo = RegPicker<LO, N / 2, CPW>::get(a, i);
            const double hi = RegPicker<LO + N / 2, N - N / 2, CPW>::get(a, i);
            return selp_f64(hi, lo, i >= LO + N / 2);
        } else {
            if (i < LO + N / 2) return RegPicker<LO, N / 2, CPW>::get(a, i);
            return RegPicker<LO + N / 2, N - N / 2, CPW>::get(a, i);
        }
    }
};

template <int CPW>
__device__ __forceinline__ double reg_pick(const double (&a)[CPW], int i) {
    return RegPicker<0, CPW, CPW>::get(a, i);
}

}  // namespace blp
