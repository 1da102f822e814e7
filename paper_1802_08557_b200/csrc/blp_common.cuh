// blp_common.cuh -- constants, batch descriptor and numpy-exact reductions
// shared by every simplex kernel variant.
//
// Bit-parity rules with the reference (numpy, /root/reference/pkg/src/batchlp):
//  * every product and sum is rounded separately: __dmul_rn / __dsub_rn /
//    __dadd_rn (numpy never fuses; nvcc would contract a - f*r into DFMA),
//    and the library is also compiled with -fmad=false;
//  * divisions are IEEE round-to-nearest (__ddiv_rn), as numpy's true_divide;
//  * arg-reductions return the FIRST extreme index, with NaN as the extreme
//    value, exactly like np.argmax / np.argmin (tableau.py:183, :212,
//    simplex.py:124).
#pragma once

#include <climits>
#include <cstdint>

namespace blp {

// Reference tolerances (tableau.py:37-39, simplex.py:26-31).
constexpr double kSentinel = 1e308;       // SENTINEL
constexpr double kTol = 1e-9;             // DEFAULT_TOL
constexpr double kPhase1ZeroTol = 1e-7;   // PHASE1_ZERO_TOL
constexpr double kDegenerateTol = 1e-9;   // DEGENERATE_RATIO_TOL
constexpr double kRedundantTol = 1e-7;    // REDUNDANT_ROW_TOL

constexpr unsigned kFull = 0xffffffffu;
constexpr int kNone = INT_MAX;            // "no candidate" index

// Per-LP status codes, equal to BLP_STATUS_* in include/blp.h.
enum : int8_t {
    kOptimal = 0,
    kUnbounded = 1,
    kInfeasible = 2,
    kIterationLimit = 3,
    kErrPhase1Unbounded = 4,
    kInvalid = 5,          // non-finite entry: the caller raises validate()'s ValueError
};

// SolverLimits (simplex.py:34-60); same layout as blp_limits.
struct Limits {
    int max_iterations;    // <= 0: 50*(m+n)
    int anti_cycling;
    int degenerate_limit;  // < 0: max(m,1)
    int reserved;
};

// One launch's worth of work: a packed batch of same-shaped LPs.
struct Batch {
    const double *A;       // [count][m][n] row-major, or [m][n] if shared_Ab
    const double *b;       // [count][m], or [m] if shared_Ab
    const double *c;       // [count][n]
    long long count;
    int m, n;
    int shared_Ab;
    int8_t *status;        // [count]
    double *objective;     // [count]
    double *x;             // [count][n]
    int *it1, *it2;        // [count]
    int *next_lp;          // LP queue head of the persistent grid, zero at launch
    double *gtab;          // global tableau slots (HBM-streamed variant), one per CTA
    long long gtab_stride; // doubles per slot
    Limits lim;
    // Deferral (lazy kernel -> dense kernel): the lazy kernel appends the LPs it
    // hands over to defer_list; a dense kernel launched with defer_list set solves
    // exactly those (*defer_count of them, read on the device).
    int *defer_list;
    int *defer_count;
    // Shared phase 1 (support mode, condensed kernels): the restored post-phase-1 tableau
    // and its status, written once per batch by condensed_phase1_kernel; null otherwise.
    const double *p1state;
    // Lazy kernel split mode: validation-chunk queue head and per-LP "non-finite A" flags
    int *vq;
    unsigned char *vflag;
    int vfirst;            // CTAs that take validation chunks before LPs (the rest: LPs first)
    int lazy_discard = 0;  // lazy kernel: discard a solved LP's replay history from L2
};

// Number of LPs a kernel launch processes, and the batch index of its k-th.
__device__ __forceinline__ long long batch_count(const Batch &B) {
    return B.defer_list ? (long long)*B.defer_count : B.count;
}
__device__ __forceinline__ long long batch_lp(const Batch &B, long long k) {
    return B.defer_list ? (long long)B.defer_list[k] : k;
}

// np.argmax order: NaN first (lowest index among NaNs), then larger value,
// then lower index.  kNone marks an empty slot.
__device__ __forceinline__ bool argmax_before(double a, int ia, double b, int ib) {
    const bool na = a != a, nb = b != b;
    if (na || nb) return na && (!nb || ia < ib);
    return a > b || (a == b && ia < ib);
}

// np.argmin order: NaN first, then smaller value, then lower index.
__device__ __forceinline__ bool argmin_before(double a, int ia, double b, int ib) {
    const bool na = a != a, nb = b != b;
    if (na || nb) return na && (!nb || ia < ib);
    return a < b || (a == b && ia < ib);
}

// a / b for tableau entries.  A zero numerator returns a itself (a signed
// zero, value-equal to IEEE's 0/b); every other quotient is __ddiv_rn.  The
// zero is replaced by 1 before dividing (not branched around: the compiler
// if-converts a branch and divides anyway), because __ddiv_rn's range check
// sends a zero numerator -- in any lane -- to the slow subroutine for the
// whole warp, and sparse pivot rows are full of zeros.
// p ? a : b as an opaque PTX selp: the compiler cannot see through it (so it
// cannot undo the operand substitutions below) and, used as a register-array
// select, it never turns into a computed index (which would demote the array
// to local memory).
__device__ __forceinline__ double selp_f64(double a, double b, bool p) {
    double r;
    asm("{ .reg .pred q; setp.ne.u32 q, %3, 0; selp.f64 %0, %1, %2, q; }" : "=d"(r) : "d"(a), "d"(b), "r"((unsigned)p));
    return r;
}

// Ordered shared-memory accesses (volatile: emitted in program order), used
// where a hand-pipelined loop must keep its loads ahead of earlier stores.
__device__ __forceinline__ double lds_f64(unsigned addr) {
    double v;
    asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void lds_v2_f64(unsigned addr, double &x, double &y) {
    asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(addr) : "memory");
}
__device__ __forceinline__ void sts_f64(unsigned addr, double v) {
    asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

__device__ __forceinline__ double div_entry(double a, double b) {
    const bool z = a == 0.0;
    const double q = __ddiv_rn(selp_f64(1.0, a, z), b);
    return z ? a : q;
}

// choose_leaving's ratio (tableau.py:210-211): rhs / a where a > tol, else
// SENTINEL.  Operands of the discarded lanes are made harmless for the same
// fast-path reason as div_entry.
__device__ __forceinline__ double ratio_entry(double rhs, double a) {
    const bool ok = a > kTol;
    const double q = div_entry(selp_f64(rhs, 1.0, ok), selp_f64(a, 1.0, ok));
    return ok ? q : kSentinel;
}

// Butterfly reductions: every lane ends with the warp-wide winner.
__device__ __forceinline__ void warp_argmax(double &v, int &i) {
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        const double ov = __shfl_xor_sync(kFull, v, off);
        const int oi = __shfl_xor_sync(kFull, i, off);
        if (argmax_before(ov, oi, v, i)) { v = ov; i = oi; }
    }
}

__device__ __forceinline__ void warp_argmin(double &v, int &i) {
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        const double ov = __shfl_xor_sync(kFull, v, off);
        const int oi = __shfl_xor_sync(kFull, i, off);
        if (argmin_before(ov, oi, v, i)) { v = ov; i = oi; }
    }
}

__device__ __forceinline__ int warp_min_int(int v) {
    return (int)__reduce_min_sync(kFull, (unsigned)v);
}

}  // namespace blp
