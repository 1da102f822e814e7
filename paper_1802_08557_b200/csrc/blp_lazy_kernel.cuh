// blp_lazy_kernel.cuh -- exact LAZY tableau for large LPs that finish in few
// pivots (C5: 500 x 500, ~14 pivots on a 501 x 1001 tableau).
//
// The dense algorithm (tableau.py:218-244) applies, at pivot t with leaving
// row l_t, entering column e_t and pivot element pe_t,
//     r^t_j = a_{l_t j} / pe_t                       (the new row l_t)
//     a_ij <- a_ij - f^t_i * r^t_j   for i != l_t,   f^t_i = a_{i e_t} (before pivot t)
// to every cell.  The algorithm, however, only ever READS the reduced-cost
// row, the rhs column, the entering column and the pivot row.  So every other
// cell can be left unevaluated: a cell's value after pivot k is recovered
// exactly by replaying its own history,
//     t0 = last pivot with l_{t0} = i (0 if none):  a = t0 ? r^{t0}_j : a^0_ij
//     for t = t0+1 .. k:                           a = a - f^t_i * r^t_j
// -- the very operations, operands and rounding order of the dense update, so
// the value is bit-identical to what the dense tableau would hold.  This
// kernel keeps the reduced-cost row, the rhs column and the basis dense (in
// shared memory), stores the history vectors f^t (m) and r^t (n+m) in a
// per-CTA global (L2-resident) scratch, and evaluates the entering column
// (m cells) and the pivot row (n+m cells) by replay: O((n+m) k) work per pivot
// instead of O(m (n+m)).
//
// Scope: single-phase LPs (b >= 0, so no artificials and every row sign is
// +1) that finish within kLazyMaxPivots pivots.  An LP that needs phase 1 or
// more pivots is appended to a deferral list and solved from scratch by the
// dense cluster kernel launched right after on the same stream (identical
// results either way).  Validation (model.py:263-301) still reads every
// entry of A (streamed with 16-byte evict-first loads before the solve; the
// CTAs resident on an SM drift apart, so one CTA's stream overlaps another's
// latency-bound solve) -- C5 is bound by one HBM read of its inputs.  In
// support mode (shared A) lazy_validate_kernel checks the polytope once.
#pragma once

#include "blp_common.cuh"
#include "blp_keys.cuh"

namespace blp {

constexpr int kLazyMaxPivots = 64;

#ifndef LAZY_SCAN_U
#define LAZY_SCAN_U 4
#endif
// Validation-stream load form, measured (bench-style back-to-back steps; C5 1e4 / random
// 300 x 300 5e3 / random 100 x 100 2e4, ms): 0 __ldcs 5.177 / 1.358 / 0.854 (default);
// 1 ld.nc.L1::no_allocate.L2::256B 5.204 / 1.357 / 0.855; 2 __ldcg 5.425 / 1.353 / 0.837;
// 3 L1::no_allocate + L2 evict_first policy 5.189 / 1.360 / 0.856.
#ifndef LAZY_SCAN_MODE
#define LAZY_SCAN_MODE 0
#endif
// One 16-byte load of the validation stream (read once: evict-first).
__device__ __forceinline__ double2 lazy_scan_load(const double2 *p) {
#if LAZY_SCAN_MODE == 1
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
#elif LAZY_SCAN_MODE == 2
    return __ldcg(p);
#elif LAZY_SCAN_MODE == 3
    double2 v;
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
#else
    return __ldcs(p);
#endif
}

struct LazyPart {
    unsigned long long ckey[32];
    int cidx[32], cbl[32];
    unsigned long long lkey[32];
    int lrow[32];
    int flag[32];
};

struct LazyLayout {
    size_t off_rhs, off_rc, off_fcur, off_basis, off_last, off_isb, off_part, off_misc, off_first, off_urow;
    size_t bytes;
};

__host__ __device__ inline LazyLayout make_lazy_layout(int m, int n) {
    LazyLayout L;
    const int nv = n + m, mm = m > 0 ? m : 1;
    size_t o = 0;
    auto al = [](size_t x) { return (x + 15) / 16 * 16; };
    L.off_rhs = o;   o = al(o + (size_t)mm * 8);
    L.off_rc = o;    o = al(o + (size_t)nv * 8);
    L.off_fcur = o;  o = al(o + (size_t)mm * 8);
    L.off_basis = o; o = al(o + (size_t)mm * 4);
    L.off_last = o;  o = al(o + (size_t)mm * 4);
    L.off_isb = o;   o = al(o + (size_t)nv);
    L.off_part = o;  o = al(o + sizeof(LazyPart));
    L.off_misc = o;  o = al(o + 64);
    L.off_first = o; o = al(o + (size_t)mm * 4);
    L.off_urow = o;  o = al(o + (size_t)kLazyMaxPivots * 4);
    L.bytes = o;
    return L;
}

// Scratch doubles per CTA: kLazyMaxPivots x (f^t: m, r^t: n+m).
__host__ __device__ inline long long lazy_scratch_doubles(int m, int n) {
    return (long long)kLazyMaxPivots * (2LL * m + n);
}

// Initial tableau cell a^0_ij of a single-phase LP (all row signs +1):
// [A | I] (tableau.py:149-170).
// Load-path knobs, measured (C5 / C4 / random 100x100): plain loads 5.74 / 65.0 / 0.83 ms;
// __ldcg history 6.39 / 73.2 / 0.95; __ldg for A no change.  Round 2 (C5 1e4 / random
// 100 x 100 2e4, two alternating runs each): history loads and stores with an L2 evict_last
// policy (mode 2) 5.34-5.35 / 0.860-0.861 ms vs plain 5.396-5.397 / 0.885-0.889 -- the default.
#ifndef LAZY_HIST_MODE
#define LAZY_HIST_MODE 2
#endif
#ifndef LAZY_A_MODE
#define LAZY_A_MODE 0
#endif
__device__ __forceinline__ double lazy_a0(const double *Ag, int n, int i, int j) {
#if LAZY_A_MODE == 1
    return j < n ? __ldg(Ag + (size_t)i * n + j) : ((j - n == i) ? 1.0 : 0.0);
#else
    return j < n ? Ag[(size_t)i * n + j] : ((j - n == i) ? 1.0 : 0.0);
#endif
}
// A replay-history load (written earlier by this CTA).  LAZY_HIST_MODE 2: history loads and
// stores carry an L2 evict_last policy (the validation stream is evict-first).
__device__ __forceinline__ unsigned long long lazy_pol() {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double lazy_h(const double *p) {
#if LAZY_HIST_MODE == 1
    return __ldcg(p);
#elif LAZY_HIST_MODE == 2
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(lazy_pol()));
    return v;
#else
    return *p;
#endif
}
__device__ __forceinline__ void lazy_hs(double *p, double v) {
#if LAZY_HIST_MODE == 2
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(lazy_pol()) : "memory");
#else
    *p = v;
#endif
}

// Replay a cell's update history from pivot t to k-1: a -= v_t * h[t], v_t
// loaded from p + t*stride (this cell's own history, coalesced across the
// warp), h the staged broadcast operand.  Loads are issued 8 at a time so a
// history of k pivots costs k/8 L2 round trips, not k.
__device__ __forceinline__ double lazy_replay(double a, const double *p, int stride, const double *h, int t, int k) {
    const double *q = p + (ptrdiff_t)t * stride;
    for (; t + 8 <= k; t += 8, q += 8 * (ptrdiff_t)stride) {      // full batches: no predicates
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = lazy_h(q + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) a = __dsub_rn(a, __dmul_rn(v[u], h[t + u]));
    }
    const int rem = k - t;                                            // tail: one predicated batch
    if (rem > 0) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = u < rem ? lazy_h(q + u * stride) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (u < rem) a = __dsub_rn(a, __dmul_rn(v[u], h[t + u]));
    }
    return a;
}
// Warp-specialised validation stream (WS = 1): the last kLazyScanWarps warps of
// the CTA stream the LP's A through a shared-memory ring filled by bulk async
// copies (cp.async.bulk, completion on an mbarrier per stage) and check it,
// while the other warps run the pivots of the same LP (named barrier 1), so an
// LP costs max(stream, solve) instead of their sum; the in-flight bytes are the
// ring's (kLazyRing x kLazyChunk per CTA), not registers.
constexpr int kLazyScanWarps = 4;
constexpr int kLazyRing = 4;
constexpr int kLazyChunk = 16384;
// Per-warp staging of the replay's broadcast operand (kLazyMaxPivots doubles per
// warp) follows the layout; the ring follows that.
__host__ __device__ inline size_t lazy_stage_bytes(int nt, int rp) { return rp ? (size_t)(nt / 32) * kLazyMaxPivots * 8 : 0; }
__host__ __device__ inline size_t lazy_ring_offset(const LazyLayout &L, int nt, int rp) {
    return (L.bytes + lazy_stage_bytes(nt, rp) + 127) / 128 * 128;
}
__host__ __device__ inline size_t lazy_smem_bytes(int m, int n, int ws, int nt, int rp) {
    const LazyLayout L = make_lazy_layout(m, n);
    return ws ? lazy_ring_offset(L, nt, rp) + (size_t)kLazyRing * kLazyChunk : L.bytes + lazy_stage_bytes(nt, rp);
}
__device__ __forceinline__ void lazy_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void lazy_mbar_wait(unsigned bar, unsigned parity) {
    unsigned done;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    } while (!done);
}
__device__ __forceinline__ void lazy_bulk_load(unsigned dst, const void *src, unsigned bytes, unsigned bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// FS = 1: the first KF pivots' f^t vectors live in shared memory after the
// layout (KF from the launch's dynamic shared-memory size), later ones in the
// L2 scratch.  FS = 2: their r^t vectors too (f^t then r^t per pivot) -- every
// later pivot replays the whole r history of the pivot row, so the first
// pivots' rows are the most re-read bytes of the kernel.
// SPX = 1 (m >= kLazyMaxPivots, direct replay): the slack block of the tableau is
// E_k..E_1 I, which differs from I only in the columns of rows that have been pivot rows,
// so the slack column of a row never pivoted on is exactly e_i (its pivot-row entries r^t
// are exactly +0: 0 / pe with pe > 0, replayed as a - f * (+0) = a).  Those columns are
// neither evaluated nor stored: the pivot row covers the n structural columns plus the
// slack columns of rows already pivoted on, and r^t keeps a slack entry per first-pivot
// slot u (row urow[u]) at offset n + u -- half the row replay and a third less history for C5.
// Measured slower and kept opt-in (BLP_LAZY_SPARSE=1; parity-tested): C5 1e4 5.61 vs 5.34 ms,
// random 100 x 100 (2e4) 0.918 vs 0.870, random 300 x 300 1.416 vs 1.385 -- a pivot is
// latency-bound, the 512 threads still need two column rounds (n + k > 512 for C5), and the
// skipped history loads were L2 hits.
template <int NT, int MINB, int WS, int RP, int FS = 0, int SPX = 0>
__global__ void __launch_bounds__(NT, MINB)
lazy_kernel(Batch B) {
    extern __shared__ __align__(16) unsigned char smem[];
    // the dense pass that follows may be a programmatic dependent launch: let it be scheduled
    // now (it waits in griddepcontrol.wait for this grid to complete)
    asm volatile("griddepcontrol.launch_dependents;");
    const int m = B.m, n = B.n, nv = n + m;
    const LazyLayout L = make_lazy_layout(m, n);
    double *rhs = reinterpret_cast<double *>(smem + L.off_rhs);
    double *rc = reinterpret_cast<double *>(smem + L.off_rc);
    double *fcur = reinterpret_cast<double *>(smem + L.off_fcur);
    int *basis = reinterpret_cast<int *>(smem + L.off_basis);
    int *lastpiv = reinterpret_cast<int *>(smem + L.off_last);     // 1-based pivot number, 0 = never
    unsigned char *isb = smem + L.off_isb;
    LazyPart *P = reinterpret_cast<LazyPart *>(smem + L.off_part);
    long long *s_lp = reinterpret_cast<long long *>(smem + L.off_misc);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int PT = WS ? NT - 32 * kLazyScanWarps : NT;    // pivot threads
    constexpr int NW = PT / 32;
    static_assert(!WS || PT >= 64, "WS needs pivot warps");
    static_assert(FS == 0 || RP == 0, "shared-memory history only with the direct replay");
    static_assert(SPX == 0 || RP == 0, "sparse slack history only with the direct replay");
    int *firstp = reinterpret_cast<int *>(smem + L.off_first);    // row -> first pivot slot, -1
    int *urow = reinterpret_cast<int *>(smem + L.off_urow);       // slot u -> row first pivoted there, -1
    int *s_res = reinterpret_cast<int *>(smem + L.off_misc + 8);             // status, iterations, deferred
    unsigned long long *fullb = reinterpret_cast<unsigned long long *>(smem + L.off_misc + 32);
    const unsigned ring = (unsigned)__cvta_generic_to_shared(smem + lazy_ring_offset(L, NT, RP));
    double *hw = reinterpret_cast<double *>(smem + L.bytes) + warp * kLazyMaxPivots;   // this warp's staging
    if (WS) {
        if (tid == 0) {
            for (int s2 = 0; s2 < kLazyRing; ++s2)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(fullb + s2)));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    unsigned gseq = 0;                                       // ring chunks consumed (scanner warps)
    auto pbar = [&]() { if (WS) lazy_bar(1, PT); else __syncthreads(); };
    // history: F[t] (m doubles), R[t] (nv doubles), t = 0 .. kLazyMaxPivots-1 (pivot t+1)
    // history layout: pivot-major across the CTAs -- row t of CTA b (f^t: m doubles, then
    // r^t: nv) at ((t * G + b) * (m + nv)) -- so the first pivots' history of every resident
    // CTA is one contiguous range (the launch marks it persisting in L2; launch_lazy)
    const size_t HS = (size_t)gridDim.x * (size_t)(m + nv);     // pivot t -> t+1, same CTA
    double *Fh = B.gtab + (size_t)blockIdx.x * (size_t)(m + nv);
    double *Rh = Fh + m;
    double *Fs = nullptr, *Rs = nullptr;
    int KF = 0;
    if constexpr (FS) {
        unsigned dyn;
        asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
        const size_t base = (lazy_smem_bytes(m, n, WS, NT, RP) + 15) / 16 * 16;
        const size_t per = 8 * (size_t)(m > 0 ? m : 1) + (FS == 2 ? 8 * (size_t)nv : 0);
        KF = (int)min((size_t)kLazyMaxPivots, (dyn - base) / per);
        Fs = reinterpret_cast<double *>(smem + base);
        Rs = Fs + (size_t)KF * m;                   // FS == 2: r^t of pivot t at Rs + t * nv
    }
    auto Fget = [&](int t, int i) -> double {
        if constexpr (FS) { if (t < KF) return Fs[(size_t)t * m + i]; }
        return lazy_h(Fh + (size_t)t * HS + i);
    };
    auto Rget = [&](int t, int j) -> double {
        if constexpr (FS == 2) { if (t < KF) return Rs[(size_t)t * nv + j]; }
        return lazy_h(Rh + (size_t)t * HS + j);
    };
    // SPX: r^t of column j (slack column n + i: u = row i's first pivot slot, -1 if none)
    auto RgetS = [&](int t, int j, int u) -> double {
        if (SPX && j >= n) return (u >= 0 && u <= t) ? Rget(t, n + u) : 0.0;
        return Rget(t, j);
    };
    const int max_iter = B.lim.max_iterations > 0 ? B.lim.max_iterations : 50 * (m + n);
    const int trigger = B.lim.degenerate_limit >= 0 ? B.lim.degenerate_limit : (m > 1 ? m : 1);
    const unsigned long long kSent = key_max(kSentinel), kDeg = key_max(kDegenerateTol), kTolK = key_max(kTol);

    // Split mode (B.vq set; independent LPs, non-WS form): the validation of A runs as its own
    // work queue instead of inline before each solve.  The first half of the CTAs take
    // validation chunks (one LP's A each) first, the second half LPs to solve first; a CTA whose
    // queue is empty takes from the other one, so the HBM stream of A (the kernel's floor)
    // overlaps the latency-bound solves across CTAs.  A flagged LP is made BLP_STATUS_INVALID
    // by lazy_finalize_kernel after the launch sequence.
    const bool split = !WS && !B.shared_Ab && B.vq != nullptr;
    const bool validator_first = split && (int)blockIdx.x < B.vfirst;
    for (;;) {
        if (tid == 0) {
            long long got = B.count;
            int kind = 0;
            if (!split) {
                got = atomicAdd(B.next_lp, 1);
            } else {
                for (int attempt = 0; attempt < 2 && got >= B.count; ++attempt) {
                    kind = (attempt == 0) == validator_first ? 1 : 0;
                    if (kind == 1 ? *((volatile int *)B.vq) < B.count : *((volatile int *)B.next_lp) < B.count)
                        got = atomicAdd(kind == 1 ? B.vq : B.next_lp, 1);
                }
            }
            *s_lp = got;
            s_res[3] = kind;
        }
        __syncthreads();
        const long long lp = *s_lp;
        if (lp >= B.count) break;
        if (split && s_res[3] == 1) {
            // ---- validation chunk (model.py:263-301): every entry of LP lp's A, streamed once ----
            const double *Av = B.A + (size_t)lp * m * n;
            const size_t total = (size_t)m * n;
            const size_t head = ((reinterpret_cast<size_t>(Av) & 15) != 0) ? 1 : 0;
            bool bad = false;
            if (tid == 0 && head && total) bad |= !isfinite(Av[0]);
            const double2 *A2 = reinterpret_cast<const double2 *>(Av + head);
            const size_t n2 = (total - head) / 2;
            size_t q = tid;
            constexpr int U = NT >= 512 ? 6 : LAZY_SCAN_U;
            for (; q + (U - 1) * NT < n2; q += U * NT) {
                double2 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) v[u] = lazy_scan_load(A2 + q + u * NT);
#pragma unroll
                for (int u = 0; u < U; ++u) bad |= !(isfinite(v[u].x) && isfinite(v[u].y));
            }
            for (; q < n2; q += NT) {
                const double2 v = __ldcs(A2 + q);
                bad |= !(isfinite(v.x) && isfinite(v.y));
            }
            if (tid == 0 && ((total - head) & 1)) bad |= !isfinite(Av[total - 1]);
            if (bad) B.vflag[lp] = 1;
            __syncthreads();   // s_lp / s_res are rewritten by the next claim
            continue;
        }
        const double *Ag = B.shared_Ab ? B.A : B.A + (size_t)lp * m * n;
        const double *bg = B.shared_Ab ? B.b : B.b + (size_t)lp * m;
        const double *cg = B.c + (size_t)lp * n;

        // ---- b: phase 1 needed? (then the dense kernel takes the LP) ----
        bool nonfinite = false, neg = false;
        for (int i = tid; i < m; i += NT) {
            const double bi = bg[i];
            nonfinite |= !isfinite(bi);
            neg |= bi < 0.0;
            rhs[i] = bi;                      // b * (+1)
            basis[i] = n + i;
            lastpiv[i] = 0;
            if (SPX) firstp[i] = -1;
        }
        if (__syncthreads_or(neg)) {
            if (tid == 0) B.defer_list[atomicAdd(B.defer_count, 1)] = (int)lp;
            __syncthreads();
            continue;
        }
        // ---- validate (model.py:263-301): every entry of A, streamed once; b above, c below ----
        // (Measured, not kept: the stream after the solve, so the solve's reads of A are still in
        // L2 when it passes them -- 1.1 GB less DRAM per C5 launch but 5.18 -> 5.36 ms.)
        if (!WS && !B.shared_Ab && !split) {
            const size_t total = (size_t)m * n;
            const size_t head = ((reinterpret_cast<size_t>(Ag) & 15) != 0) ? 1 : 0;   // 16-byte align the body
            if (tid == 0 && head && total) nonfinite |= !isfinite(Ag[0]);
            const double2 *A2 = reinterpret_cast<const double2 *>(Ag + head);
            const size_t n2 = (total - head) / 2;
            size_t q = tid;
            // 16-byte loads in flight per thread (C5, 512 threads: 4 -> 5.43 ms, 6 -> 5.22, 8 -> 5.26)
            constexpr int U = NT >= 512 ? 6 : LAZY_SCAN_U;
            for (; q + (U - 1) * NT < n2; q += U * NT) {
                double2 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) v[u] = lazy_scan_load(A2 + q + u * NT);
#pragma unroll
                for (int u = 0; u < U; ++u) nonfinite |= !(isfinite(v[u].x) && isfinite(v[u].y));
            }
            for (; q < n2; q += NT) {
                const double2 v = __ldcs(A2 + q);
                nonfinite |= !(isfinite(v.x) && isfinite(v.y));
            }
            if (tid == 0 && ((total - head) & 1)) nonfinite |= !isfinite(Ag[total - 1]);
        }
        for (int j = tid; j < nv; j += NT) {
            const double cj = j < n ? cg[j] : 0.0;
            nonfinite |= !isfinite(cj);
            rc[j] = cj;                         // phase 2 runs on c directly (simplex.py:168,180)
            isb[j] = j >= n ? 1 : 0;            // slacks basic
        }
        bool invalid = false;
        if (!WS) invalid = __syncthreads_or(nonfinite);
        else __syncthreads();

        int8_t status = kOptimal;
        int iters = 0;
        double obj = 0.0;
        bool deferred = false;
        int hrows = 0;
        // The LP's replay history is dead once it is solved: its L2 lines are discarded
        // (discard.global.L2: no write-back of the dirty lines, the capacity freed for the
        // live history of the other CTAs).  Only whole 128-byte lines inside this CTA's rows
        // (the neighbouring CTAs' rows share the boundary lines).  BLP_LAZY_DISCARD=0 (launch
        // sets B.lazy_discard) keeps them.
        auto discard_history = [&]() {
            if constexpr (WS) return;
            if (!B.lazy_discard) return;
            const size_t rowb = (size_t)(m + nv) * 8;
            for (int t = 0; t < hrows; ++t) {
                const uintptr_t base = reinterpret_cast<uintptr_t>(Fh + (size_t)t * HS);
                const uintptr_t lo = (base + 127) & ~(uintptr_t)127, hi = (base + rowb) & ~(uintptr_t)127;
                for (uintptr_t a = lo + (uintptr_t)tid * 128; a < hi; a += (uintptr_t)NT * 128)
                    asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
            }
        };
        if (WS && tid >= PT) {
            // scanner warps: A through the bulk-copy ring while the pivot warps solve
            const int stid = tid - PT;
            constexpr int ST = 32 * kLazyScanWarps;
            const size_t total = (size_t)m * n;
            const size_t head = ((reinterpret_cast<size_t>(Ag) & 15) != 0) ? 1 : 0;
            if (stid == 0 && head && total) nonfinite |= !isfinite(Ag[0]);
            const size_t nb = total > head ? (total - head) / 2 * 16 : 0;       // 16-byte body
            const unsigned nch = (unsigned)((nb + kLazyChunk - 1) / kLazyChunk);
            const char *src = reinterpret_cast<const char *>(Ag + head);
            auto issue = [&](unsigned c) {
                const unsigned st = (gseq + c) & (kLazyRing - 1);
                const size_t off = (size_t)c * kLazyChunk;
                const unsigned bytes = (unsigned)(nb - off < (size_t)kLazyChunk ? nb - off : (size_t)kLazyChunk);
                lazy_bulk_load(ring + st * kLazyChunk, src + off, bytes,
                               (unsigned)__cvta_generic_to_shared(fullb + st));
            };
            if (stid == 0)
                for (unsigned c = 0; c < nch && c < (unsigned)kLazyRing; ++c) issue(c);
            for (unsigned c = 0; c < nch; ++c) {
                const unsigned g = gseq + c, st = g & (kLazyRing - 1);
                lazy_mbar_wait((unsigned)__cvta_generic_to_shared(fullb + st), (g / kLazyRing) & 1);
                const size_t off = (size_t)c * kLazyChunk;
                const int len2 = (int)((nb - off < (size_t)kLazyChunk ? nb - off : (size_t)kLazyChunk) / 16);
                const unsigned buf = ring + st * kLazyChunk;
#pragma unroll 4
                for (int q = stid; q < len2; q += ST) {
                    double x0, x1;
                    lds_v2_f64(buf + 16u * q, x0, x1);
                    nonfinite |= !(isfinite(x0) && isfinite(x1));
                }
                lazy_bar(2, ST);                              // stage consumed: refill it
                if (stid == 0 && c + kLazyRing < nch) issue(c + kLazyRing);
            }
            gseq += nch;
            if (stid == 0 && total > head && ((total - head) & 1)) nonfinite |= !isfinite(Ag[total - 1]);
        } else if (!invalid) {
            // initial entering candidates
            {
                unsigned long long ck = kKeyEmptyMax;
                int ci = kNone, cb = kNone;
                for (int j = tid; j < nv; j += PT) {
                    if (isb[j]) continue;
                    const unsigned long long k = key_max(rc[j]);
                    if (k > ck || (k == ck && j < ci)) { ck = k; ci = j; }
                    if (rc[j] > kTol && j < cb) cb = j;
                }
                const unsigned long long kw = warp_max_key(ck);
                const int iw = warp_index_of(ck, kw, ci);
                const int bw = warp_min_int(cb);
                if (lane == 0) { P->ckey[warp] = kw; P->cidx[warp] = iw; P->cbl[warp] = bw; }
            }
            pbar();
            int degenerate_run = 0;
            bool use_bland = false;
            int prev_l = -1, prev_e = -1, prev_old = -1;
            bool prev_new = false;                    // SPX: prev_l was pivoted on for the first time
            double prev_rr = 0.0;
            // _run_phase (simplex.py:63-91)
            for (int k = 0;; ++k) {                   // pivot number k+1; history slot k
                // previous pivot's bookkeeping (after the barrier that ended it)
                if (prev_l >= 0) {
                    if (tid == 0) {
                        basis[prev_l] = prev_e; isb[prev_old] = 0; isb[prev_e] = 1;
                        if (SPX) {
                            urow[k - 1] = prev_new ? prev_l : -1;
                            if (prev_new) firstp[prev_l] = k - 1;
                        }
                    }
                    if (tid == (prev_l % PT)) { lastpiv[prev_l] = k; rhs[prev_l] = prev_rr; }
                }
                if (k == max_iter) { status = kIterationLimit; iters = max_iter; break; }
                // choose_entering[_bland] from the warp partials
                int e;
                {
                    unsigned long long kk = lane < NW ? P->ckey[lane] : kKeyEmptyMax;
                    const int ii = lane < NW ? P->cidx[lane] : kNone, bb = lane < NW ? P->cbl[lane] : kNone;
                    const unsigned long long kw = warp_max_key(kk);
                    const int ew = warp_index_of(kk, kw, ii);
                    const int bw = warp_min_int(bb);
                    if (use_bland) e = bw == kNone ? -1 : bw;
                    else e = (ew == kNone || kw <= kTolK) ? -1 : ew;
                }
                if (e < 0) { iters = k; break; }   // optimal
                if (k == kLazyMaxPivots) { deferred = true; break; }
                hrows = k + 1;                       // history rows 0..k may hold this LP's data
                const double rce = rc[e];
                // entering column by replay (f_i = a_ie before this pivot); ratio test
                unsigned long long lk = kKeyEmptyMin;
                int li = kNone;
                if constexpr (RP == 1) {
                    for (int t = lane; t < k; t += 32) hw[t] = lazy_h(Rh + (size_t)t * HS + e);   // r^t_e
                    __syncwarp();
                }
                // SPX: the entering slack's first-pivot slot (prev_l's entry is written by tid 0
                // at the top of this pivot, so it comes from the registers)
                int ue = -1;
                if (SPX && e >= n) ue = (e - n == prev_l && prev_new) ? k - 1 : firstp[e - n];
                for (int i = tid; i < m; i += PT) {
                    const int t0 = lastpiv[i];
                    double a;
                    if constexpr (RP == 1) {
                        a = t0 ? hw[t0 - 1] : lazy_a0(Ag, n, i, e);
                        a = lazy_replay(a, Fh + i, (int)HS, hw, t0, k);
                    } else {
                        a = t0 ? RgetS(t0 - 1, e, ue) : lazy_a0(Ag, n, i, e);
                        for (int t = t0; t < k; ++t)
                            a = __dsub_rn(a, __dmul_rn(Fget(t, i), RgetS(t, e, ue)));
                    }
                    fcur[i] = a;
                    if (FS && k < KF) Fs[(size_t)k * m + i] = a;
                    else lazy_hs(Fh + (size_t)k * HS + i, a);
                    const unsigned long long key = key_min(ratio_entry(rhs[i], a));
                    if (key < lk) { lk = key; li = i; }     // rows ascend per thread
                }
                {
                    const unsigned long long kw = warp_min_key(lk);
                    const int lw = warp_index_of(lk, kw, li);
                    if (lane == 0) { P->lkey[warp] = kw; P->lrow[warp] = lw; }
                }
                pbar();  // S1
                unsigned long long kmin;
                int l;
                {
                    const unsigned long long kk = lane < NW ? P->lkey[lane] : kKeyEmptyMin;
                    const int rr = lane < NW ? P->lrow[lane] : kNone;
                    kmin = warp_min_key(kk);
                    l = warp_index_of(kk, kmin, rr);
                }
                if (l == kNone || kmin >= kSent) { status = kUnbounded; iters = k; break; }
                if (kmin != 0ull && kmin <= kDeg) {                 // simplex.py:84-90
                    ++degenerate_run;
                    if (B.lim.anti_cycling && degenerate_run >= trigger) use_bland = true;
                } else {
                    degenerate_run = 0;
                    use_bland = false;
                }
                const double pe = fcur[l];
                const double rrhs = div_entry(rhs[l], pe);
                const int oldvar = basis[l];
                const int t0l = lastpiv[l];
                // pivot row by replay, divided by pe; objective row; next candidates
                unsigned long long ck = kKeyEmptyMax;
                int ci = kNone, cb = kNone;
                double *Rk = (FS == 2 && k < KF) ? Rs + (size_t)k * nv : Rh + (size_t)k * HS;
                if constexpr (RP == 1) {
                    __syncwarp();
                    for (int t = t0l + lane; t < k; t += 32) hw[t] = Fget(t, l);   // f^t_l
                    __syncwarp();
                }
                // SPX: structural columns, then the slack columns of rows pivoted on so far (slot u:
                // row urow[u]; slot k is this pivot's row if it is new), stored at n + u
                const int fl = SPX ? firstp[l] : 0;
                const bool lnew = SPX && fl < 0;
                const int jend = SPX ? n + k + 1 : nv;
                for (int jj = tid; jj < jend; jj += PT) {
                    int j = jj, u = -1;
                    if (SPX && jj >= n) {
                        u = jj - n;
                        const int row = u == k ? (lnew ? l : -1) : urow[u];
                        if (row < 0) continue;
                        j = n + row;
                    }
                    double a = t0l ? RgetS(t0l - 1, j, u) : lazy_a0(Ag, n, l, j);
                    if constexpr (RP == 1) {
                        a = lazy_replay(a, Rh + j, (int)HS, hw, t0l, k);
                    } else {
                        for (int t = t0l; t < k; ++t)
                            a = __dsub_rn(a, __dmul_rn(Fget(t, l), RgetS(t, j, u)));
                    }
                    const double r = div_entry(a, pe);
                    if (FS == 2 && k < KF) Rk[jj] = r;
                    else lazy_hs(Rk + jj, r);
                    const double v = __dsub_rn(rc[j], __dmul_rn(rce, r));
                    rc[j] = v;
                    if (!((j == e) || (j != oldvar && isb[j]))) {
                        const unsigned long long kv = key_max(v);
                        if (kv > ck || (kv == ck && j < ci)) { ck = kv; ci = j; }
                        if (v > kTol && j < cb) cb = j;
                    }
                }
                {
                    const unsigned long long kw = warp_max_key(ck);
                    const int iw = warp_index_of(ck, kw, ci);
                    const int bw = warp_min_int(cb);
                    if (lane == 0) { P->ckey[warp] = kw; P->cidx[warp] = iw; P->cbl[warp] = bw; }
                }
                // rhs[l] is read by every thread above (rrhs); its owner writes it after S3
                for (int i = tid; i < m; i += PT)
                    if (i != l) rhs[i] = __dsub_rn(rhs[i], __dmul_rn(fcur[i], rrhs));
                obj = __dadd_rn(obj, __dmul_rn(rce, rrhs));          // tableau.py:242
                prev_l = l; prev_e = e; prev_old = oldvar; prev_rr = rrhs; prev_new = lnew;
                pbar();  // S3
            }
            pbar();
            if (prev_l >= 0 && tid == 0) { basis[prev_l] = prev_e; }
            pbar();
        }
        (void)obj;
        if constexpr (WS) {
            if (tid == 0) { s_res[0] = status; s_res[1] = iters; s_res[2] = deferred; }
            invalid = __syncthreads_or(nonfinite);           // the stream's verdict joins the solve
            status = invalid ? (int8_t)kInvalid : (int8_t)s_res[0];
            iters = invalid ? 0 : s_res[1];
            deferred = !invalid && s_res[2];
        } else if (invalid) {
            status = kInvalid;
        }
        if (deferred) {
            if (tid == 0) B.defer_list[atomicAdd(B.defer_count, 1)] = (int)lp;
            __syncthreads();
            discard_history();
            continue;
        }
        // ---- _extract_point (simplex.py:146-151) and c @ x ----
        double *xs = rc;                         // n <= nv doubles, free after the solve
        double *xg = B.x + (size_t)lp * n;
        for (int j = tid; j < n; j += NT) xs[j] = 0.0;
        __syncthreads();
        if (status == kOptimal)
            for (int i = tid; i < m; i += NT)
                if (basis[i] < n) xs[basis[i]] = rhs[i];
        __syncthreads();
        // c @ x left to right (the oracle's order): a near-zero optimum is a sum of cancelling
        // terms whose rounding depends on the order (fuzz: condition numbers up to 1e15 at
        // x ~ 1), so any other order can miss 1e-9 relative.  The products are formed in
        // parallel (each rounded on its own, as in the sequential loop), the sum by one thread
        // from shared memory; zero products are skipped (s + 0 == s).
        for (int j = tid; j < n; j += NT) {
            const double xj = xs[j];
            xg[j] = xj;
            xs[j] = __dmul_rn(cg[j], xj);
        }
        __syncthreads();
        if (warp == 0) {
            double s = 0.0;
            if (status == kOptimal && lane == 0)
                for (int j = 0; j < n; ++j) {
                    const double p = xs[j];
                    if (p != 0.0) s = __dadd_rn(s, p);
                }
            if (lane == 0) {
                B.objective[lp] = status == kOptimal ? s : __longlong_as_double(0x7ff8000000000000LL);
                B.status[lp] = status;
                B.it1[lp] = 0;
                B.it2[lp] = iters;
            }
        }
        __syncthreads();
        discard_history();
    }
}

// Finiteness of every entry of A (model.py:263-301), streamed once with
// 16-byte loads; flag[lp] = 1 for an LP holding a non-finite entry.  A shared
// polytope (support mode) is scanned once and flags every LP.
__global__ void __launch_bounds__(256)
lazy_validate_kernel(const double *A, long long count, long long per_lp, int shared_Ab, unsigned char *flag) {
    const long long total = shared_Ab ? per_lp : count * per_lp;
    auto mark = [&](long long e) {
        if (shared_Ab) { for (long long k = 0; k < count; ++k) flag[k] = 1; }
        else flag[e / per_lp] = 1;
    };
    // A caller's device pointer may be only 8-byte aligned (a torch view A_all[k] with odd
    // m*n): one scalar head element, then 16-byte loads, then an odd tail element.
    const long long head = (total > 0 && (reinterpret_cast<uintptr_t>(A) & 15)) ? 1 : 0;
    const long long n2 = (total - head) / 2;
    const double2 *A2 = reinterpret_cast<const double2 *>(A + head);
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n2; q += stride) {
        const double2 v = __ldcs(A2 + q);
        if (!isfinite(v.x)) mark(head + 2 * q);
        if (!isfinite(v.y)) mark(head + 2 * q + 1);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (head && !isfinite(A[0])) mark(0);
        if (((total - head) & 1) && !isfinite(A[total - 1])) mark(total - 1);
    }
}

// Outputs of the LPs lazy_validate_kernel flagged: BLP_STATUS_INVALID, as the
// dense kernels report them (the host then raises validate()'s ValueError).
__global__ void lazy_finalize_kernel(const unsigned char *flag, Batch B) {
    for (long long lp = (long long)blockIdx.x * blockDim.x + threadIdx.x; lp < B.count;
         lp += (long long)gridDim.x * blockDim.x) {
        if (!flag[lp]) continue;
        B.status[lp] = kInvalid;
        B.objective[lp] = __longlong_as_double(0x7ff8000000000000LL);
        B.it1[lp] = 0;
        B.it2[lp] = 0;
        for (int j = 0; j < B.n; ++j) B.x[(size_t)lp * B.n + j] = 0.0;
    }
}

}  // namespace blp
