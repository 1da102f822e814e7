// blp_warplp3_kernel.cuh -- one warp per LP with the second half of every
// row in TENSOR MEMORY (m <= 32 rows, n + m + 1 <= R + T columns; C2).
//
// warplp2 (blp_warplp2_kernel.cuh) keeps positions [R, R+S) of each row in a
// shared-memory tile, and that tile is its bottleneck: the rank-1 update of
// the tile half is one LDS + one STS per cell, and the SM's shared-memory pipe
// runs at ~80% (profiles/r01_c2_warplp2_full.txt).  B200's tensor memory
// (TMEM, 256 KB per SM, 128 lanes x 512 32-bit columns) is private to the
// CTA that allocates it and lane-addressed: warp w of a CTA reads and writes
// lanes 32(w%4) .. 32(w%4)+31 with tcgen05.ld / tcgen05.st, each thread its
// own lane -- exactly the lane-owns-a-row layout of this kernel.  Measured on
// B200 (scripts/tmem_probe.cu): 395 B/clk/SM of 32x32b.x16 loads, and a
// load-update-store loop is FP64-bound at 244 B/clk/SM read + the same
// written, versus 128 B/clk/SM for shared memory.
//
// So a CTA is 4 warps = 4 independent LPs, one per TMEM lane quarter; warp 0
// allocates 2T (rounded to a power of two) TMEM columns for the CTA, and the
// warp of quarter q keeps row r's positions [R, R+T) as doubles in lane
// 32q + r, columns 2(p-R), 2(p-R)+1.  Positions [0, R) stay in registers.
// The pivot row is shared through shared memory (lane l stores its whole row
// once; lane q divides positions q, q+32), the update streams the TMEM half
// in chunks of 8 doubles (tcgen05.ld x16 -> wait -> 8 x (DMUL, DSUB) ->
// tcgen05.st x16).  Everything else is warplp2's algorithm, so results are
// identical to it and to the reference.
#pragma once

#include <cstdint>

#include "blp_common.cuh"
#include "blp_keys.cuh"
#include "blp_warplp_kernel.cuh"

namespace blp {

// ---- tensor memory (tcgen05) ------------------------------------------------
__device__ __forceinline__ void tm_ld16(uint32_t a, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(a));
}
__device__ __forceinline__ void tm_st16(uint32_t a, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
          "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tm_ld2(uint32_t a, uint32_t &x, uint32_t &y) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ double tm_f64(uint32_t lo, uint32_t hi) { return __hiloint2double((int)hi, (int)lo); }

template <int R, int T>
struct Wl3Cfg {
    static_assert(T % 8 == 0 && T >= 8, "TMEM half in chunks of 8 doubles");
    static constexpr int CPW = R + T;
    static constexpr int OPW = (CPW + 31) / 32;
    static constexpr int WARPS = 4;                                  // one LP per TMEM lane quarter
    static constexpr int TCOLS = 2 * T <= 32 ? 32 : (2 * T <= 64 ? 64 : (2 * T <= 128 ? 128 : 256));
    // per-warp shared memory
    static constexpr size_t ROWBUF = 0;                              // CPW doubles: the shared pivot row
    static constexpr size_t RVEC = ROWBUF + (size_t)((CPW + 1) & ~1) * 8;   // CPW doubles: r
    static constexpr size_t CBV = RVEC + (size_t)((CPW + 1) & ~1) * 8;
    static constexpr size_t WBYTES = CBV + 32 * 8;
    static constexpr size_t BYTES = WARPS * WBYTES + 16;            // + the TMEM base address
};

template <int R, int T>
struct Wl3State {
    static constexpr int OPW = Wl3Cfg<R, T>::OPW;
    double a[R];            // positions [0, R) of row `lane` (rhs at 0)
    double rc[OPW];         // transposed objective row; position 0 holds the objective value
    double arc[OPW];        // phase-1 reduced cost of the artificial paired with a slack position
    int artk[OPW];
    unsigned bas;           // bit t: position's variable basic; bit 16+t: paired artificial basic
    int basis_r, art_of_r;
    unsigned long long ckey;
    int cidx, cbl;
};

template <int R, int T, int KIND>
__device__ __forceinline__ void wl3_candidates(const WlpDims &D, Wl3State<R, T> &St) {
    unsigned long long ck = kKeyEmptyMax;
    int ci = kNone, cb = kNone;
#pragma unroll
    for (int t = 0; t < Wl3State<R, T>::OPW; ++t) {
        const int pos = D.lane + 32 * t;
        if (pos >= 1 && pos < D.ncols) {
            const int j = pos - 1;
            if (!(St.bas & (1u << t))) {
                const unsigned long long k = key_max(St.rc[t]);
                if (k > ck || (k == ck && j < ci)) { ck = k; ci = j; }
                if (St.rc[t] > kTol && j < cb) cb = j;
            }
            if (KIND == kWlpPhase1 && St.artk[t] >= 0 && !(St.bas & (0x10000u << t))) {
                const int ja = D.nvc + St.artk[t];
                const unsigned long long k = key_max(St.arc[t]);
                if (k > ck || (k == ck && ja < ci)) { ck = k; ci = ja; }
                if (St.arc[t] > kTol && ja < cb) cb = ja;
            }
        }
    }
    St.ckey = warp_max_key(ck);
    St.cidx = warp_index_of(ck, St.ckey, ci);
    St.cbl = (int)__reduce_min_sync(kFull, (unsigned)cb);
}

// Entry of this lane's row at a warp-uniform position (TMEM half: one x2 load).
template <int R, int T>
__device__ __forceinline__ double wl3_at(const Wl3State<R, T> &St, uint32_t tb, int pos) {
    if (pos < R) return reg_pick<R>(St.a, pos);
    uint32_t lo, hi;
    tm_ld2(tb + 2u * (uint32_t)(pos - R), lo, hi);
    tm_wait_ld();
    return tm_f64(lo, hi);
}

// Row `row` into rowbuf (all R + T positions): the lane holding it stores, the
// whole warp takes part in the (warp-collective) TMEM loads.
template <int R, int T>
__device__ __forceinline__ void wl3_share_row(const WlpDims &D, const Wl3State<R, T> &St, unsigned char *wsm,
                                              uint32_t tb, int row) {
    const unsigned rb = (unsigned)__cvta_generic_to_shared(wsm + Wl3Cfg<R, T>::ROWBUF);
    const bool mine = D.lane == row;
    __syncwarp();
#pragma unroll
    for (int c = 0; c < R; c += 2) st_shared_v2_if(mine, rb + 8u * c, St.a[c], St.a[c + 1]);
#pragma unroll
    for (int k = 0; k < T / 8; ++k) {
        uint32_t v[16];
        tm_ld16(tb + 16u * k, v);
        tm_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; i += 2)
            st_shared_v2_if(mine, rb + 8u * (R + 8 * k + i), tm_f64(v[2 * i], v[2 * i + 1]),
                            tm_f64(v[2 * i + 2], v[2 * i + 3]));
    }
    __syncwarp();
}

// pivot (tableau.py:218-244): av = this lane's entry of the entering column,
// l = leaving row, fm = reduced cost of the entering column.
template <int R, int T, int KIND>
__device__ __forceinline__ void wl3_pivot(const WlpDims &D, Wl3State<R, T> &St, unsigned char *wsm, uint32_t tb,
                                          int e, int l, double av, double fm, int oldvar) {
    using C = Wl3Cfg<R, T>;
    const double *rowbuf = reinterpret_cast<const double *>(wsm + C::ROWBUF);
    double *rvec = reinterpret_cast<double *>(wsm + C::RVEC);
    const unsigned rv = (unsigned)__cvta_generic_to_shared(rvec);
    const double pe = __shfl_sync(kFull, av, l);
    const bool mine = D.lane == l;
    wl3_share_row<R, T>(D, St, wsm, tb, l);
    if (mine) St.basis_r = e;
#pragma unroll
    for (int t = 0; t < Wl3State<R, T>::OPW; ++t) {
        const int pos = D.lane + 32 * t;
        if (pos < D.ncols) {
            const double r = div_entry(rowbuf[pos], pe);
            rvec[pos] = r;
            if (pos == 0) {
                St.rc[t] = __dadd_rn(St.rc[t], __dmul_rn(fm, r));   // tableau.py:242
            } else {
                St.rc[t] = __dsub_rn(St.rc[t], __dmul_rn(fm, r));
                const int j = pos - 1;
                if (j == e) St.bas |= (1u << t);
                if (j == oldvar) St.bas &= ~(1u << t);
                if (KIND == kWlpPhase1 && St.artk[t] >= 0) {
                    St.arc[t] = __dsub_rn(St.arc[t], __dmul_rn(fm, -r));
                    const int ja = D.nvc + St.artk[t];
                    if (ja == e) St.bas |= (0x10000u << t);
                    if (ja == oldvar) St.bas &= ~(0x10000u << t);
                }
            }
        }
    }
    if (KIND != kWlpRestore) wl3_candidates<R, T, KIND>(D, St);
    __syncwarp();
    // TMEM half: chunks of 8 doubles; row l takes r (numpy: r - 0*r == r)
#pragma unroll
    for (int k = 0; k < T / 8; ++k) {
        uint32_t v[16];
        tm_ld16(tb + 16u * k, v);
        double r[8];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
            const double2 r2 = reinterpret_cast<const double2 *>(rvec + R + 8 * k)[i / 2];
            r[i] = r2.x;
            r[i + 1] = r2.y;
        }
        tm_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double t = tm_f64(v[2 * i], v[2 * i + 1]);
            const double u = mine ? r[i] : __dsub_rn(t, __dmul_rn(av, r[i]));
            v[2 * i] = (uint32_t)__double2loint(u);
            v[2 * i + 1] = (uint32_t)__double2hiint(u);
        }
        tm_st16(tb + 16u * k, v);
    }
#pragma unroll
    for (int c = 0; c < R; c += 2) {
        const double2 r2 = reinterpret_cast<const double2 *>(rvec)[c / 2];
        St.a[c] = __dsub_rn(St.a[c], __dmul_rn(av, r2.x));
        St.a[c + 1] = __dsub_rn(St.a[c + 1], __dmul_rn(av, r2.y));
    }
#pragma unroll
    for (int c = 0; c < R; c += 2) ld_shared_v2_if(mine, rv + 8u * c, St.a[c], St.a[c + 1]);
    tm_wait_st();
    __syncwarp();
}

// _run_phase (simplex.py:63-91); entering candidates already in St.
template <int R, int T, int KIND>
__device__ __forceinline__ WlpPhase wl3_run_phase(const WlpDims &D, Wl3State<R, T> &St, unsigned char *wsm,
                                                  uint32_t tb, const Limits &lim) {
    const int max_iter = lim.max_iterations > 0 ? lim.max_iterations : 50 * (D.m + D.n);
    const int trigger = lim.degenerate_limit >= 0 ? lim.degenerate_limit : (D.m > 1 ? D.m : 1);
    const unsigned long long kSent = key_max(kSentinel), kDeg = key_max(kDegenerateTol), kTolK = key_max(kTol);
    int degenerate_run = 0;
    bool use_bland = false;
    for (int it = 0;; ++it) {
        if (it == max_iter) return {2, max_iter};
        int e;
        if (use_bland) e = St.cbl == kNone ? -1 : St.cbl;                // choose_entering_bland
        else e = (St.cidx == kNone || St.ckey <= kTolK) ? -1 : St.cidx;    // choose_entering
        if (e < 0) return {0, it};
        const bool art_e = e >= D.nvc;
        const int epos = art_e ? 1 + D.n + wlp_row_of_art(St.art_of_r, e - D.nvc) : e + 1;
        double av = wl3_at<R, T>(St, tb, epos);
        if (art_e) av = -av;
        unsigned long long lk = kKeyEmptyMin;                               // choose_leaving
        const double ratio = ratio_entry(St.a[0], av);
        if (D.lane < D.m) lk = key_min(ratio);
        const unsigned long long kmin = warp_min_key(lk);
        const int l = warp_index_of(lk, kmin, D.lane);
        if (l == kNone || kmin >= kSent) return {1, it};   // unbounded (a NaN ratio keys to 0)
        double myfm = 0.0;
#pragma unroll
        for (int t = 0; t < Wl3State<R, T>::OPW; ++t)
            myfm = selp_f64(art_e ? St.arc[t] : St.rc[t], myfm, t == (epos >> 5));
        const double fm = __shfl_sync(kFull, myfm, epos & 31);
        const int oldvar = __shfl_sync(kFull, St.basis_r, l);
        if (kmin != 0ull && kmin <= kDeg) {                 // simplex.py:84-90
            ++degenerate_run;
            if (lim.anti_cycling && degenerate_run >= trigger) use_bland = true;
        } else {
            degenerate_run = 0;
            use_bland = false;
        }
        wl3_pivot<R, T, KIND>(D, St, wsm, tb, e, l, D.lane < D.m ? av : 0.0, fm, oldvar);
    }
}

// _price_out (simplex.py:133-143), transposed: lane q rebuilds the reduced
// costs of positions q, q+32, rows in reference order, skipping cb == 0 rows.
template <int R, int T, int PHASE>
__device__ __forceinline__ void wl3_price_out(const WlpDims &D, Wl3State<R, T> &St, unsigned char *wsm, uint32_t tb,
                                              const double *cg) {
    using C = Wl3Cfg<R, T>;
    double *cbv = reinterpret_cast<double *>(wsm + C::CBV);
    const double *rowbuf = reinterpret_cast<const double *>(wsm + C::ROWBUF);
    cbv[D.lane] = D.lane < D.m ? (PHASE == 1 ? (St.basis_r >= D.nvc ? -1.0 : 0.0)
                                             : (St.basis_r < D.n ? cg[St.basis_r] : 0.0))
                               : 0.0;
    double rc[Wl3State<R, T>::OPW], ac[Wl3State<R, T>::OPW];
#pragma unroll
    for (int t = 0; t < Wl3State<R, T>::OPW; ++t) {
        const int pos = D.lane + 32 * t, j = pos - 1;
        rc[t] = (PHASE == 2 && pos >= 1 && j < D.n) ? cg[j] : 0.0;
        ac[t] = -1.0;
    }
    __syncwarp();
    for (int r = 0; r < D.m; ++r) {
        const double cb = cbv[r];
        if (cb == 0.0) continue;          // uniform: every lane reads the same cbv[r]
        wl3_share_row<R, T>(D, St, wsm, tb, r);
#pragma unroll
        for (int t = 0; t < Wl3State<R, T>::OPW; ++t) {
            const int pos = D.lane + 32 * t;
            if (pos < D.ncols) {
                const double v = rowbuf[pos];
                if (pos == 0) {
                    rc[t] = __dadd_rn(rc[t], __dmul_rn(cb, v));
                } else {
                    rc[t] = __dsub_rn(rc[t], __dmul_rn(cb, v));
                    if (PHASE == 1 && St.artk[t] >= 0) ac[t] = __dsub_rn(ac[t], __dmul_rn(cb, -v));
                }
            }
        }
    }
#pragma unroll
    for (int t = 0; t < Wl3State<R, T>::OPW; ++t) {
        const int pos = D.lane + 32 * t;
        if (pos < D.ncols) {
            St.rc[t] = rc[t];
            if (PHASE == 1 && St.artk[t] >= 0) St.arc[t] = ac[t];
        }
    }
    wl3_candidates<R, T, PHASE == 1 ? kWlpPhase1 : kWlpPhase2>(D, St);
}

// restore_objective pivot-outs (simplex.py:109-126), uncounted.
template <int R, int T>
__device__ __forceinline__ void wl3_restore(const WlpDims &D, Wl3State<R, T> &St, unsigned char *wsm, uint32_t tb) {
    const double *rowbuf = reinterpret_cast<const double *>(wsm + Wl3Cfg<R, T>::ROWBUF);
    const unsigned long long kRed = key_max(kRedundantTol);
    for (int row = 0; row < D.m; ++row) {
        if (__shfl_sync(kFull, St.basis_r, row) < D.nvc) continue;
        wl3_share_row<R, T>(D, St, wsm, tb, row);
        unsigned long long bk = kKeyEmptyMax;
        int bj = kNone;
#pragma unroll
        for (int t = 0; t < Wl3State<R, T>::OPW; ++t) {
            const int pos = D.lane + 32 * t;
            if (pos >= 1 && pos < D.ncols) {
                const unsigned long long k = key_max(fabs(rowbuf[pos]));
                if (k > bk) { bk = k; bj = pos - 1; }     // positions ascend per lane
            }
        }
        const unsigned long long kb = warp_max_key(bk);
        const int j = warp_index_of(bk, kb, bj);
        // entries[j] > REDUNDANT_ROW_TOL; a NaN entry compares False in numpy
        if (j != kNone && kb > kRed && kb != ~0ull) {
            const double av = wl3_at<R, T>(St, tb, j + 1);
            const int oldvar = __shfl_sync(kFull, St.basis_r, row);
            wl3_pivot<R, T, kWlpRestore>(D, St, wsm, tb, j, row, D.lane < D.m ? av : 0.0, 0.0, oldvar);
        }
    }
}

template <int R, int T, int kMinBlocks>
__global__ void __launch_bounds__(32 * Wl3Cfg<R, T>::WARPS, kMinBlocks)
warplp3_kernel(Batch B) {
    using C = Wl3Cfg<R, T>;
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5;
    uint32_t *tbase = reinterpret_cast<uint32_t *>(smem + C::WARPS * C::WBYTES);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"((unsigned)__cvta_generic_to_shared(tbase)), "n"(C::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = *tbase + ((uint32_t)(32 * (warp & 3)) << 16);   // this warp's lane quarter
    unsigned char *wsm = smem + warp * C::WBYTES;

    WlpDims D;
    D.m = B.m; D.n = B.n; D.nvc = B.n + B.m; D.ncols = B.n + B.m + 1; D.lane = threadIdx.x & 31;
    const int m = D.m, n = D.n, nvc = D.nvc;
    {
        double *rvec = reinterpret_cast<double *>(wsm + C::RVEC);
        for (int q = D.lane; q < C::CPW; q += 32) rvec[q] = 0.0;
    }
    Wl3State<R, T> St;
    long long lp = 0;
    if (D.lane == 0) lp = atomicAdd(B.next_lp, 1);
    lp = __shfl_sync(kFull, lp, 0);
    for (;;) {
        if (lp >= B.count) break;
        long long nxt = 0;                 // claim the next LP and warm L2 with its inputs
        if (D.lane == 0) nxt = atomicAdd(B.next_lp, 1);
        nxt = __shfl_sync(kFull, nxt, 0);
        if (nxt < B.count) prefetch_lp_inputs(B, nxt, D.lane);
        const double *Ag = B.shared_Ab ? B.A : B.A + (size_t)lp * m * n;
        const double *bg = B.shared_Ab ? B.b : B.b + (size_t)lp * m;
        const double *cg = B.c + (size_t)lp * n;

        // ---- build_tableau (tableau.py:139-172): lane r loads row r; validation fused ----
        const bool live = D.lane < m;
        const double bi = live ? bg[D.lane] : 0.0;
        bool nonfinite = !isfinite(bi);
        const bool neg = live && bi < 0.0;
        const unsigned negmask = __ballot_sync(kFull, neg);
        const int n_art = __popc(negmask);
        const double sgn = neg ? -1.0 : 1.0;
        St.art_of_r = neg ? __popc(negmask & ((1u << D.lane) - 1u)) : -1;
        St.basis_r = neg ? nvc + St.art_of_r : n + D.lane;
        const double *arow = Ag + (size_t)(live ? D.lane : 0) * n;
#pragma unroll
        for (int p = 0; p < R; ++p) {
            const int j = p - 1;
            double v = 0.0;
            if (live) {
                if (p == 0) v = __dmul_rn(bi, sgn);
                else if (j < n) { const double a = arow[j]; nonfinite |= !isfinite(a); v = __dmul_rn(a, sgn); }
                else if (j < nvc) v = (j - n == D.lane) ? sgn : 0.0;
            }
            St.a[p] = v;
        }
#pragma unroll
        for (int k = 0; k < T / 8; ++k) {
            uint32_t v[16];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int j = R + 8 * k + i - 1;
                double x = 0.0;
                if (live) {
                    if (j < n) { const double a = arow[j]; nonfinite |= !isfinite(a); x = __dmul_rn(a, sgn); }
                    else if (j < nvc) x = (j - n == D.lane) ? sgn : 0.0;
                }
                v[2 * i] = (uint32_t)__double2loint(x);
                v[2 * i + 1] = (uint32_t)__double2hiint(x);
            }
            tm_st16(tb + 16u * k, v);
        }
        for (int j = D.lane; j < n; j += 32) nonfinite |= !isfinite(cg[j]);
        const bool invalid = __any_sync(kFull, nonfinite);
        St.bas = 0;
#pragma unroll
        for (int t = 0; t < C::OPW; ++t) {
            const int pos = D.lane + 32 * t;
            const int j = pos - 1;
            St.rc[t] = (pos >= 1 && j < n) ? cg[j] : 0.0;
            St.arc[t] = 0.0;
            const int row = j - n;   // slack position of row `row`
            const int k = __shfl_sync(kFull, St.art_of_r, row & 31);
            St.artk[t] = (j >= n && j < nvc) ? k : -1;
            if (j >= n && j < nvc) St.bas |= (k < 0) ? (1u << t) : (0x10000u << t);
        }
        tm_wait_st();
        __syncwarp();

        int8_t status = kOptimal;
        int it1 = 0, it2 = 0;
        bool done = false;
        if (invalid) {
            status = kInvalid;
            done = true;
        } else if (n_art > 0) {
            wl3_price_out<R, T, 1>(D, St, wsm, tb, cg);                     // build_auxiliary
            const WlpPhase p1 = wl3_run_phase<R, T, kWlpPhase1>(D, St, wsm, tb, B.lim);
            it1 = p1.iters;
            const double obj = __shfl_sync(kFull, St.rc[0], 0);
            if (p1.state == 2) { status = kIterationLimit; done = true; }
            else if (p1.state == 1) { status = kErrPhase1Unbounded; done = true; }
            else if (fabs(obj) > kPhase1ZeroTol) { status = kInfeasible; done = true; }
            else {
                wl3_restore<R, T>(D, St, wsm, tb);
                wl3_price_out<R, T, 2>(D, St, wsm, tb, cg);
            }
        } else {
            wl3_candidates<R, T, kWlpPhase2>(D, St);
        }
        if (!done) {
            const WlpPhase p2 = wl3_run_phase<R, T, kWlpPhase2>(D, St, wsm, tb, B.lim);
            it2 = p2.iters;
            if (p2.state == 2) status = kIterationLimit;
            else if (p2.state == 1) status = kUnbounded;
        }

        // ---- _extract_point (simplex.py:146-151) and c @ x ----
        double *xs = reinterpret_cast<double *>(wsm + C::RVEC);   // n <= CPW doubles of scratch
        __syncwarp();
        for (int j = D.lane; j < n; j += 32) xs[j] = 0.0;
        __syncwarp();
        if (status == kOptimal && live && St.basis_r < n) xs[St.basis_r] = St.a[0];
        __syncwarp();
        double *xg = B.x + (size_t)lp * n;
        for (int j = D.lane; j < n; j += 32) xg[j] = xs[j];
        if (D.lane == 0) {
            double obj = __longlong_as_double(0x7ff8000000000000LL);
            if (status == kOptimal) {
                obj = 0.0;
                for (int j = 0; j < n; ++j) obj = __dadd_rn(obj, __dmul_rn(cg[j], xs[j]));
            }
            B.objective[lp] = obj;
            B.status[lp] = status;
            B.it1[lp] = it1;
            B.it2[lp] = it2;
        }
        __syncwarp();
        for (int q = D.lane; q < C::CPW; q += 32) xs[q] = 0.0;   // rvec padding must read as 0
        __syncwarp();
        lp = nxt;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tbase), "n"(C::TCOLS));
}

}  // namespace blp
