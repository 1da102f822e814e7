// blp_warplp_kernel.cuh -- one WARP per LP, whole tableau in registers
// (m <= 32 constraint rows, n + m + 1 <= CPW columns: the C1 / C2 shapes).
//
// Each CTA is a single warp that pulls LP indices from the batch queue.
// Lane r holds constraint row r of the compact tableau (rhs at position 0,
// variable j at position j+1; tableau.py:56-79 minus the artificial columns)
// in CPW registers; the objective row is transposed (lane q holds the reduced
// cost of positions q, q+32); the basis, the artificial bookkeeping and the
// entering/leaving candidates are lane registers too.  Shared memory is used
// only to turn the pivot row around (row -> per-column divisions -> broadcast)
// and, once per phase, as the staging area of the tableau build and price-out.
// No CTA barrier exists in the pivot loop: everything is warp-synchronous.
//
// Numerics follow blp_tableau_kernel.cuh / the reference exactly (separately
// rounded __dmul_rn/__dsub_rn, IEEE __ddiv_rn, numpy arg-reduction order via
// the keys of blp_keys.cuh).  The new pivot row is r_j itself, reloaded by
// its lane, value-equal to numpy's r_j - 0 * r_j for every finite r_j.
#pragma once

#include "blp_common.cuh"
#include "blp_keys.cuh"

namespace blp {

template <int CPW>
struct WlpCfg {
    static constexpr int OPW = (CPW + 31) / 32;
    static constexpr int LDG = CPW + 1;            // odd stage row stride: conflict-free transposes
    static constexpr size_t ROWBUF = 0;            // CPW doubles
    static constexpr size_t RVEC = ROWBUF + CPW * 8;
    static constexpr size_t CBV = RVEC + CPW * 8;  // 32 doubles
    static constexpr size_t STAGE = CBV + 32 * 8;  // m * LDG doubles
    static size_t __host__ __device__ bytes(int m) { return STAGE + (size_t)(m > 0 ? m : 1) * LDG * 8; }
};

enum { kWlpRestore = 0, kWlpPhase1 = 1, kWlpPhase2 = 2 };

template <int CPW>
struct WlpState {
    static constexpr int OPW = (CPW + 31) / 32;
    double a[CPW];          // constraint row `lane` (zero for lanes >= m)
    double rc[OPW];         // transposed objective row; position 0 holds the objective value
    double arc[OPW];        // phase-1 reduced cost of the artificial paired with a slack position
    int artk[OPW];          // that artificial's index or -1
    unsigned bas;           // bit t: position's variable basic; bit 16+t: paired artificial basic
    int basis_r;            // basic variable of row `lane`
    int art_of_r;           // artificial index of row `lane` or -1
    unsigned long long ckey;// entering candidates (warp-uniform after reduction)
    int cidx, cbl;
};

struct WlpDims { int m, n, nvc, ncols, lane; };

template <int CPW, int KIND>
__device__ __forceinline__ void wlp_candidates(const WlpDims &D, WlpState<CPW> &S) {
    unsigned long long ck = kKeyEmptyMax;
    int ci = kNone, cb = kNone;
#pragma unroll
    for (int t = 0; t < WlpState<CPW>::OPW; ++t) {
        const int pos = D.lane + 32 * t;
        if (pos >= 1 && pos < D.ncols) {
            const int j = pos - 1;
            if (!(S.bas & (1u << t))) {
                const unsigned long long k = key_max(S.rc[t]);
                if (k > ck || (k == ck && j < ci)) { ck = k; ci = j; }
                if (S.rc[t] > kTol && j < cb) cb = j;
            }
            if (KIND == kWlpPhase1 && S.artk[t] >= 0 && !(S.bas & (0x10000u << t))) {
                const int ja = D.nvc + S.artk[t];
                const unsigned long long k = key_max(S.arc[t]);
                if (k > ck || (k == ck && ja < ci)) { ck = k; ci = ja; }
                if (S.arc[t] > kTol && ja < cb) cb = ja;
            }
        }
    }
    S.ckey = warp_max_key(ck);
    S.cidx = warp_index_of(ck, S.ckey, ci);
    S.cbl = (int)__reduce_min_sync(kFull, (unsigned)cb);
}

// Predicated 16-byte shared-memory store / load (one lane of the warp acts;
// the others keep their registers).  Written as PTX so the row write is 32
// single-instruction predicated stores instead of a divergent block.
__device__ __forceinline__ void st_shared_v2_if(bool p, unsigned addr, double x, double y) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.shared.v2.f64 [%1], {%2, %3}; }"
                 ::"r"((unsigned)p), "r"(addr), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void ld_shared_v2_if(bool p, unsigned addr, double &x, double &y) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q ld.volatile.shared.v2.f64 {%0, %1}, [%3]; }"
                 : "+d"(x), "+d"(y) : "r"((unsigned)p), "r"(addr) : "memory");
}

// pivot (tableau.py:218-244): entering column values av (this lane's row),
// leaving row l, fm = reduced cost of the entering column.  Row l is stored
// to smem, every lane divides its transposed positions (r = a_lq / pe) and
// updates its objective slots, every row takes a_ij - f_i * r_j, and the
// leaving row's lane finally reloads r itself (numpy: r - 0*r == r).
template <int CPW, int KIND>
__device__ __forceinline__ void wlp_pivot(const WlpDims &D, WlpState<CPW> &S, unsigned char *smem, int e,
                                          int l, double av, double fm, int oldvar) {
    using C = WlpCfg<CPW>;
    double *rowbuf = reinterpret_cast<double *>(smem + C::ROWBUF);
    double *rvec = reinterpret_cast<double *>(smem + C::RVEC);
    const unsigned rb = (unsigned)__cvta_generic_to_shared(rowbuf);
    const unsigned rv = (unsigned)__cvta_generic_to_shared(rvec);
    const double pe = __shfl_sync(kFull, av, l);
    const bool mine = D.lane == l;
#pragma unroll
    for (int c = 0; c < CPW; c += 2) st_shared_v2_if(mine, rb + 8u * c, S.a[c], S.a[c + 1]);
    if (mine) S.basis_r = e;
    __syncwarp();
#pragma unroll
    for (int t = 0; t < WlpState<CPW>::OPW; ++t) {
        const int pos = D.lane + 32 * t;
        if (pos < D.ncols) {
            const double r = div_entry(rowbuf[pos], pe);
            rvec[pos] = r;
            if (pos == 0) {
                S.rc[t] = __dadd_rn(S.rc[t], __dmul_rn(fm, r));   // tableau.py:242
            } else {
                S.rc[t] = __dsub_rn(S.rc[t], __dmul_rn(fm, r));
                const int j = pos - 1;
                if (j == e) S.bas |= (1u << t);
                if (j == oldvar) S.bas &= ~(1u << t);
                if (KIND == kWlpPhase1 && S.artk[t] >= 0) {
                    S.arc[t] = __dsub_rn(S.arc[t], __dmul_rn(fm, -r));
                    const int ja = D.nvc + S.artk[t];
                    if (ja == e) S.bas |= (0x10000u << t);
                    if (ja == oldvar) S.bas &= ~(0x10000u << t);
                }
            }
        }
    }
    if (KIND != kWlpRestore) wlp_candidates<CPW, KIND>(D, S);
    __syncwarp();
#pragma unroll
    for (int c = 0; c < CPW; c += 2) {
        const double2 r2 = reinterpret_cast<const double2 *>(rvec)[c / 2];
        S.a[c] = __dsub_rn(S.a[c], __dmul_rn(av, r2.x));
        S.a[c + 1] = __dsub_rn(S.a[c + 1], __dmul_rn(av, r2.y));
    }
#pragma unroll
    for (int c = 0; c < CPW; c += 2) ld_shared_v2_if(mine, rv + 8u * c, S.a[c], S.a[c + 1]);
}

// Row of artificial k (the lane whose row got it).
__device__ __forceinline__ int wlp_row_of_art(int art_of_r, int k) {
    return __ffs(__ballot_sync(kFull, art_of_r == k)) - 1;
}

struct WlpPhase { int state, iters; };

// _run_phase (simplex.py:63-91); entering candidates already in S.
template <int CPW, int KIND>
__device__ __forceinline__ WlpPhase wlp_run_phase(const WlpDims &D, WlpState<CPW> &S, unsigned char *smem, const Limits &lim) {
    const int max_iter = lim.max_iterations > 0 ? lim.max_iterations : 50 * (D.m + D.n);
    const int trigger = lim.degenerate_limit >= 0 ? lim.degenerate_limit : (D.m > 1 ? D.m : 1);
    const unsigned long long kSent = key_max(kSentinel), kDeg = key_max(kDegenerateTol), kTolK = key_max(kTol);
    int degenerate_run = 0;
    bool use_bland = false;
    for (int it = 0;; ++it) {
        if (it == max_iter) return {2, max_iter};
        int e;
        if (use_bland) e = S.cbl == kNone ? -1 : S.cbl;           // choose_entering_bland
        else e = (S.cidx == kNone || S.ckey <= kTolK) ? -1 : S.cidx;  // choose_entering
        if (e < 0) return {0, it};
        const bool art_e = e >= D.nvc;
        const int epos = art_e ? 1 + D.n + wlp_row_of_art(S.art_of_r, e - D.nvc) : e + 1;
        double av = reg_pick<CPW>(S.a, epos);
        if (art_e) av = -av;
        // choose_leaving (tableau.py:200-215): rhs is register 0
        unsigned long long lk = kKeyEmptyMin;
        const double ratio = ratio_entry(S.a[0], av);
        if (D.lane < D.m) lk = key_min(ratio);
        const unsigned long long kmin = warp_min_key(lk);
        const int l = warp_index_of(lk, kmin, D.lane);
        if (l == kNone || kmin >= kSent) return {1, it};   // unbounded (a NaN ratio keys to 0)
        double myfm = 0.0;   // selp, not a branch: a computed index would demote S to local memory
#pragma unroll
        for (int t = 0; t < WlpState<CPW>::OPW; ++t)
            myfm = selp_f64(art_e ? S.arc[t] : S.rc[t], myfm, t == (epos >> 5));
        const double fm = __shfl_sync(kFull, myfm, epos & 31);
        const int oldvar = __shfl_sync(kFull, S.basis_r, l);
        if (kmin != 0ull && kmin <= kDeg) {                 // simplex.py:84-90
            ++degenerate_run;
            if (lim.anti_cycling && degenerate_run >= trigger) use_bland = true;
        } else {
            degenerate_run = 0;
            use_bland = false;
        }
        wlp_pivot<CPW, KIND>(D, S, smem, e, l, D.lane < D.m ? av : 0.0, fm, oldvar);
    }
}

// _price_out (simplex.py:133-143) from the stage, transposed: lane q rebuilds
// the reduced costs of positions q, q+32 with the rows in reference order.
template <int CPW, int PHASE>
__device__ __forceinline__ void wlp_price_out(const WlpDims &D, WlpState<CPW> &S, unsigned char *smem,
                                              const double *cg) {
    using C = WlpCfg<CPW>;
    double *cbv = reinterpret_cast<double *>(smem + C::CBV);
    const double *stage = reinterpret_cast<const double *>(smem + C::STAGE);
    cbv[D.lane] = D.lane < D.m ? (PHASE == 1 ? (S.basis_r >= D.nvc ? -1.0 : 0.0)
                                             : (S.basis_r < D.n ? cg[S.basis_r] : 0.0))
                               : 0.0;
    __syncwarp();
#pragma unroll
    for (int t = 0; t < WlpState<CPW>::OPW; ++t) {
        const int pos = D.lane + 32 * t;
        if (pos < D.ncols) {
            const double *col = stage + pos;
            const int j = pos - 1;
            const bool art = PHASE == 1 && S.artk[t] >= 0;
            double rc = (PHASE == 2 && pos >= 1 && j < D.n) ? cg[j] : 0.0;
            double ac = -1.0;
            for (int r = 0; r < D.m; ++r) {
                const double cb = cbv[r];
                if (cb != 0.0) {
                    const double v = col[r * C::LDG];
                    if (pos == 0) {
                        rc = __dadd_rn(rc, __dmul_rn(cb, v));
                    } else {
                        rc = __dsub_rn(rc, __dmul_rn(cb, v));
                        if (art) ac = __dsub_rn(ac, __dmul_rn(cb, -v));
                    }
                }
            }
            S.rc[t] = rc;
            if (art) S.arc[t] = ac;
        }
    }
    wlp_candidates<CPW, PHASE == 1 ? kWlpPhase1 : kWlpPhase2>(D, S);
}

template <int CPW>
__device__ __forceinline__ void wlp_tile_to_stage(const WlpDims &D, const WlpState<CPW> &S, unsigned char *smem) {
    double *stage = reinterpret_cast<double *>(smem + WlpCfg<CPW>::STAGE);
    if (D.lane < D.m) {
#pragma unroll
        for (int c = 0; c < CPW; ++c) stage[D.lane * WlpCfg<CPW>::LDG + c] = S.a[c];
    }
    __syncwarp();
}

// restore_objective pivot-outs (simplex.py:109-126), uncounted.
template <int CPW>
__device__ __forceinline__ void wlp_restore(const WlpDims &D, WlpState<CPW> &S, unsigned char *smem) {
    const unsigned long long kRed = key_max(kRedundantTol);
    for (int row = 0; row < D.m; ++row) {
        if (__shfl_sync(kFull, S.basis_r, row) < D.nvc) continue;
        unsigned long long bk = kKeyEmptyMax;
        int bj = kNone;
        if (D.lane == row) {
#pragma unroll
            for (int c = 1; c < CPW; ++c) {
                if (c < D.ncols) {
                    const unsigned long long k = key_max(fabs(S.a[c]));
                    if (k > bk) { bk = k; bj = c - 1; }
                }
            }
        }
        bk = __shfl_sync(kFull, bk, row);
        bj = __shfl_sync(kFull, bj, row);
        // entries[j] > REDUNDANT_ROW_TOL; a NaN entry compares False in numpy
        if (bj != kNone && bk > kRed && bk != ~0ull) {
            const double av = reg_pick<CPW>(S.a, bj + 1);
            const int oldvar = __shfl_sync(kFull, S.basis_r, row);
            wlp_pivot<CPW, kWlpRestore>(D, S, smem, bj, row, D.lane < D.m ? av : 0.0, 0.0, oldvar);
        }
    }
}

// L2 prefetch of one LP's A, b, c (128-byte lines spread over the warp).
__device__ __forceinline__ void prefetch_lp_inputs(const Batch &B, long long lp, int lane) {
    const size_t mn = (size_t)B.m * B.n;
    if (!B.shared_Ab) {
        const char *a = reinterpret_cast<const char *>(B.A + (size_t)lp * mn);
        for (size_t off = (size_t)lane * 128; off < mn * 8; off += 32 * 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a + off));
        if (lane == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(B.b + (size_t)lp * B.m));
    }
    if (lane == 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(B.c + (size_t)lp * B.n));
}

template <int CPW, int kMinBlocks>
__global__ void __launch_bounds__(32, kMinBlocks)
warplp_kernel(Batch B) {
    using C = WlpCfg<CPW>;
    extern __shared__ __align__(16) unsigned char smem[];
    WlpDims D;
    D.m = B.m; D.n = B.n; D.nvc = B.n + B.m; D.ncols = B.n + B.m + 1; D.lane = threadIdx.x;
    const int m = D.m, n = D.n, nvc = D.nvc;
    double *stage = reinterpret_cast<double *>(smem + C::STAGE);
    {
        double *rowbuf = reinterpret_cast<double *>(smem + C::ROWBUF);
        double *rvec = reinterpret_cast<double *>(smem + C::RVEC);
        for (int q = D.lane; q < CPW; q += 32) { rowbuf[q] = 0.0; rvec[q] = 0.0; }
    }
    WlpState<CPW> S;
    long long lp = 0;
    if (D.lane == 0) lp = atomicAdd(B.next_lp, 1);
    lp = __shfl_sync(kFull, lp, 0);
    for (;;) {
        if (lp >= B.count) break;
        // Claim the next LP now and pull its inputs into L2 while this one is
        // solved: the queue atomic and the HBM latency leave the critical path.
        long long nxt = 0;
        if (D.lane == 0) nxt = atomicAdd(B.next_lp, 1);
        nxt = __shfl_sync(kFull, nxt, 0);
        if (nxt < B.count) prefetch_lp_inputs(B, nxt, D.lane);
        const double *Ag = B.shared_Ab ? B.A : B.A + (size_t)lp * m * n;
        const double *bg = B.shared_Ab ? B.b : B.b + (size_t)lp * m;
        const double *cg = B.c + (size_t)lp * n;

        // ---- build_tableau (tableau.py:139-172) through the stage; validation fused ----
        const double bi = D.lane < m ? bg[D.lane] : 0.0;
        bool nonfinite = !isfinite(bi);
        const bool neg = D.lane < m && bi < 0.0;
        const unsigned negmask = __ballot_sync(kFull, neg);
        const int n_art = __popc(negmask);
        const double sgn = neg ? -1.0 : 1.0;
        S.art_of_r = neg ? __popc(negmask & ((1u << D.lane) - 1u)) : -1;
        S.basis_r = neg ? nvc + S.art_of_r : n + D.lane;
        if (D.lane < m) stage[D.lane * C::LDG] = __dmul_rn(bi, sgn);
        // A: lane j loads column j of every row, all loads in flight at once
#pragma unroll
        for (int cc = 0; cc < C::OPW; ++cc) {
            const int j = D.lane + 32 * cc;
            double v[32];
#pragma unroll
            for (int r = 0; r < 32; ++r) v[r] = (r < m && j < n) ? Ag[(size_t)r * n + j] : 0.0;
#pragma unroll
            for (int r = 0; r < 32; ++r) {
                const double sr = __shfl_sync(kFull, sgn, r);
                if (r < m && j < n) {
                    nonfinite |= !isfinite(v[r]);
                    stage[r * C::LDG + 1 + j] = __dmul_rn(v[r], sr);
                }
            }
        }
        for (int r = 0; r < m; ++r) {
            const double sr = __shfl_sync(kFull, sgn, r);
            for (int q = D.lane; q < m; q += 32) stage[r * C::LDG + 1 + n + q] = q == r ? sr : 0.0;
        }
        for (int j = D.lane; j < n; j += 32) nonfinite |= !isfinite(cg[j]);
        const bool invalid = __any_sync(kFull, nonfinite);
        __syncwarp();
#pragma unroll
        for (int c = 0; c < CPW; ++c)
            S.a[c] = (D.lane < m && c < D.ncols) ? stage[D.lane * C::LDG + c] : 0.0;
        S.bas = 0;
#pragma unroll
        for (int t = 0; t < C::OPW; ++t) {
            const int pos = D.lane + 32 * t;
            const int j = pos - 1;
            S.rc[t] = (pos >= 1 && j < n) ? cg[j] : 0.0;
            S.arc[t] = 0.0;
            const int row = j - n;   // slack position of row `row`
            const int k = __shfl_sync(kFull, S.art_of_r, row & 31);
            S.artk[t] = (j >= n && j < nvc) ? k : -1;
            if (j >= n && j < nvc) S.bas |= (k < 0) ? (1u << t) : (0x10000u << t);
        }

        int8_t status = kOptimal;
        int it1 = 0, it2 = 0;
        bool done = false;
        if (invalid) {
            status = kInvalid;
            done = true;
        } else if (n_art > 0) {
            wlp_price_out<CPW, 1>(D, S, smem, cg);                      // build_auxiliary
            const WlpPhase p1 = wlp_run_phase<CPW, kWlpPhase1>(D, S, smem, B.lim);
            it1 = p1.iters;
            const double obj = __shfl_sync(kFull, S.rc[0], 0);
            if (p1.state == 2) { status = kIterationLimit; done = true; }
            else if (p1.state == 1) { status = kErrPhase1Unbounded; done = true; }
            else if (fabs(obj) > kPhase1ZeroTol) { status = kInfeasible; done = true; }
            else {
                wlp_restore<CPW>(D, S, smem);
                __syncwarp();
                wlp_tile_to_stage<CPW>(D, S, smem);
                wlp_price_out<CPW, 2>(D, S, smem, cg);
            }
        } else {
            wlp_candidates<CPW, kWlpPhase2>(D, S);
        }
        if (!done) {
            const WlpPhase p2 = wlp_run_phase<CPW, kWlpPhase2>(D, S, smem, B.lim);
            it2 = p2.iters;
            if (p2.state == 2) status = kIterationLimit;
            else if (p2.state == 1) status = kUnbounded;
        }

        // ---- _extract_point (simplex.py:146-151) and c @ x ----
        __syncwarp();
        double *xs = stage;
        for (int j = D.lane; j < n; j += 32) xs[j] = 0.0;
        __syncwarp();
        if (status == kOptimal && D.lane < m && S.basis_r < n) xs[S.basis_r] = S.a[0];
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
        lp = nxt;
    }
}

}  // namespace blp
