// blp_warplp2_kernel.cuh -- one warp per LP, tableau split between registers
// and shared memory (m <= 32 rows, n + m + 1 <= R + S columns; C1 / C2).
//
// Same algorithm and numerics as blp_warplp_kernel.cuh, with the row of lane
// r split in two: positions [0, R) in registers (a[]), positions [R, R+S)
// in a per-warp shared-memory tile stored column-major (tile[c][row], so a
// warp's 32 rows of one column are 256 contiguous bytes: conflict-free).
// Why: a 64-double register row caps the SM at 12 resident LPs (168
// registers per thread); a 38/24 split runs 16 LPs per SM for ~4% more
// instructions per pivot.  The shared-memory half also needs no transfer for
// the pivot row (lane q reads tile[q-R][l] directly and writes r_q back into
// row l), and there is no staging buffer: rows are loaded straight from HBM
// into their lane, and price-out streams one row at a time through smem.
#pragma once

#ifndef WL2_PIPE
#define WL2_PIPE 1   // C2 1e5: 8.43 -> 8.30 ms, and no spills
#endif

#include "blp_common.cuh"
#include "blp_keys.cuh"
#include "blp_warplp_kernel.cuh"

namespace blp {

template <int R, int S>
struct Wl2Cfg {
    static constexpr int CPW = R + S;
    static constexpr int OPW = (CPW + 31) / 32;
    // column stride 33 doubles: a row read across columns (lane q -> tile[q][l],
    // the pivot row's division) hits 16 distinct bank pairs instead of one
    static constexpr int TS = 33;
    static constexpr size_t TILE = 0;                              // S x TS doubles
    static constexpr size_t ROWBUF = TILE + (size_t)S * TS * 8;    // R doubles
    static constexpr size_t RVEC = ROWBUF + (size_t)R * 8;         // CPW doubles
    static constexpr size_t CBV = RVEC + (size_t)((CPW + 1) & ~1) * 8;
    static constexpr size_t BYTES = CBV + 32 * 8;
};

template <int R, int S>
struct Wl2State {
    static constexpr int OPW = Wl2Cfg<R, S>::OPW;
    double a[R];            // positions [0, R) of row `lane` (rhs at 0)
    double rc[OPW];         // transposed objective row; position 0 holds the objective value
    double arc[OPW];        // phase-1 reduced cost of the artificial paired with a slack position
    int artk[OPW];
    unsigned bas;           // bit t: position's variable basic; bit 16+t: paired artificial basic
    int basis_r, art_of_r;
    unsigned long long ckey;
    int cidx, cbl;
};

template <int R, int S, int KIND>
__device__ __forceinline__ void wl2_candidates(const WlpDims &D, Wl2State<R, S> &St) {
    unsigned long long ck = kKeyEmptyMax;
    int ci = kNone, cb = kNone;
#pragma unroll
    for (int t = 0; t < Wl2State<R, S>::OPW; ++t) {
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

// Entry of this lane's row at a warp-uniform position.
template <int R, int S>
__device__ __forceinline__ double wl2_at(const Wl2State<R, S> &St, const double *tile, int lane, int pos) {
    if (pos < R) return reg_pick<R>(St.a, pos);
    return tile[(pos - R) * Wl2Cfg<R, S>::TS + lane];
}

// pivot (tableau.py:218-244): av = this lane's entry of the entering column,
// l = leaving row, fm = reduced cost of the entering column.
template <int R, int S, int KIND>
__device__ __forceinline__ void wl2_pivot(const WlpDims &D, Wl2State<R, S> &St, unsigned char *smem, int e,
                                          int l, double av, double fm, int oldvar) {
    using C = Wl2Cfg<R, S>;
    double *tile = reinterpret_cast<double *>(smem + C::TILE);
    double *rowbuf = reinterpret_cast<double *>(smem + C::ROWBUF);
    double *rvec = reinterpret_cast<double *>(smem + C::RVEC);
    const unsigned rb = (unsigned)__cvta_generic_to_shared(rowbuf);
    const unsigned rv = (unsigned)__cvta_generic_to_shared(rvec);
    const double pe = __shfl_sync(kFull, av, l);
    const bool mine = D.lane == l;
#pragma unroll
    for (int c = 0; c < R; c += 2) st_shared_v2_if(mine, rb + 8u * c, St.a[c], St.a[c + 1]);
    if (mine) St.basis_r = e;
    __syncwarp();
#pragma unroll
    for (int t = 0; t < Wl2State<R, S>::OPW; ++t) {
        const int pos = D.lane + 32 * t;
        if (pos < D.ncols) {
            double *src = pos < R ? rowbuf + pos : tile + (pos - R) * C::TS + l;
            const double r = div_entry(*src, pe);
            rvec[pos] = r;
            if (pos >= R) *src = r;                              // row l of an smem column: final
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
    if (KIND != kWlpRestore) wl2_candidates<R, S, KIND>(D, St);
    __syncwarp();
#pragma unroll
    for (int c = 0; c < R; c += 2) {
        const double2 r2 = reinterpret_cast<const double2 *>(rvec)[c / 2];
        St.a[c] = __dsub_rn(St.a[c], __dmul_rn(av, r2.x));
        St.a[c + 1] = __dsub_rn(St.a[c + 1], __dmul_rn(av, r2.y));
    }
    const double fs = mine ? 0.0 : av;     // row l of the smem columns already holds r
#if WL2_PIPE
    {
        // software-pipelined: batch b+1 (4 columns + their pivot-row entries) is loaded
        // before batch b is stored (tile and rvec share shared memory, so the compiler
        // would otherwise order each load after every earlier store)
        constexpr int K = 4, NB = (S + K - 1) / K;
        const unsigned ca = (unsigned)__cvta_generic_to_shared(tile + D.lane);
        const unsigned ra = (unsigned)__cvta_generic_to_shared(rvec + R);
        double t[2][K], r[2][K];
        auto load = [&](int b, int sl) {
#pragma unroll
            for (int k = 0; k < K; k += 2) {
                const int c = b * K + k;
                if (c < S) {
                    lds_v2_f64(ra + 8u * c, r[sl][k], r[sl][k + 1]);
                    t[sl][k] = lds_f64(ca + 8u * C::TS * c);
                    if (c + 1 < S) t[sl][k + 1] = lds_f64(ca + 8u * C::TS * (c + 1));
                }
            }
        };
        load(0, 0);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            if (b + 1 < NB) load(b + 1, (b + 1) & 1);
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int c = b * K + k;
                if (c < S) sts_f64(ca + 8u * C::TS * c, __dsub_rn(t[b & 1][k], __dmul_rn(fs, r[b & 1][k])));
            }
        }
    }
#else
    double *col = tile + D.lane;
#pragma unroll
    for (int c = 0; c < S; c += 2) {
        const double2 r2 = reinterpret_cast<const double2 *>(rvec + R)[c / 2];
        const double t0 = col[c * C::TS], t1 = col[(c + 1) * C::TS];
        col[c * C::TS] = __dsub_rn(t0, __dmul_rn(fs, r2.x));
        col[(c + 1) * C::TS] = __dsub_rn(t1, __dmul_rn(fs, r2.y));
    }
#endif
#pragma unroll
    for (int c = 0; c < R; c += 2) ld_shared_v2_if(mine, rv + 8u * c, St.a[c], St.a[c + 1]);
    __syncwarp();
}

// _run_phase (simplex.py:63-91); entering candidates already in St.
template <int R, int S, int KIND>
__device__ __forceinline__ WlpPhase wl2_run_phase(const WlpDims &D, Wl2State<R, S> &St, unsigned char *smem,
                                                  const Limits &lim) {
    const double *tile = reinterpret_cast<const double *>(smem + Wl2Cfg<R, S>::TILE);
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
        double av = wl2_at<R, S>(St, tile, D.lane, epos);
        if (art_e) av = -av;
        unsigned long long lk = kKeyEmptyMin;                               // choose_leaving
        const double ratio = ratio_entry(St.a[0], av);
        if (D.lane < D.m) lk = key_min(ratio);
        const unsigned long long kmin = warp_min_key(lk);
        const int l = warp_index_of(lk, kmin, D.lane);
        if (l == kNone || kmin >= kSent) return {1, it};   // unbounded (a NaN ratio keys to 0)
        double myfm = 0.0;
#pragma unroll
        for (int t = 0; t < Wl2State<R, S>::OPW; ++t)
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
        wl2_pivot<R, S, KIND>(D, St, smem, e, l, D.lane < D.m ? av : 0.0, fm, oldvar);
    }
}

// Row `row` broadcast for column-wise scans: its register part goes to
// rowbuf; entries are then read as rowbuf[p] (p < R) or tile[p-R][row].
template <int R, int S>
__device__ __forceinline__ void wl2_share_row(const WlpDims &D, const Wl2State<R, S> &St, unsigned char *smem,
                                              int row) {
    const unsigned rb = (unsigned)__cvta_generic_to_shared(smem + Wl2Cfg<R, S>::ROWBUF);
    __syncwarp();
#pragma unroll
    for (int c = 0; c < R; c += 2) st_shared_v2_if(D.lane == row, rb + 8u * c, St.a[c], St.a[c + 1]);
    __syncwarp();
}

template <int R, int S>
__device__ __forceinline__ double wl2_row_entry(unsigned char *smem, int row, int pos) {
    using C = Wl2Cfg<R, S>;
    return pos < R ? reinterpret_cast<const double *>(smem + C::ROWBUF)[pos]
                   : reinterpret_cast<const double *>(smem + C::TILE)[(pos - R) * C::TS + row];
}

// _price_out (simplex.py:133-143), transposed: lane q rebuilds the reduced
// costs of positions q, q+32, rows in reference order, skipping cb == 0 rows.
template <int R, int S, int PHASE>
__device__ __forceinline__ void wl2_price_out(const WlpDims &D, Wl2State<R, S> &St, unsigned char *smem,
                                              const double *cg) {
    double *cbv = reinterpret_cast<double *>(smem + Wl2Cfg<R, S>::CBV);
    cbv[D.lane] = D.lane < D.m ? (PHASE == 1 ? (St.basis_r >= D.nvc ? -1.0 : 0.0)
                                             : (St.basis_r < D.n ? cg[St.basis_r] : 0.0))
                               : 0.0;
    double rc[Wl2State<R, S>::OPW], ac[Wl2State<R, S>::OPW];
#pragma unroll
    for (int t = 0; t < Wl2State<R, S>::OPW; ++t) {
        const int pos = D.lane + 32 * t, j = pos - 1;
        rc[t] = (PHASE == 2 && pos >= 1 && j < D.n) ? cg[j] : 0.0;
        ac[t] = -1.0;
    }
    __syncwarp();
    for (int r = 0; r < D.m; ++r) {
        const double cb = cbv[r];
        if (cb == 0.0) continue;          // uniform: every lane reads the same cbv[r]
        wl2_share_row<R, S>(D, St, smem, r);
#pragma unroll
        for (int t = 0; t < Wl2State<R, S>::OPW; ++t) {
            const int pos = D.lane + 32 * t;
            if (pos < D.ncols) {
                const double v = wl2_row_entry<R, S>(smem, r, pos);
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
    for (int t = 0; t < Wl2State<R, S>::OPW; ++t) {
        const int pos = D.lane + 32 * t;
        if (pos < D.ncols) {
            St.rc[t] = rc[t];
            if (PHASE == 1 && St.artk[t] >= 0) St.arc[t] = ac[t];
        }
    }
    wl2_candidates<R, S, PHASE == 1 ? kWlpPhase1 : kWlpPhase2>(D, St);
}

// restore_objective pivot-outs (simplex.py:109-126), uncounted.
template <int R, int S>
__device__ __forceinline__ void wl2_restore(const WlpDims &D, Wl2State<R, S> &St, unsigned char *smem) {
    const double *tile = reinterpret_cast<const double *>(smem + Wl2Cfg<R, S>::TILE);
    const unsigned long long kRed = key_max(kRedundantTol);
    for (int row = 0; row < D.m; ++row) {
        if (__shfl_sync(kFull, St.basis_r, row) < D.nvc) continue;
        wl2_share_row<R, S>(D, St, smem, row);
        unsigned long long bk = kKeyEmptyMax;
        int bj = kNone;
#pragma unroll
        for (int t = 0; t < Wl2State<R, S>::OPW; ++t) {
            const int pos = D.lane + 32 * t;
            if (pos >= 1 && pos < D.ncols) {
                const unsigned long long k = key_max(fabs(wl2_row_entry<R, S>(smem, row, pos)));
                if (k > bk) { bk = k; bj = pos - 1; }     // positions ascend per lane
            }
        }
        const unsigned long long kb = warp_max_key(bk);
        const int j = warp_index_of(bk, kb, bj);
        // entries[j] > REDUNDANT_ROW_TOL; a NaN entry compares False in numpy
        if (j != kNone && kb > kRed && kb != ~0ull) {
            const double av = wl2_at<R, S>(St, tile, D.lane, j + 1);
            const int oldvar = __shfl_sync(kFull, St.basis_r, row);
            wl2_pivot<R, S, kWlpRestore>(D, St, smem, j, row, D.lane < D.m ? av : 0.0, 0.0, oldvar);
        }
    }
}

template <int R, int S, int kMinBlocks>
__global__ void __launch_bounds__(32, kMinBlocks)
warplp2_kernel(Batch B) {
    using C = Wl2Cfg<R, S>;
    extern __shared__ __align__(16) unsigned char smem[];
    WlpDims D;
    D.m = B.m; D.n = B.n; D.nvc = B.n + B.m; D.ncols = B.n + B.m + 1; D.lane = threadIdx.x;
    const int m = D.m, n = D.n, nvc = D.nvc;
    double *tile = reinterpret_cast<double *>(smem + C::TILE);
    {
        double *rvec = reinterpret_cast<double *>(smem + C::RVEC);
        for (int q = D.lane; q < C::CPW; q += 32) rvec[q] = 0.0;
    }
    Wl2State<R, S> St;
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
#pragma unroll 4
        for (int c = 0; c < S; ++c) {
            const int j = R + c - 1;
            double v = 0.0;
            if (live) {
                if (j < n) { const double a = arow[j]; nonfinite |= !isfinite(a); v = __dmul_rn(a, sgn); }
                else if (j < nvc) v = (j - n == D.lane) ? sgn : 0.0;
            }
            tile[c * C::TS + D.lane] = v;
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
        __syncwarp();

        int8_t status = kOptimal;
        int it1 = 0, it2 = 0;
        bool done = false;
        if (invalid) {
            status = kInvalid;
            done = true;
        } else if (n_art > 0) {
            wl2_price_out<R, S, 1>(D, St, smem, cg);                     // build_auxiliary
            const WlpPhase p1 = wl2_run_phase<R, S, kWlpPhase1>(D, St, smem, B.lim);
            it1 = p1.iters;
            const double obj = __shfl_sync(kFull, St.rc[0], 0);
            if (p1.state == 2) { status = kIterationLimit; done = true; }
            else if (p1.state == 1) { status = kErrPhase1Unbounded; done = true; }
            else if (fabs(obj) > kPhase1ZeroTol) { status = kInfeasible; done = true; }
            else {
                wl2_restore<R, S>(D, St, smem);
                wl2_price_out<R, S, 2>(D, St, smem, cg);
            }
        } else {
            wl2_candidates<R, S, kWlpPhase2>(D, St);
        }
        if (!done) {
            const WlpPhase p2 = wl2_run_phase<R, S, kWlpPhase2>(D, St, smem, B.lim);
            it2 = p2.iters;
            if (p2.state == 2) status = kIterationLimit;
            else if (p2.state == 1) status = kUnbounded;
        }

        // ---- _extract_point (simplex.py:146-151) and c @ x ----
        double *xs = reinterpret_cast<double *>(smem + C::RVEC);   // n <= CPW doubles of scratch
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
}

}  // namespace blp
