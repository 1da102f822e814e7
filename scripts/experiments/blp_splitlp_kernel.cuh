// blp_splitlp_kernel.cuh -- one CTA per LP with every row SPLIT over NCH
// threads (column halves), so a 100 x 100 tableau (C3) lives almost entirely
// in registers: 4 row-warps x 2 halves = 256 threads, each holding R = 96
// columns of its row in registers and S = 4 in a small shared tile.
//
// quadlp (blp_pairlp_kernel.cuh, NWR = 4) keeps 96 columns of a row in one
// thread's registers and the other 106 in a shared tile, two LPs per SM; its
// bottleneck is that tile (the update is 29% of instructions, the shared pipe
// the busiest).  Here the register file of a whole SM (256 threads x 255
// registers) holds one LP, so the rank-1 update is DMUL/DSUB on registers
// (FP64-bound) with the pivot row broadcast from shared memory.
//
// Layout: thread t = (row-warp w % NWR, half h = w / NWR, lane L) holds row
// r = 32 (w % NWR) + L, columns [h CPH, (h+1) CPH) with CPH = R + S
// (structural + slack columns; j < R of a half in registers, the rest in
// tile_h[c][r]); the rhs is replicated in both halves' registers.  The
// transposed objective row is dealt round-robin over all NT threads
// (position 0 = the objective value, position 1 + j = column j).
// Per pivot (tableau.py:175-244), three CTA barriers as in pairlp:
//   A  the half owning the entering column computes its entries (fvec, for
//      the other half) and the ratio test;
//   B  both halves of the leaving row publish their register columns (rowbuf);
//   C  the transposed threads divide the pivot row, price and nominate the
//      next entering column; then every thread updates its columns.
// Arithmetic and selection rules are pairlp's, so results are identical to it
// and to the reference.
#pragma once

#include "blp_common.cuh"
#include "blp_keys.cuh"
#include "blp_warplp_kernel.cuh"

namespace blp {

struct SplitXch {
    unsigned long long ckey[32];  // per-warp entering candidates
    int cidx[32], cbl[32];
    unsigned long long lkey[32];  // per-warp leaving partials
    int lrow[32];
    int nneg[32];
    double pe, fm, obj;
    int oldvar;
};

template <int R, int S, int NWR, int NCH, int ST>
struct SplitCfg {
    static constexpr int CPH = R + S;                     // columns per half
    static constexpr int COLS = NCH * CPH;                // column capacity (>= n + m)
    static constexpr int ROWS = 32 * NWR;
    static constexpr int NT = ROWS * NCH;
    static constexpr int NWARPS = NT / 32;
    static constexpr int NPOS = COLS + 1;                 // transposed positions
    static constexpr int OPW = (NPOS + NT - 1) / NT;
    static_assert((ST & 1) && (CPH % 2 == 0) && (R % 2 == 0) && S >= 1 && NWARPS <= 32, "split layout");
    static constexpr size_t TILE = 0;                                      // NCH x S x ST doubles
    static constexpr size_t ROWBUF = TILE + (size_t)NCH * S * ST * 8;      // COLS doubles + rhs_l
    static constexpr size_t RVEC = ROWBUF + (size_t)(COLS + 2) * 8;        // COLS doubles + r_rhs
    static constexpr size_t FVEC = RVEC + (size_t)(COLS + 2) * 8;          // ROWS doubles
    static constexpr size_t CBV = FVEC + (size_t)ROWS * 8;                 // ROWS doubles
    static constexpr size_t ARTROW = CBV + (size_t)ROWS * 8;               // ROWS ints
    static constexpr size_t ARTOF = ARTROW + (size_t)ROWS * 4;             // ROWS ints
    static constexpr size_t XCH = ARTOF + (size_t)ROWS * 4;
    static constexpr size_t BYTES = XCH + (sizeof(SplitXch) + 15) / 16 * 16;
};


template <int R, int S, int NWR, int NCH, int ST>
struct SplitState {
    static constexpr int OPW = SplitCfg<R, S, NWR, NCH, ST>::OPW;
    double a[R];            // this half's register columns of row `row`
    double rhs;             // rhs of row `row` (replicated in both halves)
    double rc[OPW];         // transposed objective row; position 0 = objective value
    double arc[OPW];        // phase-1 reduced cost of the artificial paired with a slack position
    int artk[OPW];
    unsigned bas;           // bit t: position's variable basic; bit 16+t: paired artificial basic
    int basis_r;
};

struct SplitDims { int m, n, nvc, ncols, tid, lane, warp, row, half; };

template <int NT>
__device__ __forceinline__ int split_pos(const SplitDims &D, int t) { return D.tid + NT * t; }

template <int R, int S, int NWR, int NCH, int ST, int KIND>
__device__ __forceinline__ void split_candidates(const SplitDims &D, const SplitState<R, S, NWR, NCH, ST> &St,
                                                 SplitXch *X) {
    using C = SplitCfg<R, S, NWR, NCH, ST>;
    unsigned long long ck = kKeyEmptyMax;
    int ci = kNone, cb = kNone;
#pragma unroll
    for (int t = 0; t < C::OPW; ++t) {
        const int pos = split_pos<C::NT>(D, t);
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
    const unsigned long long kw = warp_max_key(ck);
    const int iw = warp_index_of(ck, kw, ci);
    const int bw = (int)__reduce_min_sync(kFull, (unsigned)cb);
    if (D.lane == 0) { X->ckey[D.warp] = kw; X->cidx[D.warp] = iw; X->cbl[D.warp] = bw; }
}

// Combine per-warp (max key, lowest index) partials over all warps.
template <int NWARPS>
__device__ __forceinline__ void split_combine_max(const SplitXch *X, unsigned long long &k, int &i) {
    k = X->ckey[0];
    i = X->cidx[0];
#pragma unroll
    for (int w = 1; w < NWARPS; ++w)
        if (X->ckey[w] > k || (X->ckey[w] == k && X->cidx[w] < i)) { k = X->ckey[w]; i = X->cidx[w]; }
}

template <int NWARPS>
__device__ __forceinline__ int split_select(const SplitXch *X, bool use_bland) {
    if (use_bland) {
        int b = X->cbl[0];
#pragma unroll
        for (int w = 1; w < NWARPS; ++w) b = min(b, X->cbl[w]);
        return b == kNone ? -1 : b;
    }
    unsigned long long k;
    int e;
    split_combine_max<NWARPS>(X, k, e);
    if (e == kNone || k <= key_max(kTol)) return -1;
    return e;
}

// This thread's entry of column j (a column of this thread's half).
template <int R, int S, int NWR, int NCH, int ST>
__device__ __forceinline__ double split_at(const SplitState<R, S, NWR, NCH, ST> &St, const double *mytile, int c) {
    if (c < R) return reg_pick<R>(St.a, c);
    return mytile[(c - R) * ST];
}

// Both halves of row `row` store their register columns into rowbuf (the
// tile columns are read in place); the row's half-0 thread also its rhs.
template <int R, int S, int NWR, int NCH, int ST>
__device__ __forceinline__ void split_share_row(const SplitDims &D, const SplitState<R, S, NWR, NCH, ST> &St,
                                                unsigned char *smem, int row) {
    using C = SplitCfg<R, S, NWR, NCH, ST>;
    const bool mine = D.row == row;
    if ((row >> 5) == (D.warp % NWR)) {      // warp-uniform: the two warps holding the row
        const unsigned rb = (unsigned)__cvta_generic_to_shared(smem + C::ROWBUF) + 8u * (D.half * C::CPH);
#pragma unroll
        for (int c = 0; c < R; c += 2) st_shared_v2_if(mine, rb + 8u * c, St.a[c], St.a[c + 1]);
        if (mine && D.half == 0) reinterpret_cast<double *>(smem + C::ROWBUF)[C::COLS] = St.rhs;
    }
}

// Entry (row, column j) after split_share_row(row) and a barrier.
template <int R, int S, int NWR, int NCH, int ST>
__device__ __forceinline__ double split_row_entry(const unsigned char *smem, int row, int j) {
    using C = SplitCfg<R, S, NWR, NCH, ST>;
    const int h = j / C::CPH, c = j - h * C::CPH;
    return c < R ? reinterpret_cast<const double *>(smem + C::ROWBUF)[h * C::CPH + c]
                 : reinterpret_cast<const double *>(smem + C::TILE)[(size_t)h * S * ST + (size_t)(c - R) * ST + row];
}

// Rank-1 update of this thread's tile columns: col[c*ST] -= fs * r[c] (loads ahead of stores).
template <int S, int ST>
__device__ __forceinline__ void split_update_tile(double *col, const double *rv, double fs) {
    const unsigned ca = (unsigned)__cvta_generic_to_shared(col);
    const unsigned ra = (unsigned)__cvta_generic_to_shared(rv);
    double t[S], r[S];
#pragma unroll
    for (int c = 0; c < S; ++c) { r[c] = lds_f64(ra + 8u * c); t[c] = lds_f64(ca + 8u * ST * c); }
#pragma unroll
    for (int c = 0; c < S; ++c) sts_f64(ca + 8u * ST * c, __dsub_rn(t[c], __dmul_rn(fs, r[c])));
}

// Second half of a pivot, after barrier B: divisions + pricing of the
// transposed positions, candidates, barrier C, then the rank-1 update.
template <int R, int S, int NWR, int NCH, int ST, int KIND>
__device__ __forceinline__ void split_finish_pivot(const SplitDims &D, SplitState<R, S, NWR, NCH, ST> &St,
                                                   unsigned char *smem, SplitXch *X, int e, int l, double av) {
    using C = SplitCfg<R, S, NWR, NCH, ST>;
    double *tiles = reinterpret_cast<double *>(smem + C::TILE);
    double *rowbuf = reinterpret_cast<double *>(smem + C::ROWBUF);
    double *rvec = reinterpret_cast<double *>(smem + C::RVEC);
    const double pe = X->pe, fm = X->fm;
    const int oldvar = X->oldvar;
#pragma unroll
    for (int t = 0; t < C::OPW; ++t) {
        const int pos = split_pos<C::NT>(D, t);
        if (pos == 0) {
            const double r = div_entry(rowbuf[C::COLS], pe);
            rvec[C::COLS] = r;
            St.rc[t] = __dadd_rn(St.rc[t], __dmul_rn(fm, r));   // tableau.py:242
        } else if (pos < D.ncols) {
            const int j = pos - 1, h = j / C::CPH, c = j - h * C::CPH;
            double *src = c < R ? rowbuf + h * C::CPH + c : tiles + (size_t)h * S * ST + (size_t)(c - R) * ST + l;
            const double r = div_entry(*src, pe);
            rvec[j] = r;
            if (c >= R) *src = r;                            // row l of a tile column: final
            St.rc[t] = __dsub_rn(St.rc[t], __dmul_rn(fm, r));
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
    if (KIND != kWlpRestore) split_candidates<R, S, NWR, NCH, ST, KIND>(D, St, X);
    __syncthreads();  // C
    const bool mine = D.row == l;
    if (mine) St.basis_r = e;
    if (D.row < D.m) {                      // padding rows (>= m) stay as built
        const double2 *r2 = reinterpret_cast<const double2 *>(rvec + D.half * C::CPH);
#pragma unroll
        for (int c = 0; c < R; c += 2) {
            const double2 r = r2[c / 2];
            St.a[c] = __dsub_rn(St.a[c], __dmul_rn(av, r.x));
            St.a[c + 1] = __dsub_rn(St.a[c + 1], __dmul_rn(av, r.y));
        }
        split_update_tile<S, ST>(tiles + (size_t)D.half * S * ST + D.row, rvec + D.half * C::CPH + R, mine ? 0.0 : av);
        St.rhs = mine ? rvec[C::COLS] : __dsub_rn(St.rhs, __dmul_rn(av, rvec[C::COLS]));
    }
    if ((l >> 5) == (D.warp % NWR)) {       // warp-uniform: row l <- r (register columns)
        const unsigned rv = (unsigned)__cvta_generic_to_shared(rvec + D.half * C::CPH);
#pragma unroll
        for (int c = 0; c < R; c += 2) ld_shared_v2_if(mine, rv + 8u * c, St.a[c], St.a[c + 1]);
    }
}

// Pivot on column `col` (a structural/slack column; `neg`: the artificial
// paired with it, i.e. the negated column) at leaving row l: the owner half
// computes its entries, the other half reads them from fvec.  Ends after the
// update.  Entry: every thread knows col and (for run_phase) has already
// chosen l; here used by restore_objective, where l is given.
template <int R, int S, int NWR, int NCH, int ST>
__device__ __forceinline__ double split_column_entry(const SplitDims &D, const SplitState<R, S, NWR, NCH, ST> &St,
                                                     const unsigned char *smem, int col) {
    using C = SplitCfg<R, S, NWR, NCH, ST>;
    const double *mytile = reinterpret_cast<const double *>(smem + C::TILE) + (size_t)D.half * S * ST +
                           (D.row < ST ? D.row : 0);
    const int h = col / C::CPH;
    double av = 0.0;
    if (D.half == h) av = split_at<R, S, NWR, NCH, ST>(St, mytile, col - h * C::CPH);
    return av;
}

template <int R, int S, int NWR, int NCH, int ST, int KIND>
__device__ __forceinline__ WlpPhase split_run_phase(const SplitDims &D, SplitState<R, S, NWR, NCH, ST> &St,
                                                    unsigned char *smem, SplitXch *X, const Limits &lim) {
    using C = SplitCfg<R, S, NWR, NCH, ST>;
    const int *art_row = reinterpret_cast<const int *>(smem + C::ARTROW);
    double *fvec = reinterpret_cast<double *>(smem + C::FVEC);
    const int max_iter = lim.max_iterations > 0 ? lim.max_iterations : 50 * (D.m + D.n);
    const int trigger = lim.degenerate_limit >= 0 ? lim.degenerate_limit : (D.m > 1 ? D.m : 1);
    const unsigned long long kSent = key_max(kSentinel), kDeg = key_max(kDegenerateTol);
    int degenerate_run = 0;
    bool use_bland = false;
    for (int it = 0;; ++it) {
        if (it == max_iter) return {2, max_iter};
        const int e = split_select<C::NWARPS>(X, use_bland);
        if (e < 0) return {0, it};
        const bool art_e = e >= D.nvc;
        const int ecol = art_e ? D.n + art_row[e - D.nvc] : e;
        const int he = ecol / C::CPH;
        double av = 0.0;
        unsigned long long lk = kKeyEmptyMin;
        if (D.half == he) {                  // warp-uniform: the owner half
            av = split_column_entry<R, S, NWR, NCH, ST>(D, St, smem, ecol);
            if (art_e) av = -av;
            if (D.row >= D.m) av = 0.0;
            fvec[D.row] = av;
            const double ratio = ratio_entry(St.rhs, av);       // choose_leaving
            if (D.row < D.m) lk = key_min(ratio);
        }
        {
            const unsigned long long kw = warp_min_key(lk);
            const int lw = warp_index_of(lk, kw, D.row);
            if (D.lane == 0) { X->lkey[D.warp] = kw; X->lrow[D.warp] = lw; }
        }
        // the transposed holder of ecol publishes the entering reduced cost
#pragma unroll
        for (int t = 0; t < C::OPW; ++t)
            if (split_pos<C::NT>(D, t) == ecol + 1) X->fm = art_e ? St.arc[t] : St.rc[t];
        __syncthreads();  // A
        unsigned long long kmin = kKeyEmptyMin;
        int l = kNone;
#pragma unroll
        for (int w = 0; w < C::NWARPS; ++w)      // first minimum: lowest key, then lowest row
            if (X->lkey[w] < kmin || (X->lkey[w] == kmin && X->lrow[w] < l)) { kmin = X->lkey[w]; l = X->lrow[w]; }
        if (l == kNone || kmin >= kSent) return {1, it};   // unbounded (a NaN ratio keys to 0)
        if (kmin != 0ull && kmin <= kDeg) {                 // simplex.py:84-90
            ++degenerate_run;
            if (lim.anti_cycling && degenerate_run >= trigger) use_bland = true;
        } else {
            degenerate_run = 0;
            use_bland = false;
        }
        if (D.half != he) av = D.row < D.m ? fvec[D.row] : 0.0;
        split_share_row<R, S, NWR, NCH, ST>(D, St, smem, l);
        if (D.row == l && D.half == 0) { X->pe = av; X->oldvar = St.basis_r; }
        __syncthreads();  // B
        split_finish_pivot<R, S, NWR, NCH, ST, KIND>(D, St, smem, X, e, l, av);
    }
}

template <int R, int S, int NWR, int NCH, int ST, int PHASE>
__device__ __forceinline__ void split_price_out(const SplitDims &D, SplitState<R, S, NWR, NCH, ST> &St,
                                                unsigned char *smem, SplitXch *X, const double *cg) {
    using C = SplitCfg<R, S, NWR, NCH, ST>;
    double *cbv = reinterpret_cast<double *>(smem + C::CBV);
    const double *rowbuf = reinterpret_cast<const double *>(smem + C::ROWBUF);
    if (D.half == 0)
        cbv[D.row] = D.row < D.m ? (PHASE == 1 ? (St.basis_r >= D.nvc ? -1.0 : 0.0)
                                               : (St.basis_r < D.n ? cg[St.basis_r] : 0.0))
                                 : 0.0;
    double rc[C::OPW], ac[C::OPW];
#pragma unroll
    for (int t = 0; t < C::OPW; ++t) {
        const int pos = split_pos<C::NT>(D, t), j = pos - 1;
        rc[t] = (PHASE == 2 && pos >= 1 && j < D.n) ? cg[j] : 0.0;
        ac[t] = -1.0;
    }
    __syncthreads();
    for (int r = 0; r < D.m; ++r) {
        const double cb = cbv[r];
        if (cb == 0.0) continue;             // uniform across the CTA
        split_share_row<R, S, NWR, NCH, ST>(D, St, smem, r);
        __syncthreads();
#pragma unroll
        for (int t = 0; t < C::OPW; ++t) {
            const int pos = split_pos<C::NT>(D, t);
            if (pos == 0) {
                rc[t] = __dadd_rn(rc[t], __dmul_rn(cb, rowbuf[C::COLS]));
            } else if (pos < D.ncols) {
                const double v = split_row_entry<R, S, NWR, NCH, ST>(smem, r, pos - 1);
                rc[t] = __dsub_rn(rc[t], __dmul_rn(cb, v));
                if (PHASE == 1 && St.artk[t] >= 0) ac[t] = __dsub_rn(ac[t], __dmul_rn(cb, -v));
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int t = 0; t < C::OPW; ++t) {
        const int pos = split_pos<C::NT>(D, t);
        if (pos < D.ncols) {
            St.rc[t] = rc[t];
            if (PHASE == 1 && St.artk[t] >= 0) St.arc[t] = ac[t];
        }
    }
    split_candidates<R, S, NWR, NCH, ST, PHASE == 1 ? kWlpPhase1 : kWlpPhase2>(D, St, X);
    __syncthreads();
}

// restore_objective pivot-outs (simplex.py:109-126), uncounted.
template <int R, int S, int NWR, int NCH, int ST>
__device__ __forceinline__ void split_restore(const SplitDims &D, SplitState<R, S, NWR, NCH, ST> &St,
                                              unsigned char *smem, SplitXch *X) {
    using C = SplitCfg<R, S, NWR, NCH, ST>;
    int *basis_of = reinterpret_cast<int *>(smem + C::ARTOF);   // reused: basis per row during restore
    double *fvec = reinterpret_cast<double *>(smem + C::FVEC);
    const unsigned long long kRed = key_max(kRedundantTol);
    for (int row = 0; row < D.m; ++row) {
        if (D.half == 0) basis_of[D.row] = St.basis_r;
        __syncthreads();
        const bool art_basic = basis_of[row] >= D.nvc;
        __syncthreads();
        if (!art_basic) continue;           // uniform
        split_share_row<R, S, NWR, NCH, ST>(D, St, smem, row);
        __syncthreads();
        unsigned long long bk = kKeyEmptyMax;
        int bj = kNone;
#pragma unroll
        for (int t = 0; t < C::OPW; ++t) {
            const int pos = split_pos<C::NT>(D, t);
            if (pos >= 1 && pos < D.ncols) {
                const unsigned long long k = key_max(fabs(split_row_entry<R, S, NWR, NCH, ST>(smem, row, pos - 1)));
                if (k > bk) { bk = k; bj = pos - 1; }
            }
        }
        const unsigned long long kw = warp_max_key(bk);
        const int jw = warp_index_of(bk, kw, bj);
        if (D.lane == 0) { X->ckey[D.warp] = kw; X->cidx[D.warp] = jw; }
        __syncthreads();
        unsigned long long kb;
        int j;
        split_combine_max<C::NWARPS>(X, kb, j);
        // entries[j] > REDUNDANT_ROW_TOL; a NaN entry compares False in numpy
        if (j != kNone && kb > kRed && kb != ~0ull) {
            const int h = j / C::CPH;
            double av = 0.0;
            if (D.half == h) {
                av = split_column_entry<R, S, NWR, NCH, ST>(D, St, smem, j);
                if (D.row >= D.m) av = 0.0;
                fvec[D.row] = av;
            }
            __syncthreads();
            if (D.half != h) av = D.row < D.m ? fvec[D.row] : 0.0;
            if (D.row == row && D.half == 0) { X->pe = av; X->oldvar = St.basis_r; }
            X->fm = 0.0;
            __syncthreads();
            split_finish_pivot<R, S, NWR, NCH, ST, kWlpRestore>(D, St, smem, X, j, row, av);
        }
        __syncthreads();
    }
}

template <int R, int S, int NWR, int NCH, int ST>
__global__ void __launch_bounds__(32 * NWR * NCH, 1)
splitlp_kernel(Batch B) {
    using C = SplitCfg<R, S, NWR, NCH, ST>;
    extern __shared__ __align__(16) unsigned char smem[];
    SplitDims D;
    D.m = B.m; D.n = B.n; D.nvc = B.n + B.m; D.ncols = B.n + B.m + 1;
    D.tid = threadIdx.x; D.lane = threadIdx.x & 31; D.warp = threadIdx.x >> 5;
    D.row = 32 * (D.warp % NWR) + D.lane; D.half = D.warp / NWR;
    const int m = D.m, n = D.n, nvc = D.nvc;
    double *mytile = reinterpret_cast<double *>(smem + C::TILE) + (size_t)D.half * S * ST + D.row;
    int *art_row = reinterpret_cast<int *>(smem + C::ARTROW);
    int *art_of = reinterpret_cast<int *>(smem + C::ARTOF);
    SplitXch *X = reinterpret_cast<SplitXch *>(smem + C::XCH);
    __shared__ long long s_lp;
    {
        double *rvec = reinterpret_cast<double *>(smem + C::RVEC);
        for (int q = threadIdx.x; q < C::COLS + 2; q += C::NT) rvec[q] = 0.0;
    }
    SplitState<R, S, NWR, NCH, ST> St;
    for (;;) {
        if (threadIdx.x == 0) s_lp = atomicAdd(B.next_lp, 1);
        __syncthreads();
        if (s_lp >= batch_count(B)) break;    // the deferred LPs when launched after the lazy kernel
        const long long lp = batch_lp(B, s_lp);
        const double *Ag = B.shared_Ab ? B.A : B.A + (size_t)lp * m * n;
        const double *bg = B.shared_Ab ? B.b : B.b + (size_t)lp * m;
        const double *cg = B.c + (size_t)lp * n;

        // ---- build_tableau (tableau.py:139-172): thread (row, half) loads its half-row ----
        const bool live = D.row < m;
        const double bi = live ? bg[D.row] : 0.0;
        bool nonfinite = !isfinite(bi);
        const bool neg = live && bi < 0.0;
        const unsigned negmask = __ballot_sync(kFull, neg);
        if (D.lane == 0 && D.half == 0) X->nneg[D.warp] = __popc(negmask);
        __syncthreads();
        int before = __popc(negmask & ((1u << D.lane) - 1u));
        for (int w = 0; w < (D.warp % NWR); ++w) before += X->nneg[w];
        const double sgn = neg ? -1.0 : 1.0;
        const int my_art = neg ? before : -1;
        St.basis_r = neg ? nvc + my_art : n + D.row;
        St.rhs = live ? __dmul_rn(bi, sgn) : 0.0;
        if (D.half == 0) {
            art_of[D.row] = my_art;
            if (neg) art_row[my_art] = D.row;
        }
        const double *arow = Ag + (size_t)(live ? D.row : 0) * n;
        const int j0 = D.half * C::CPH;
#pragma unroll
        for (int c = 0; c < R; ++c) {
            const int j = j0 + c;
            double v = 0.0;
            if (live) {
                if (j < n) { const double a = arow[j]; nonfinite |= !isfinite(a); v = __dmul_rn(a, sgn); }
                else if (j < nvc) v = (j - n == D.row) ? sgn : 0.0;
            }
            St.a[c] = v;
        }
#pragma unroll
        for (int c = 0; c < S; ++c) {
            const int j = j0 + R + c;
            double v = 0.0;
            if (live) {
                if (j < n) { const double a = arow[j]; nonfinite |= !isfinite(a); v = __dmul_rn(a, sgn); }
                else if (j < nvc) v = (j - n == D.row) ? sgn : 0.0;
            }
            if (D.row < ST) mytile[c * ST] = v;
        }
        for (int j = threadIdx.x; j < n; j += C::NT) nonfinite |= !isfinite(cg[j]);
        const int n_art = __syncthreads_count(neg && D.half == 0);
        const bool invalid = __syncthreads_or(nonfinite);
        St.bas = 0;
#pragma unroll
        for (int t = 0; t < C::OPW; ++t) {
            const int pos = split_pos<C::NT>(D, t);
            const int j = pos - 1;
            St.rc[t] = (pos >= 1 && j < n) ? cg[j] : 0.0;
            St.arc[t] = 0.0;
            St.artk[t] = -1;
            if (j >= n && j < nvc) {
                const int k = art_of[j - n];
                St.artk[t] = k;
                St.bas |= (k < 0) ? (1u << t) : (0x10000u << t);
            }
        }
        __syncthreads();

        int8_t status = kOptimal;
        int it1 = 0, it2 = 0;
        bool done = false;
        if (invalid) {
            status = kInvalid;
            done = true;
        } else if (n_art > 0) {
            split_price_out<R, S, NWR, NCH, ST, 1>(D, St, smem, X, cg);                 // build_auxiliary
            const WlpPhase p1 = split_run_phase<R, S, NWR, NCH, ST, kWlpPhase1>(D, St, smem, X, B.lim);
            it1 = p1.iters;
            __syncthreads();
            if (threadIdx.x == 0) X->obj = St.rc[0];                            // position 0 = objective
            __syncthreads();
            const double obj = X->obj;
            __syncthreads();
            if (p1.state == 2) { status = kIterationLimit; done = true; }
            else if (p1.state == 1) { status = kErrPhase1Unbounded; done = true; }
            else if (fabs(obj) > kPhase1ZeroTol) { status = kInfeasible; done = true; }
            else {
                split_restore<R, S, NWR, NCH, ST>(D, St, smem, X);
                split_price_out<R, S, NWR, NCH, ST, 2>(D, St, smem, X, cg);
            }
        } else {
            split_candidates<R, S, NWR, NCH, ST, kWlpPhase2>(D, St, X);
            __syncthreads();
        }
        if (!done) {
            const WlpPhase p2 = split_run_phase<R, S, NWR, NCH, ST, kWlpPhase2>(D, St, smem, X, B.lim);
            it2 = p2.iters;
            if (p2.state == 2) status = kIterationLimit;
            else if (p2.state == 1) status = kUnbounded;
        }

        // ---- _extract_point (simplex.py:146-151) and c @ x ----
        __syncthreads();
        double *xs = reinterpret_cast<double *>(smem + C::RVEC);
        for (int j = threadIdx.x; j < n; j += C::NT) xs[j] = 0.0;
        __syncthreads();
        if (status == kOptimal && live && D.half == 0 && St.basis_r < n) xs[St.basis_r] = St.rhs;
        __syncthreads();
        double *xg = B.x + (size_t)lp * n;
        for (int j = threadIdx.x; j < n; j += C::NT) xg[j] = xs[j];
        if (threadIdx.x == 0) {
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
        __syncthreads();
        for (int q = threadIdx.x; q < C::COLS + 2; q += C::NT) xs[q] = 0.0;   // rvec padding reads as 0
        __syncthreads();
    }
}

}  // namespace blp
