// blp_pairlp_kernel.cuh -- one CTA of NWR row-warps per LP: NWR = 2 for
// 33..64 constraint rows (C4, the 64 x 32 support function: pairlp_*) and
// NWR = 4 for 65..128 (C3, 100 x 100: quadlp_*).
//
// The warplp2 layout (blp_warplp2_kernel.cuh) stretched over NWR warps by
// rows: thread r holds tableau row r; a row's positions [0, R) are
// registers, [R, R+S) live in a column-major shared tile tile[c][row] with an
// odd row stride ST >= m (conflict-free both along a column and along a row).
// The transposed objective row is dealt to the warps in 32-position blocks
// (position p -> warp (p/32)%NWR, lane p%32, slot p/(32 NWR)), so each lane
// divides and prices at most OPW positions per pivot.  Per pivot three CTA
// barriers separate: the per-warp leaving-row partials (A); the pivot
// element, the old basic variable and the register half of the pivot row
// published by the leaving row's lane (B); the pivot row r and the per-warp
// entering candidates (C).  (Publishing every warp's candidate row before A
// instead removes B but costs NWR x the row-transfer wavefronts: measured
// slower, C4 17.5 -> 18.5 ms.)  The row and column arithmetic is exactly the
// one-warp kernel's, so results are identical to it and to the reference.
#pragma once

#include "blp_common.cuh"
#include "blp_keys.cuh"
#include "blp_warplp_kernel.cuh"

namespace blp {

template <int R, int S, int NWR, int ST>
struct PairCfg {
    static constexpr int CPW = R + S;
    static constexpr int ROWS = 32 * NWR;
    static constexpr int OPW = (CPW + ROWS - 1) / ROWS;             // transposed slots per lane
    // ST (>= m, checked by the planner) is odd so that a row read across columns
    // (lane q -> tile[q][l], the pivot row's division) is bank-conflict free
    static_assert(ST <= ROWS + 1 && (ST & 1), "odd tile stride, at most one padding row");
    static constexpr size_t TILE = 0;                               // S x ST doubles, tile[c][row]
    static constexpr size_t ROWBUF = TILE + (size_t)S * ST * 8;     // R doubles
    static constexpr size_t RVEC = ROWBUF + (size_t)R * 8;          // CPW doubles
    static constexpr size_t CBV = RVEC + (size_t)((CPW + 1) & ~1) * 8;  // ROWS doubles
    static constexpr size_t ARTROW = CBV + (size_t)ROWS * 8;        // ROWS ints: row of artificial k
    static constexpr size_t ARTOF = ARTROW + (size_t)ROWS * 4;      // ROWS ints: artificial of row i
    static constexpr size_t XCH = ARTOF + (size_t)ROWS * 4;         // exchange slots
    static constexpr size_t BYTES = XCH + 256;
};

// Per-pivot exchange between the two warps.
struct PairXch {
    unsigned long long ckey[4];   // entering candidates per warp
    int cidx[4], cbl[4];
    unsigned long long lkey[4];   // leaving partials per warp
    int lrow[4];
    double pe, fm;
    int oldvar;
    int nneg[4];
};

template <int R, int S, int NWR, int ST>
struct PairState {
    static constexpr int OPW = PairCfg<R, S, NWR, ST>::OPW;
    double a[R];
    double rc[OPW], arc[OPW];
    int artk[OPW];
    unsigned bas;
    int basis_r;
};

struct PairDims { int m, n, nvc, ncols, lane, warp, row; };

template <int NWR>
__device__ __forceinline__ int pair_pos(const PairDims &D, int t) { return 32 * NWR * t + 32 * D.warp + D.lane; }

template <int R, int S, int NWR, int ST, int KIND>
__device__ __forceinline__ void pair_candidates(const PairDims &D, const PairState<R, S, NWR, ST> &St, PairXch *X) {
    unsigned long long ck = kKeyEmptyMax;
    int ci = kNone, cb = kNone;
#pragma unroll
    for (int t = 0; t < PairState<R, S, NWR, ST>::OPW; ++t) {
        const int pos = pair_pos<NWR>(D, t);
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

// Combine per-warp (max key, lowest index) partials.
template <int NWR>
__device__ __forceinline__ void pair_combine_max(const unsigned long long *keys, const int *idx,
                                                 unsigned long long &k, int &i) {
    k = keys[0];
    i = idx[0];
#pragma unroll
    for (int w = 1; w < NWR; ++w)
        if (keys[w] > k || (keys[w] == k && idx[w] < i)) { k = keys[w]; i = idx[w]; }
}

// choose_entering / choose_entering_bland from the warps' partials (after a barrier).
template <int NWR>
__device__ __forceinline__ int pair_select(const PairXch *X, bool use_bland) {
    if (use_bland) {
        int b = X->cbl[0];
#pragma unroll
        for (int w = 1; w < NWR; ++w) b = min(b, X->cbl[w]);
        return b == kNone ? -1 : b;
    }
    unsigned long long k;
    int e;
    pair_combine_max<NWR>(X->ckey, X->cidx, k, e);
    if (e == kNone || k <= key_max(kTol)) return -1;
    return e;
}

template <int R, int S, int NWR, int ST>
__device__ __forceinline__ double pair_at(const PairState<R, S, NWR, ST> &St, const double *mycol, int pos) {
    if (pos < R) return reg_pick<R>(St.a, pos);
    return mycol[(pos - R) * ST];
}

// Rank-1 update of this row's shared-tile columns: col[c*ST] -= fs * r[R + c].
// The tile and the pivot row share one smem array, so the compiler cannot move
// a load above an earlier store; the loop is software-pipelined by hand: batch
// b+1 (K columns and their pivot-row entries) is loaded before batch b stores.
// Zero-skipping form (the two-warp C4 kernel, where it measures 16.6 -> 15.3 ms
// per 2e5 directions; the four-warp C3 kernel and warplp2 are faster without):
// a batch whose pivot-row entries are all zero leaves its columns unchanged
// (a - f*0 == a; the slack part of a pivot row stays sparse for many pivots),
// so its column loads and stores are skipped.  The test is warp-uniform;
// batches are not pipelined (the branch would split the pipeline's live ranges).
template <int R, int S, int ST, int K = 4>
__device__ __forceinline__ void pair_update_tile_skip0(double *col, const double *rvec, double fs) {
    const unsigned ca = (unsigned)__cvta_generic_to_shared(col);
    const unsigned ra = (unsigned)__cvta_generic_to_shared(rvec + R);
#pragma unroll
    for (int c0 = 0; c0 < S; c0 += K) {
        double r[K], t[K];
        bool any = false;
#pragma unroll
        for (int k = 0; k < K; k += 2) {
            if (c0 + k < S) {
                lds_v2_f64(ra + 8u * (c0 + k), r[k], r[k + 1]);
                any |= r[k] != 0.0 || (c0 + k + 1 < S && r[k + 1] != 0.0);
            }
        }
        if (!any) continue;
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (c0 + k < S) t[k] = lds_f64(ca + 8u * ST * (c0 + k));
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (c0 + k < S) sts_f64(ca + 8u * ST * (c0 + k), __dsub_rn(t[k], __dmul_rn(fs, r[k])));
    }
}

template <int R, int S, int ST, int K = 4>
__device__ __forceinline__ void pair_update_tile(double *col, const double *rvec, double fs) {
    constexpr int NB = (S + K - 1) / K;
    const unsigned ca = (unsigned)__cvta_generic_to_shared(col);
    const unsigned ra = (unsigned)__cvta_generic_to_shared(rvec + R);
    double t[2][K], r[2][K];
    auto load = [&](int b, int s) {
#pragma unroll
        for (int k = 0; k < K; k += 2) {
            const int c = b * K + k;
            if (c < S) {
                lds_v2_f64(ra + 8u * c, r[s][k], r[s][k + 1]);
                t[s][k] = lds_f64(ca + 8u * ST * c);
                if (c + 1 < S) t[s][k + 1] = lds_f64(ca + 8u * ST * (c + 1));
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
            if (c < S) sts_f64(ca + 8u * ST * c, __dsub_rn(t[b & 1][k], __dmul_rn(fs, r[b & 1][k])));
        }
    }
}
// Second half of a pivot, after barrier B: divisions + pricing of the
// transposed positions, candidates, barrier C, then the rank-1 update.
// l = leaving row, av = this lane's entry of the entering column.
template <int R, int S, int NWR, int ST, int KIND>
__device__ __forceinline__ void pair_finish_pivot(const PairDims &D, PairState<R, S, NWR, ST> &St, unsigned char *smem,
                                                  PairXch *X, int e, int l, double av) {
    using C = PairCfg<R, S, NWR, ST>;
    double *tiles = reinterpret_cast<double *>(smem + C::TILE);
    double *rowbuf = reinterpret_cast<double *>(smem + C::ROWBUF);
    double *rvec = reinterpret_cast<double *>(smem + C::RVEC);
    const double pe = X->pe, fm = X->fm;
    const int oldvar = X->oldvar;
    double *lcol = tiles + l;                               // row l of the tile
#pragma unroll
    for (int t = 0; t < PairState<R, S, NWR, ST>::OPW; ++t) {
        const int pos = pair_pos<NWR>(D, t);
        if (pos < D.ncols) {
            double *src = pos < R ? rowbuf + pos : lcol + (pos - R) * ST;
            const double r = div_entry(*src, pe);
            rvec[pos] = r;
            if (pos >= R) *src = r;                         // row l of an smem column: final
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
    if (KIND != kWlpRestore) pair_candidates<R, S, NWR, ST, KIND>(D, St, X);
    __syncthreads();  // C
    const bool mine = D.row == l;
    if (mine) St.basis_r = e;
    if (D.row < D.m) {                      // padding rows (>= m) stay as built: no smem traffic
#pragma unroll
        for (int c = 0; c < R; c += 2) {
            const double2 r2 = reinterpret_cast<const double2 *>(rvec)[c / 2];
            St.a[c] = __dsub_rn(St.a[c], __dmul_rn(av, r2.x));
            St.a[c + 1] = __dsub_rn(St.a[c + 1], __dmul_rn(av, r2.y));
        }
        const double fs = mine ? 0.0 : av;  // row l of the smem columns already holds r
        if constexpr (NWR == 2) pair_update_tile_skip0<R, S, ST>(tiles + D.row, rvec, fs);
        else pair_update_tile<R, S, ST>(tiles + D.row, rvec, fs);
    }
    if ((l >> 5) == D.warp) {               // warp-uniform: only the leaving row's warp issues the reload
        const unsigned rv = (unsigned)__cvta_generic_to_shared(rvec);
#pragma unroll
        for (int c = 0; c < R; c += 2) ld_shared_v2_if(mine, rv + 8u * c, St.a[c], St.a[c + 1]);
    }
}

// The leaving row's lane publishes pe, oldvar and its register half (before barrier B).
template <int R, int S, int NWR, int ST>
__device__ __forceinline__ void pair_publish_row(const PairDims &D, const PairState<R, S, NWR, ST> &St, unsigned char *smem,
                                                 PairXch *X, int l, double av, bool with_pe) {
    const bool mine = D.row == l;
    const unsigned rb = (unsigned)__cvta_generic_to_shared(smem + PairCfg<R, S, NWR, ST>::ROWBUF);
    if ((l >> 5) == D.warp) {               // warp-uniform: the other warps issue no (empty) stores
#pragma unroll
        for (int c = 0; c < R; c += 2) st_shared_v2_if(mine, rb + 8u * c, St.a[c], St.a[c + 1]);
    }
    if (mine) {
        if (with_pe) X->pe = av;
        X->oldvar = St.basis_r;
    }
}

template <int R, int S, int NWR, int ST, int KIND>
__device__ __forceinline__ WlpPhase pair_run_phase(const PairDims &D, PairState<R, S, NWR, ST> &St, unsigned char *smem,
                                                   PairXch *X, const Limits &lim) {
    using C = PairCfg<R, S, NWR, ST>;
    const double *mycol = reinterpret_cast<const double *>(smem + C::TILE) + (D.row < ST ? D.row : 0);
    const int *art_row = reinterpret_cast<const int *>(smem + C::ARTROW);
    const int max_iter = lim.max_iterations > 0 ? lim.max_iterations : 50 * (D.m + D.n);
    const int trigger = lim.degenerate_limit >= 0 ? lim.degenerate_limit : (D.m > 1 ? D.m : 1);
    const unsigned long long kSent = key_max(kSentinel), kDeg = key_max(kDegenerateTol);
    int degenerate_run = 0;
    bool use_bland = false;
    for (int it = 0;; ++it) {
        if (it == max_iter) return {2, max_iter};
        const int e = pair_select<NWR>(X, use_bland);
        if (e < 0) return {0, it};
        const bool art_e = e >= D.nvc;
        const int epos = art_e ? 1 + D.n + art_row[e - D.nvc] : e + 1;
        double av = pair_at<R, S, NWR, ST>(St, mycol, epos);
        if (art_e) av = -av;
        if (D.row >= D.m) av = 0.0;
        unsigned long long lk = kKeyEmptyMin;                                // choose_leaving
        const double ratio = ratio_entry(St.a[0], av);
        if (D.row < D.m) lk = key_min(ratio);
        const unsigned long long kw = warp_min_key(lk);
        const int lw = warp_index_of(lk, kw, D.row);
        if (D.lane == 0) { X->lkey[D.warp] = kw; X->lrow[D.warp] = lw; }
        // the transposed holder of epos publishes the entering reduced cost
#pragma unroll
        for (int t = 0; t < PairState<R, S, NWR, ST>::OPW; ++t)
            if (pair_pos<NWR>(D, t) == epos) X->fm = art_e ? St.arc[t] : St.rc[t];
        __syncthreads();  // A
        unsigned long long kmin = X->lkey[0];
        int l = X->lrow[0];
#pragma unroll
        for (int w = 1; w < NWR; ++w)             // rows ascend with the warp: first minimum wins
            if (X->lkey[w] < kmin) { kmin = X->lkey[w]; l = X->lrow[w]; }
        if (l == kNone || kmin >= kSent) return {1, it};   // unbounded (a NaN ratio keys to 0)
        if (kmin != 0ull && kmin <= kDeg) {                   // simplex.py:84-90
            ++degenerate_run;
            if (lim.anti_cycling && degenerate_run >= trigger) use_bland = true;
        } else {
            degenerate_run = 0;
            use_bland = false;
        }
        pair_publish_row<R, S, NWR, ST>(D, St, smem, X, l, av, true);
        __syncthreads();  // B
        pair_finish_pivot<R, S, NWR, ST, KIND>(D, St, smem, X, e, l, av);
    }
}

// Row `row` shared for column scans: register half into rowbuf; entries read
// back as rowbuf[p] (p < R) or the row's warp tile.
template <int R, int S, int NWR, int ST>
__device__ __forceinline__ double pair_row_entry(unsigned char *smem, int row, int pos) {
    using C = PairCfg<R, S, NWR, ST>;
    return pos < R ? reinterpret_cast<const double *>(smem + C::ROWBUF)[pos]
                   : reinterpret_cast<const double *>(smem + C::TILE)[(size_t)(pos - R) * ST + row];
}

template <int R, int S, int NWR, int ST, int PHASE>
__device__ __forceinline__ void pair_price_out(const PairDims &D, PairState<R, S, NWR, ST> &St, unsigned char *smem,
                                               PairXch *X, const double *cg) {
    using C = PairCfg<R, S, NWR, ST>;
    double *cbv = reinterpret_cast<double *>(smem + C::CBV);
    const unsigned rb = (unsigned)__cvta_generic_to_shared(smem + C::ROWBUF);
    cbv[D.row] = D.row < D.m ? (PHASE == 1 ? (St.basis_r >= D.nvc ? -1.0 : 0.0)
                                           : (St.basis_r < D.n ? cg[St.basis_r] : 0.0))
                             : 0.0;
    double rc[PairState<R, S, NWR, ST>::OPW], ac[PairState<R, S, NWR, ST>::OPW];
#pragma unroll
    for (int t = 0; t < PairState<R, S, NWR, ST>::OPW; ++t) {
        const int pos = pair_pos<NWR>(D, t), j = pos - 1;
        rc[t] = (PHASE == 2 && pos >= 1 && j < D.n) ? cg[j] : 0.0;
        ac[t] = -1.0;
    }
    __syncthreads();
    for (int r = 0; r < D.m; ++r) {
        const double cb = cbv[r];
        if (cb == 0.0) continue;           // uniform across the CTA
        if ((r >> 5) == D.warp) {
#pragma unroll
            for (int c = 0; c < R; c += 2) st_shared_v2_if(D.row == r, rb + 8u * c, St.a[c], St.a[c + 1]);
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < PairState<R, S, NWR, ST>::OPW; ++t) {
            const int pos = pair_pos<NWR>(D, t);
            if (pos < D.ncols) {
                const double v = pair_row_entry<R, S, NWR, ST>(smem, r, pos);
                if (pos == 0) {
                    rc[t] = __dadd_rn(rc[t], __dmul_rn(cb, v));
                } else {
                    rc[t] = __dsub_rn(rc[t], __dmul_rn(cb, v));
                    if (PHASE == 1 && St.artk[t] >= 0) ac[t] = __dsub_rn(ac[t], __dmul_rn(cb, -v));
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int t = 0; t < PairState<R, S, NWR, ST>::OPW; ++t) {
        const int pos = pair_pos<NWR>(D, t);
        if (pos < D.ncols) {
            St.rc[t] = rc[t];
            if (PHASE == 1 && St.artk[t] >= 0) St.arc[t] = ac[t];
        }
    }
    pair_candidates<R, S, NWR, ST, PHASE == 1 ? kWlpPhase1 : kWlpPhase2>(D, St, X);
    __syncthreads();
}

// restore_objective pivot-outs (simplex.py:109-126), uncounted.
template <int R, int S, int NWR, int ST>
__device__ __forceinline__ void pair_restore(const PairDims &D, PairState<R, S, NWR, ST> &St, unsigned char *smem,
                                             PairXch *X) {
    using C = PairCfg<R, S, NWR, ST>;
    const double *mycol = reinterpret_cast<const double *>(smem + C::TILE) + (D.row < ST ? D.row : 0);
    int *basis_of = reinterpret_cast<int *>(smem + C::ARTOF);   // reused: basis per row during restore
    const unsigned long long kRed = key_max(kRedundantTol);
    for (int row = 0; row < D.m; ++row) {
        basis_of[D.row] = St.basis_r;
        __syncthreads();
        const bool art_basic = basis_of[row] >= D.nvc;
        __syncthreads();
        if (!art_basic) continue;           // uniform
        pair_publish_row<R, S, NWR, ST>(D, St, smem, X, row, 0.0, false);
        __syncthreads();
        unsigned long long bk = kKeyEmptyMax;
        int bj = kNone;
#pragma unroll
        for (int t = 0; t < PairState<R, S, NWR, ST>::OPW; ++t) {
            const int pos = pair_pos<NWR>(D, t);
            if (pos >= 1 && pos < D.ncols) {
                const unsigned long long k = key_max(fabs(pair_row_entry<R, S, NWR, ST>(smem, row, pos)));
                if (k > bk) { bk = k; bj = pos - 1; }
            }
        }
        const unsigned long long kw = warp_max_key(bk);
        const int jw = warp_index_of(bk, kw, bj);
        if (D.lane == 0) { X->ckey[D.warp] = kw; X->cidx[D.warp] = jw; }
        __syncthreads();
        unsigned long long kb;
        int j;
        pair_combine_max<NWR>(X->ckey, X->cidx, kb, j);
        // entries[j] > REDUNDANT_ROW_TOL; a NaN entry compares False in numpy
        if (j != kNone && kb > kRed && kb != ~0ull) {
            double av = pair_at<R, S, NWR, ST>(St, mycol, j + 1);
            if (D.row >= D.m) av = 0.0;
            if (D.row == row) X->pe = av;
            X->fm = 0.0;
            __syncthreads();
            pair_finish_pivot<R, S, NWR, ST, kWlpRestore>(D, St, smem, X, j, row, av);
        }
        __syncthreads();
    }
}

template <int R, int S, int NWR, int ST, int kMinBlocks>
__global__ void __launch_bounds__(32 * NWR, kMinBlocks)
pairlp_kernel(Batch B) {
    using C = PairCfg<R, S, NWR, ST>;
    extern __shared__ __align__(16) unsigned char smem[];
    PairDims D;
    D.m = B.m; D.n = B.n; D.nvc = B.n + B.m; D.ncols = B.n + B.m + 1;
    D.lane = threadIdx.x & 31; D.warp = threadIdx.x >> 5; D.row = threadIdx.x;
    const int m = D.m, n = D.n, nvc = D.nvc;
    double *tile = reinterpret_cast<double *>(smem + C::TILE) + D.row;
    int *art_row = reinterpret_cast<int *>(smem + C::ARTROW);
    int *art_of = reinterpret_cast<int *>(smem + C::ARTOF);
    PairXch *X = reinterpret_cast<PairXch *>(smem + C::XCH);
    __shared__ long long s_lp;
    {
        double *rvec = reinterpret_cast<double *>(smem + C::RVEC);
        for (int q = threadIdx.x; q < C::CPW; q += 32 * NWR) rvec[q] = 0.0;
    }
    PairState<R, S, NWR, ST> St;
    for (;;) {
        if (threadIdx.x == 0) s_lp = atomicAdd(B.next_lp, 1);
        __syncthreads();
        if (s_lp >= batch_count(B)) break;    // the deferred LPs when launched after the lazy kernel
        const long long lp = batch_lp(B, s_lp);
        const double *Ag = B.shared_Ab ? B.A : B.A + (size_t)lp * m * n;
        const double *bg = B.shared_Ab ? B.b : B.b + (size_t)lp * m;
        const double *cg = B.c + (size_t)lp * n;

        // ---- build_tableau (tableau.py:139-172): row r loaded by its own lane ----
        const bool live = D.row < m;
        const double bi = live ? bg[D.row] : 0.0;
        bool nonfinite = !isfinite(bi);
        const bool neg = live && bi < 0.0;
        const unsigned negmask = __ballot_sync(kFull, neg);
        if (D.lane == 0) X->nneg[D.warp] = __popc(negmask);
        __syncthreads();
        int before = __popc(negmask & ((1u << D.lane) - 1u));
        for (int w = 0; w < D.warp; ++w) before += X->nneg[w];
        const double sgn = neg ? -1.0 : 1.0;
        const int my_art = neg ? before : -1;
        St.basis_r = neg ? nvc + my_art : n + D.row;
        art_of[D.row] = my_art;
        if (neg) art_row[my_art] = D.row;
        const double *arow = Ag + (size_t)(live ? D.row : 0) * n;
#pragma unroll
        for (int p = 0; p < R; ++p) {
            const int j = p - 1;
            double v = 0.0;
            if (live) {
                if (p == 0) v = __dmul_rn(bi, sgn);
                else if (j < n) { const double a = arow[j]; nonfinite |= !isfinite(a); v = __dmul_rn(a, sgn); }
                else if (j < nvc) v = (j - n == D.row) ? sgn : 0.0;
            }
            St.a[p] = v;
        }
#pragma unroll 4
        for (int c = 0; c < S; ++c) {
            const int j = R + c - 1;
            double v = 0.0;
            if (live) {
                if (j < n) { const double a = arow[j]; nonfinite |= !isfinite(a); v = __dmul_rn(a, sgn); }
                else if (j < nvc) v = (j - n == D.row) ? sgn : 0.0;
            }
            if (D.row < ST) tile[c * ST] = v;
        }
        for (int j = threadIdx.x; j < n; j += 32 * NWR) nonfinite |= !isfinite(cg[j]);
        const int n_art = __syncthreads_count(neg);
        const bool invalid = __syncthreads_or(nonfinite);
        St.bas = 0;
#pragma unroll
        for (int t = 0; t < C::OPW; ++t) {
            const int pos = pair_pos<NWR>(D, t);
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
            pair_price_out<R, S, NWR, ST, 1>(D, St, smem, X, cg);                  // build_auxiliary
            const WlpPhase p1 = pair_run_phase<R, S, NWR, ST, kWlpPhase1>(D, St, smem, X, B.lim);
            it1 = p1.iters;
            __syncthreads();
            double *objx = reinterpret_cast<double *>(smem + C::CBV);
            if (threadIdx.x == 0) objx[0] = St.rc[0];                      // position 0 = objective
            __syncthreads();
            const double obj = objx[0];
            __syncthreads();
            if (p1.state == 2) { status = kIterationLimit; done = true; }
            else if (p1.state == 1) { status = kErrPhase1Unbounded; done = true; }
            else if (fabs(obj) > kPhase1ZeroTol) { status = kInfeasible; done = true; }
            else {
                pair_restore<R, S, NWR, ST>(D, St, smem, X);
                pair_price_out<R, S, NWR, ST, 2>(D, St, smem, X, cg);
            }
        } else {
            pair_candidates<R, S, NWR, ST, kWlpPhase2>(D, St, X);
            __syncthreads();
        }
        if (!done) {
            const WlpPhase p2 = pair_run_phase<R, S, NWR, ST, kWlpPhase2>(D, St, smem, X, B.lim);
            it2 = p2.iters;
            if (p2.state == 2) status = kIterationLimit;
            else if (p2.state == 1) status = kUnbounded;
        }

        // ---- _extract_point (simplex.py:146-151) and c @ x ----
        __syncthreads();
        double *xs = reinterpret_cast<double *>(smem + C::RVEC);
        for (int j = threadIdx.x; j < n; j += 32 * NWR) xs[j] = 0.0;
        __syncthreads();
        if (status == kOptimal && live && St.basis_r < n) xs[St.basis_r] = St.a[0];
        __syncthreads();
        double *xg = B.x + (size_t)lp * n;
        for (int j = threadIdx.x; j < n; j += 32 * NWR) xg[j] = xs[j];
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
        for (int q = threadIdx.x; q < C::CPW; q += 32 * NWR) xs[q] = 0.0;   // rvec padding reads as 0
        __syncthreads();
    }
}

}  // namespace blp
