// blp_cmulti_kernel.cuh -- the condensed tableau (blp_condensed_kernel.cuh) on one
// CTA of NWR row-warps per LP, for 33..256 constraint rows (C4 64 x 32: NWR = 2; C3,
// 100 x 100: NWR = 4; 129..256 rows: NWR = 8, one LP per SM).
//
// Same exactness argument as the one-warp kernel: only the n nonbasic columns and
// the rhs are stored and updated -- a basic column is exactly e_r and the reference
// rewrites it without changing a value -- so a pivot touches (m+1) x (n+1) cells
// instead of the reference's (m+1) x (n+m+n_art+1), and the artificial/slack pair
// bookkeeping (states A/B/C, trivial members) is the one-warp kernel's.
//
// Layout: thread t holds constraint row t (rows >= m are padding): slots [0, R) in
// registers, [R, R+S) in a shared tile of column pairs (tix) with an odd row
// stride ST >= m, and its rhs; the transposed objective row is dealt one slot per
// thread (slot q -> thread q: its reduced cost, variable and partner).  Per pivot
// three CTA barriers separate (A) the per-warp leaving-row partials and the
// entering reduced cost, (B) the leaving row's register half, pivot element and
// bookkeeping, published by its thread, and (C) the pivot row r = row_l / pe, the
// reduced-cost update and the per-warp entering candidates of the next pivot; then
// every row applies a - f*r to its registers and tile columns.
//
// Where the C3 time goes (vs the dense quadlp kernel): quadlp keeps 106 of each
// row's 201 positions in the shared tile, so the update is bound by the shared-
// memory pipe (~2,000 wavefronts per LP-pivot); here a row is 101 cells, at most
// 2 x S of them through shared memory, so the update is register/FP64 work.
#pragma once

#include "blp_common.cuh"
#include "blp_condensed_kernel.cuh"
#include "blp_keys.cuh"

namespace blp {

template <int NWR, int R, int S, int ST>
struct CmCfg {
    static_assert(NWR == 2 || NWR == 4 || NWR == 8 || NWR == 16, "row-warps per LP");
    static constexpr int NS = R + S;                 // nonbasic slots per row
    static constexpr int ROWS = 32 * NWR;
    static_assert(NS <= ROWS, "one transposed slot per thread");
    static_assert(S == 0 || ((ST & 1) && ST <= ROWS + 1), "odd tile stride, at most one padding row");
    static_assert(R % 2 == 0, "register half in double2 pairs");
    static_assert(S % 2 == 0, "tile slots in column pairs");
    static constexpr size_t TILE = 0;                                  // S x ST doubles, column pairs (tix)
    static constexpr size_t ROWBUF = TILE + (size_t)S * ST * 8;        // 2 x R doubles (double-buffered)
    static constexpr size_t RVEC = ROWBUF + (size_t)2 * R * 8;         // NS (even) doubles
    static constexpr size_t CBV = RVEC + (size_t)((NS + 1) & ~1) * 8;  // ROWS doubles
    static constexpr size_t RHSV = CBV + (size_t)ROWS * 8;             // ROWS doubles
    static constexpr size_t FLAG = RHSV + (size_t)ROWS * 8;            // ROWS ints
    static constexpr size_t XCH = FLAG + (size_t)ROWS * 4;
    static constexpr size_t BYTES = XCH + 768;
};

// Per-pivot exchange between the warps (768 bytes reserved).
struct CmXch {
    unsigned long long ckey[16];   // entering candidates per warp (Dantzig key, composite id)
    int cid[16];
    int cbl[16];                   // Bland: lowest composite id with rc > tol
    unsigned long long lkey[16];   // leaving partials per warp
    int lrow[16];
    int nneg[16];                  // negated rows per warp (artificial numbering)
    int nonfinite;
    long long lp;                  // the LP the CTA solves next
    double pe, fm, rr, oldprc, newtriv_rc;
    int oldvar, oldpart, newtriv;
};

template <int R>
struct CmState {
    double a[R];        // row tid: register slots
    double rhs, prc;
    int basis, ppart;   // basic variable of the row; its pair's trivial member (or -1)
    double rc, rcp;     // transposed: slot tid's reduced cost and its partner's
    int svar, spart;
    double obj;         // objective cell (the same in every thread)
};

struct CmDims { int m, n, nvc, lane, warp, row; };

// Composite candidate id: variable in the high bits (lowest id among equal keys = numpy's
// first index), kind and slot in the low 10 (slots up to 255).
__device__ __forceinline__ int cm_cid(int var, int kind, int q) { return (var << 10) | (kind << 8) | q; }
__device__ __forceinline__ int cm_kind(int cid) { return (cid >> 8) & 3; }

// Tile layout: column pairs, row-major within a pair -- slot c of row r at
// ((c/2) * ST + r) * 2 + c%2 -- so a row's update moves 16 bytes per access (LDS.128 /
// STS.128, a warp's 32 rows contiguous: conflict-free) and a column read down the rows
// (the build, a single slot) stays a plain 8-byte access.
template <int ST>
__device__ __forceinline__ size_t tix(int c, int row) { return ((size_t)(c >> 1) * ST + row) * 2 + (c & 1); }

template <int NWR, int R, int S, int ST>
__device__ __forceinline__ double cm_slot(const CmState<R> &St, const double *tile, int row, int s) {
    if (s < R) return reg_pick<R>(St.a, s);
    return tile[tix<ST>(s - R, row)];
}

__device__ __forceinline__ void sts_v2_f64(unsigned addr, double x, double y) {
    asm volatile("st.volatile.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(x), "d"(y) : "memory");
}

// Rank-1 update of this row's tile slots, col pairs p: t -= fs * r, software-pipelined by hand
// (the tile and rvec share the shared-memory array, so the compiler would serialise each
// load behind the previous store): pair p+1 and its pivot-row entries load before pair p stores.
// CM_TILE_DEPTH: column pairs loaded ahead of the one being updated.  The tile loop's stalls
// are mostly shared-memory results (C3 source page: 50-64% short_sb), but deeper prefetch
// measured no better (bench-style steps, ms, depth 1 / 2 / 3): C3 2e4 71.9, 71.5 / 71.8,
// 71.3 / 71.3, 71.4; C4 1e6 37.19 / 38.14 / 38.20; afiro 150 x 150 (cm8) 57.9 / 59.6 / 60.6.
#ifndef CM_TILE_DEPTH
#define CM_TILE_DEPTH 1
#endif
template <int R, int S, int ST>
__device__ __forceinline__ void cm_update_tile(double *tile, int row, const double *rvec, double fs) {
    constexpr int NP = S / 2, DP = CM_TILE_DEPTH, NB = DP + 1;
    const unsigned ta = (unsigned)__cvta_generic_to_shared(tile) + 16u * row;
    const unsigned ra = (unsigned)__cvta_generic_to_shared(rvec + R);
    double t[NB][2], r[NB][2];
#pragma unroll
    for (int p = 0; p < DP && p < NP; ++p) {
        lds_v2_f64(ta + 16u * ST * p, t[p][0], t[p][1]);
        lds_v2_f64(ra + 16u * p, r[p][0], r[p][1]);
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int b = p % NB;
        if (p + DP < NP) {
            const int bn = (p + DP) % NB;
            lds_v2_f64(ta + 16u * ST * (p + DP), t[bn][0], t[bn][1]);
            lds_v2_f64(ra + 16u * (p + DP), r[bn][0], r[bn][1]);
        }
        sts_v2_f64(ta + 16u * ST * p, __dsub_rn(t[b][0], __dmul_rn(fs, r[b][0])),
                   __dsub_rn(t[b][1], __dmul_rn(fs, r[b][1])));
    }
}

// Entering candidates of this thread (its slot, its slot's partner, its row's trivial
// member) reduced per warp into X (choose_entering, Dantzig, and the Bland minimum).
// skip_row_triv: the row's trivial member is stale (this row just left; the slot
// holder that knows the new one passes it as extra_triv).
template <int NWR, int R, bool PH1>
__device__ __forceinline__ void cm_candidates(const CmDims &D, const CmState<R> &St, CmXch *X, bool skip_row_triv,
                                              int extra_triv, double extra_rc) {
    unsigned long long ck = kKeyEmptyMax;
    int ci = kNone, cb = kNone;
    auto consider = [&](double v, int id) {
        const unsigned long long k = key_max(v);
        if (k > ck || (k == ck && id < ci)) { ck = k; ci = id; }
        if (v > kTol && id < cb) cb = id;
    };
    const int q = D.row;
    if (q < D.n) {
        if (PH1 || St.svar < D.nvc) consider(St.rc, cm_cid(St.svar, kCtSlot, q));
        if (St.spart >= 0 && (PH1 || St.spart < D.nvc)) consider(St.rcp, cm_cid(St.spart, kCtPartner, q));
    }
    if (!skip_row_triv && D.row < D.m && St.ppart >= 0 && (PH1 || St.ppart < D.nvc))
        consider(St.prc, cm_cid(St.ppart, kCtTrivial, 0));
    if (extra_triv >= 0 && (PH1 || extra_triv < D.nvc)) consider(extra_rc, cm_cid(extra_triv, kCtTrivial, 0));
    const unsigned long long kw = warp_max_key(ck);
    const int iw = warp_index_of(ck, kw, ci);
    const int bw = (int)__reduce_min_sync(kFull, (unsigned)cb);
    if (D.lane == 0) { X->ckey[D.warp] = kw; X->cid[D.warp] = iw; X->cbl[D.warp] = bw; }
}

template <int NWR>
__device__ __forceinline__ int cm_select(const CmXch *X, bool use_bland) {
    if (use_bland) {
        int b = X->cbl[0];
#pragma unroll
        for (int w = 1; w < NWR; ++w) b = min(b, X->cbl[w]);
        return b;
    }
    unsigned long long k = X->ckey[0];
    int i = X->cid[0];
#pragma unroll
    for (int w = 1; w < NWR; ++w)
        if (X->ckey[w] > k || (X->ckey[w] == k && X->cid[w] < i)) { k = X->ckey[w]; i = X->cid[w]; }
    return (i == kNone || k <= key_max(kTol)) ? kNone : i;
}

// The register half of row `row` into rowbuf (its thread; warp-uniform guard so the
// other warps issue nothing).
template <int NWR, int R>
__device__ __forceinline__ void cm_publish_regs(const CmDims &D, const CmState<R> &St, double *rowbuf, int row) {
    if ((row >> 5) == D.warp) {
        const unsigned rb = (unsigned)__cvta_generic_to_shared(rowbuf);
        const bool mine = D.row == row;
#pragma unroll
        for (int c = 0; c < R; c += 2) st_shared_v2_if(mine, rb + 8u * c, St.a[c], St.a[c + 1]);
    }
}

// pivot (tableau.py:218-244) on the condensed tableau, after the leaving row l is known
// to every thread: e enters from slot s (its negated partner if `partner`); av = this
// row's entry of the entering column.  The leaving row's thread passes pe and rr (the
// winning ratio, rhs_l / pe) through X.  fm = the entering reduced cost (0 for restore
// pivots, whose objective row is rebuilt by the price-out that follows).  With CAND the
// next pivot's entering candidates are left in X (valid after the final barrier).
template <int NWR, int R, int S, int ST, bool PH1, bool CAND>
__device__ __forceinline__ void cm_pivot(const CmDims &D, CmState<R> &St, unsigned char *smem, CmXch *X, int e,
                                         int s, bool partner, int l, double av, double pe_l, double rr_l) {
    using C = CmCfg<NWR, R, S, ST>;
    double *tile = reinterpret_cast<double *>(smem + C::TILE);
    double *rowbuf = reinterpret_cast<double *>(smem + C::ROWBUF);
    double *rvec = reinterpret_cast<double *>(smem + C::RVEC);
    const bool mine = D.row == l;
    // ---- the leaving row publishes (before barrier B) ----
    cm_publish_regs<NWR, R>(D, St, rowbuf, l);
    if (mine) {
        // slot s then holds the leaving variable's column: e_l, 1 in row l
        if (s < R) rowbuf[s] = 1.0;
        else tile[tix<ST>(s - R, l)] = 1.0;
        X->pe = pe_l;
        X->rr = rr_l;
        X->oldvar = St.basis;
        X->oldpart = St.ppart;
        X->oldprc = St.prc;
    }
    __syncthreads();   // B
    const double pe = X->pe, rr = X->rr, fm = X->fm;
    // ---- transposed: slot q's pivot-row entry r_q = a_lq / pe, reduced costs, candidates ----
    int newtriv = -1;
    double newtriv_rc = 0.0;
    const int q = D.row;
    if (q < D.n) {
        double *src = q < R ? rowbuf + q : tile + tix<ST>(q - R, l);
        const double r = div_entry(*src, pe);
        rvec[q] = r;
        if (q >= R) *src = r;                            // row l of a tile column: final
        const bool here = q == s;
        if (here) {
            // the entering variable's pair member (if any) becomes trivial at row l
            newtriv = partner ? St.svar : St.spart;
            newtriv_rc = __dsub_rn(partner ? St.rc : St.rcp, __dmul_rn(fm, -1.0));
            X->newtriv = newtriv;
            X->newtriv_rc = newtriv_rc;
        }
        const double fr = __dmul_rn(fm, r), fnr = __dmul_rn(fm, -r);
        St.rc = __dsub_rn(here ? 0.0 : St.rc, fr);
        const int sp = here ? X->oldpart : St.spart;
        St.rcp = sp >= 0 ? __dsub_rn(here ? X->oldprc : St.rcp, fnr) : 0.0;
        St.svar = here ? X->oldvar : St.svar;
        St.spart = sp;
    }
    St.obj = __dadd_rn(St.obj, __dmul_rn(fm, rr));       // tableau.py:236-237,242
    if (CAND) cm_candidates<NWR, R, PH1>(D, St, X, mine, newtriv, newtriv_rc);
    __syncthreads();   // C
    if (mine) {
        St.basis = e;
        St.ppart = X->newtriv < 0 ? -1 : X->newtriv;
        St.prc = X->newtriv_rc;
    }
    if (D.row < D.m) {                                   // padding rows stay as built
        const double f = mine ? 0.0 : av;
        St.rhs = mine ? rr : __dsub_rn(St.rhs, __dmul_rn(f, rr));
        if (s < R) reg_put<R>(St.a, s, 0.0);            // the leaving column: e_l
        else if (!mine) tile[tix<ST>(s - R, D.row)] = 0.0;
#pragma unroll
        for (int c = 0; c < R; c += 2) {
            const double2 r2 = reinterpret_cast<const double2 *>(rvec)[c / 2];
            St.a[c] = __dsub_rn(St.a[c], __dmul_rn(av, r2.x));
            St.a[c + 1] = __dsub_rn(St.a[c + 1], __dmul_rn(av, r2.y));
        }
        // tile slots: software-pipelined (the tile and rvec share the shared-memory array, so
        // plain loads would serialise behind the previous column's store); row l: r - 0*r, as numpy
        if constexpr (S > 0) cm_update_tile<R, S, ST>(tile, D.row, rvec, mine ? 0.0 : av);
    }
    if ((l >> 5) == D.warp) {        // numpy: r - 0*r == r; warp-uniform reload of row l
        const unsigned rv = (unsigned)__cvta_generic_to_shared(rvec);
#pragma unroll
        for (int c = 0; c < R; c += 2) ld_shared_v2_if(mine, rv + 8u * c, St.a[c], St.a[c + 1]);
    }
    // the next writes to rowbuf / rvec / X come after barrier A of the next pivot (X->fm and
    // the leaving partials: before it, but after every reader has passed barrier C here)
}

// _run_phase (simplex.py:63-91); entering candidates already in X.
template <int NWR, int R, int S, int ST, bool PH1>
__device__ __forceinline__ WlpPhase cm_run_phase(const CmDims &D, CmState<R> &St, unsigned char *smem, CmXch *X,
                                                 const Limits &lim) {
    using C = CmCfg<NWR, R, S, ST>;
    const double *tile = reinterpret_cast<const double *>(smem + C::TILE);
    const int max_iter = lim.max_iterations > 0 ? lim.max_iterations : 50 * (D.m + D.n);
    const int trigger = lim.degenerate_limit >= 0 ? lim.degenerate_limit : (D.m > 1 ? D.m : 1);
    const unsigned long long kSent = key_max(kSentinel), kDeg = key_max(kDegenerateTol);
    int degenerate_run = 0;
    bool use_bland = false;
    for (int it = 0;; ++it) {
        if (it == max_iter) return {2, max_iter};
        const int cid = cm_select<NWR>(X, use_bland);    // choose_entering[_bland]
        if (cid == kNone) return {0, it};
        if (cm_kind(cid) == kCtTrivial) return {1, it};  // column -e_r: no positive entry
        const int e = cid >> 10, s = cid & 255;
        const bool partner = cm_kind(cid) == kCtPartner;
        double av = D.row < D.m ? cm_slot<NWR, R, S, ST>(St, tile, D.row, s) : 0.0;
        if (partner) av = -av;
        unsigned long long lk = kKeyEmptyMin;            // choose_leaving
        const double ratio = ratio_entry(St.rhs, av);
        if (D.row < D.m) lk = key_min(ratio);
        const unsigned long long kw = warp_min_key(lk);
        const int lw = warp_index_of(lk, kw, D.row);
        if (D.lane == 0) { X->lkey[D.warp] = kw; X->lrow[D.warp] = lw; }
        if (D.row == s) X->fm = partner ? St.rcp : St.rc;
        __syncthreads();   // A
        unsigned long long kmin = X->lkey[0];
        int l = X->lrow[0];
#pragma unroll
        for (int w = 1; w < NWR; ++w)                    // rows ascend with the warp: first minimum wins
            if (X->lkey[w] < kmin) { kmin = X->lkey[w]; l = X->lrow[w]; }
        if (l == kNone || kmin >= kSent) return {1, it};   // unbounded (a NaN ratio keys to 0)
        if (kmin != 0ull && kmin <= kDeg) {             // simplex.py:84-90
            ++degenerate_run;
            if (lim.anti_cycling && degenerate_run >= trigger) use_bland = true;
        } else {
            degenerate_run = 0;
            use_bland = false;
        }
        cm_pivot<NWR, R, S, ST, PH1, true>(D, St, smem, X, e, s, partner, l, av, av, ratio);
    }
}

// _price_out (simplex.py:133-143): rows in reference order, cb == 0 skipped; one barrier
// per priced row (the row buffer is double-buffered).
template <int NWR, int R, int S, int ST, bool PH1>
__device__ __forceinline__ void cm_price_out(const CmDims &D, CmState<R> &St, unsigned char *smem, CmXch *X,
                                             const double *cg) {
    using C = CmCfg<NWR, R, S, ST>;
    const double *tile = reinterpret_cast<const double *>(smem + C::TILE);
    double *rowbuf = reinterpret_cast<double *>(smem + C::ROWBUF);
    double *cbv = reinterpret_cast<double *>(smem + C::CBV);
    double *rhsv = reinterpret_cast<double *>(smem + C::RHSV);
    auto cext = [&](int v) -> double {
        if (PH1) return v >= D.nvc ? -1.0 : 0.0;
        return v < D.n ? cg[v] : 0.0;
    };
    const double cbr = D.row < D.m ? cext(St.basis) : 0.0;
    cbv[D.row] = cbr;
    rhsv[D.row] = St.rhs;
    const bool live = D.row < D.n;
    double racc = live ? cext(St.svar) : 0.0;
    double pacc = (live && St.spart >= 0) ? cext(St.spart) : 0.0;
    double obj = 0.0;
    __syncthreads();
    int k = 0;
    for (int r = 0; r < D.m; ++r) {
        const double cb = cbv[r];
        if (cb == 0.0) continue;             // uniform: every thread reads the same cbv[r]
        double *rb = rowbuf + (k & 1) * R;
        ++k;
        cm_publish_regs<NWR, R>(D, St, rb, r);
        __syncthreads();
        if (live) {
            const int q = D.row;
            const double v = q < R ? rb[q] : tile[tix<ST>(q - R, r)];
            racc = __dsub_rn(racc, __dmul_rn(cb, v));
            if (St.spart >= 0) pacc = __dsub_rn(pacc, __dmul_rn(cb, -v));
        }
        obj = __dadd_rn(obj, __dmul_rn(cb, rhsv[r]));
    }
    St.rc = racc;
    St.rcp = pacc;
    // a trivial member's column is -e_row: only its own row's cb contributes
    if (D.row < D.m && St.ppart >= 0) {
        const double c0 = cext(St.ppart);
        St.prc = cbr != 0.0 ? __dsub_rn(c0, __dmul_rn(cbr, -1.0)) : c0;
    }
    St.obj = obj;
    cm_candidates<NWR, R, PH1>(D, St, X, false, -1, 0.0);
    __syncthreads();
}

// restore_objective pivot-outs (simplex.py:109-126), uncounted: for each row whose basic
// variable is artificial, the first largest |entry| over the selectable columns.
template <int NWR, int R, int S, int ST>
__device__ __forceinline__ void cm_restore(const CmDims &D, CmState<R> &St, unsigned char *smem, CmXch *X) {
    using C = CmCfg<NWR, R, S, ST>;
    double *tile = reinterpret_cast<double *>(smem + C::TILE);
    double *rowbuf = reinterpret_cast<double *>(smem + C::ROWBUF);
    int *flag = reinterpret_cast<int *>(smem + C::FLAG);
    const unsigned long long kRed = key_max(kRedundantTol);
    // rows with an artificial basic variable (only a pivot on that row changes it)
    flag[D.row] = D.row < D.m && St.basis >= D.nvc;
    __syncthreads();
    for (int row = 0; row < D.m; ++row) {
        if (!flag[row]) continue;            // uniform
        cm_publish_regs<NWR, R>(D, St, rowbuf, row);
        __syncthreads();
        unsigned long long bk = kKeyEmptyMax;
        int bj = kNone;
        auto consider = [&](double v, int id) {
            const unsigned long long k = key_max(v);
            if (k > bk || (k == bk && id < bj)) { bk = k; bj = id; }
        };
        const int q = D.row;
        if (q < D.n) {
            const double v = fabs(q < R ? rowbuf[q] : tile[tix<ST>(q - R, row)]);
            if (St.svar < D.nvc) consider(v, cm_cid(St.svar, kCtSlot, q));
            if (St.spart >= 0 && St.spart < D.nvc) consider(v, cm_cid(St.spart, kCtPartner, q));
        }
        // the basic artificial's slack: column -e_row, |entry| = 1
        if (D.row == row && St.ppart >= 0 && St.ppart < D.nvc) consider(1.0, cm_cid(St.ppart, kCtTrivial, 0));
        const unsigned long long kw = warp_max_key(bk);
        const int iw = warp_index_of(bk, kw, bj);
        if (D.lane == 0) { X->ckey[D.warp] = kw; X->cid[D.warp] = iw; }
        __syncthreads();
        unsigned long long kb = X->ckey[0];
        int cid = X->cid[0];
#pragma unroll
        for (int w = 1; w < NWR; ++w)
            if (X->ckey[w] > kb || (X->ckey[w] == kb && X->cid[w] < cid)) { kb = X->ckey[w]; cid = X->cid[w]; }
        __syncthreads();   // X and rowbuf are rewritten below
        // entries[j] > REDUNDANT_ROW_TOL; a NaN entry compares False in numpy
        if (cid == kNone || kb <= kRed || kb == ~0ull) continue;
        const int j = cid >> 10;
        if (cm_kind(cid) == kCtTrivial) {
            // pivot on the trivial slack: pe = -1, f_i = 0 off row `row`: the row is negated
            if (D.row == row) {
#pragma unroll
                for (int c = 0; c < R; ++c) St.a[c] = -St.a[c];
#pragma unroll
                for (int c = 0; c < S; ++c) tile[tix<ST>(c, row)] = -tile[tix<ST>(c, row)];
                St.rhs = -St.rhs;
                St.ppart = St.basis;
                St.basis = j;
            }
            __syncthreads();
            continue;
        }
        const int s = cid & 255;
        const bool partner = cm_kind(cid) == kCtPartner;
        double av = D.row < D.m ? cm_slot<NWR, R, S, ST>(St, tile, D.row, s) : 0.0;
        if (partner) av = -av;
        if (D.row == 0) X->fm = 0.0;
        cm_pivot<NWR, R, S, ST, false, false>(D, St, smem, X, j, s, partner, row, av, av,
                                              D.row == row ? div_entry(St.rhs, av) : 0.0);
        __syncthreads();   // row publish of the next restore row reuses rowbuf
    }
}

// build_tableau (tableau.py:139-172): row tid into its thread (slots [R, NS) into the tile),
// validation fused; slot q starts as structural x_q with reduced cost c_q (0 without c: the
// shared phase-1 prologue).  Returns "some entry is non-finite" (CTA-wide) and n_art.
template <int NWR, int R, int S, int ST>
__device__ __forceinline__ bool cm_build(const CmDims &D, CmState<R> &St, unsigned char *smem, CmXch *X,
                                         const double *Ag, const double *bg, const double *cg, int &n_art) {
    using C = CmCfg<NWR, R, S, ST>;
    double *tile = reinterpret_cast<double *>(smem + C::TILE);
    const int m = D.m, n = D.n;
    bool nonfinite = false;
    const bool live = D.row < m;
    const double bi = live ? bg[D.row] : 0.0;
    nonfinite |= !isfinite(bi);
    const bool neg = live && bi < 0.0;
    const double sgn = neg ? -1.0 : 1.0;
    St.rhs = live ? __dmul_rn(bi, sgn) : 0.0;
    {
        const double *arow = Ag + (size_t)(live ? D.row : 0) * n;
#pragma unroll
        for (int c = 0; c < R; ++c) {
            double v = 0.0;
            if (live && c < n) {
                const double x = arow[c];
                nonfinite |= !isfinite(x);
                v = __dmul_rn(x, sgn);
            }
            St.a[c] = v;
        }
        if (live) {                            // padding rows never touch the tile (ST >= m only)
#pragma unroll
            for (int c = 0; c < S; ++c) {
                double v = 0.0;
                if (R + c < n) {
                    const double x = arow[R + c];
                    nonfinite |= !isfinite(x);
                    v = __dmul_rn(x, sgn);
                }
                tile[tix<ST>(c, D.row)] = v;
            }
        }
    }
    const unsigned negm = __ballot_sync(kFull, neg);
    if (D.lane == 0) X->nneg[D.warp] = __popc(negm);
    if (cg && D.row < n) {
        St.rc = cg[D.row];
        nonfinite |= !isfinite(St.rc);
    } else {
        St.rc = 0.0;
    }
    const bool invalid = __syncthreads_or(nonfinite);
    int art = __popc(negm & ((1u << D.lane) - 1u));
    n_art = 0;
#pragma unroll
    for (int w = 0; w < NWR; ++w) {
        art += w < D.warp ? X->nneg[w] : 0;
        n_art += X->nneg[w];
    }
    St.basis = neg ? D.nvc + art : n + D.row;
    St.ppart = neg ? n + D.row : -1;      // the negated row's slack: column -e_row
    St.prc = 0.0;
    St.svar = D.row;                       // slot q: structural x_q
    St.spart = -1;
    St.rcp = 0.0;
    St.obj = 0.0;
    return invalid;
}

// Phase 1 (simplex.py:168-178): build_auxiliary, _run_phase, the infeasibility test and
// restore_objective (c-independent).  Returns the status if the LP ends here, else kOptimal.
template <int NWR, int R, int S, int ST>
__device__ __forceinline__ int cm_phase1(const CmDims &D, CmState<R> &St, unsigned char *smem, CmXch *X,
                                         const Limits &lim, int &it1) {
    cm_price_out<NWR, R, S, ST, true>(D, St, smem, X, nullptr);
    const WlpPhase p1 = cm_run_phase<NWR, R, S, ST, true>(D, St, smem, X, lim);
    it1 = p1.iters;
    if (p1.state == 2) return kIterationLimit;
    if (p1.state == 1) return kErrPhase1Unbounded;
    if (fabs(St.obj) > kPhase1ZeroTol) return kInfeasible;
    __syncthreads();
    cm_restore<NWR, R, S, ST>(D, St, smem, X);
    return kOptimal;
}

// Shared phase 1 (support mode): the restored tableau of the shared A, b, dumped once by
// cmulti_phase1_kernel and loaded by every direction (coalesced: field-major, thread-minor;
// the tile copied as is).  info (4 ints after the state): [0] status, [1] phase-1 iterations,
// [2] mode (0: b >= 0, build as usual; 1: shared).
template <int NWR, int R, int S, int ST>
struct CmP1 {
    static constexpr int ROWS = 32 * NWR;
    static constexpr int ND = R + 2;                     // a, rhs, prc
    static constexpr int NI = 4;                         // basis, ppart, svar, spart
    static constexpr size_t TILE_OFF = (size_t)ROWS * ND;               // doubles
    static constexpr size_t INT_OFF = TILE_OFF + (size_t)S * ST;         // doubles
    static constexpr size_t BYTES = INT_OFF * 8 + (size_t)ROWS * NI * 4 + 16;
};

template <int NWR, int R, int S, int ST>
__device__ __forceinline__ void cm_dump(const CmDims &D, const CmState<R> &St, const unsigned char *smem,
                                        double *st) {
    using P = CmP1<NWR, R, S, ST>;
    constexpr int ROWS = P::ROWS;
    const double *tile = reinterpret_cast<const double *>(smem + CmCfg<NWR, R, S, ST>::TILE);
    int *si = reinterpret_cast<int *>(st + P::INT_OFF);
    const int t = D.row;
#pragma unroll
    for (int c = 0; c < R; ++c) st[c * ROWS + t] = St.a[c];
    st[R * ROWS + t] = St.rhs;
    st[(R + 1) * ROWS + t] = St.prc;
    for (int i = t; i < S * ST; i += ROWS) st[P::TILE_OFF + i] = tile[i];
    si[t] = St.basis;
    si[ROWS + t] = St.ppart;
    si[2 * ROWS + t] = St.svar;
    si[3 * ROWS + t] = St.spart;
}

template <int NWR, int R, int S, int ST>
__device__ __forceinline__ void cm_load(const CmDims &D, CmState<R> &St, unsigned char *smem, const double *st) {
    using P = CmP1<NWR, R, S, ST>;
    constexpr int ROWS = P::ROWS;
    double *tile = reinterpret_cast<double *>(smem + CmCfg<NWR, R, S, ST>::TILE);
    const int *si = reinterpret_cast<const int *>(st + P::INT_OFF);
    const int t = D.row;
#pragma unroll
    for (int c = 0; c < R; ++c) St.a[c] = st[c * ROWS + t];
    St.rhs = st[R * ROWS + t];
    St.prc = st[(R + 1) * ROWS + t];
    for (int i = t; i < S * ST; i += ROWS) tile[i] = st[P::TILE_OFF + i];
    St.basis = si[t];
    St.ppart = si[ROWS + t];
    St.svar = si[2 * ROWS + t];
    St.spart = si[3 * ROWS + t];
    St.obj = 0.0;
}

// One CTA: the shared polytope's phase 1 into `st` (support mode only).
template <int NWR, int R, int S, int ST>
__global__ void __launch_bounds__(32 * NWR, 1) cmulti_phase1_kernel(Batch B, double *st) {
    using C = CmCfg<NWR, R, S, ST>;
    extern __shared__ __align__(16) unsigned char smem[];
    CmXch *X = reinterpret_cast<CmXch *>(smem + C::XCH);
    int *info = reinterpret_cast<int *>(reinterpret_cast<char *>(st) + CmP1<NWR, R, S, ST>::BYTES - 16);
    CmDims D;
    D.m = B.m; D.n = B.n; D.nvc = B.n + B.m;
    D.lane = threadIdx.x & 31; D.warp = threadIdx.x >> 5; D.row = threadIdx.x;
    for (int q = threadIdx.x; q < C::NS; q += C::ROWS) reinterpret_cast<double *>(smem + C::RVEC)[q] = 0.0;
    __syncthreads();
    CmState<R> St;
    int n_art = 0, it1 = 0, status = kOptimal;
    const bool invalid = cm_build<NWR, R, S, ST>(D, St, smem, X, B.A, B.b, nullptr, n_art);
    if (invalid) status = kInvalid;
    else if (n_art > 0) status = cm_phase1<NWR, R, S, ST>(D, St, smem, X, B.lim, it1);
    __syncthreads();
    cm_dump<NWR, R, S, ST>(D, St, smem, st);
    if (threadIdx.x == 0) {
        info[0] = status;
        info[1] = it1;
        info[2] = (invalid || n_art > 0) ? 1 : 0;
    }
}

template <int NWR, int R, int S, int ST, int kMinBlocks>
__global__ void __launch_bounds__(32 * NWR, kMinBlocks)
cmulti_kernel(Batch B) {
    using C = CmCfg<NWR, R, S, ST>;
    extern __shared__ __align__(16) unsigned char smem[];
    CmXch *X = reinterpret_cast<CmXch *>(smem + C::XCH);
    CmDims D;
    D.m = B.m; D.n = B.n; D.nvc = B.n + B.m;
    D.lane = threadIdx.x & 31; D.warp = threadIdx.x >> 5; D.row = threadIdx.x;
    const int m = D.m, n = D.n;
    {
        double *rvec = reinterpret_cast<double *>(smem + C::RVEC);
        for (int q = threadIdx.x; q < C::NS; q += C::ROWS) rvec[q] = 0.0;   // unused slots read as 0
    }
    // LP queue over the batch, or over the lazy kernel's deferral list (batch_lp)
    const long long total = batch_count(B);
    if (threadIdx.x == 0) X->lp = atomicAdd(B.next_lp, 1);
    __syncthreads();
    long long k = X->lp;
    CmState<R> St;
    for (;;) {
        if (k >= total) break;
        const long long lp = batch_lp(B, k);
        long long nxt = 0;                  // claim the next LP and warm L2 with its inputs
        if (threadIdx.x == 0) nxt = atomicAdd(B.next_lp, 1);
        if (D.warp == 0) {
            nxt = __shfl_sync(kFull, nxt, 0);
            if (nxt < total) prefetch_lp_inputs(B, batch_lp(B, nxt), D.lane);
        }
        const double *Ag = B.shared_Ab ? B.A : B.A + (size_t)lp * m * n;
        const double *bg = B.shared_Ab ? B.b : B.b + (size_t)lp * m;
        const double *cg = B.c + (size_t)lp * n;

        int8_t status = kOptimal;
        int it1 = 0, it2 = 0;
        bool done = false;
        // support mode with b < 0: phase 1 was solved once by cmulti_phase1_kernel (its info is
        // re-read per LP -- an L1 hit -- rather than held in registers across the solve)
        const int *p1info = B.p1state ? reinterpret_cast<const int *>(reinterpret_cast<const char *>(B.p1state) +
                                                                      CmP1<NWR, R, S, ST>::BYTES - 16) : nullptr;
        if (p1info && p1info[2] == 1) {
            const int p1status = p1info[0], p1iters = p1info[1];
            const bool nonfinite = D.row < n && !isfinite(cg[D.row]);
            if (__syncthreads_or(nonfinite) || p1status == kInvalid) {
                status = kInvalid;
                done = true;
            } else if (p1status != kOptimal) {
                status = (int8_t)p1status;
                it1 = p1iters;
                done = true;
            } else {
                it1 = p1iters;
                cm_load<NWR, R, S, ST>(D, St, smem, B.p1state);
                cm_price_out<NWR, R, S, ST, false>(D, St, smem, X, cg);
            }
        } else {
            int n_art = 0;
            const bool invalid = cm_build<NWR, R, S, ST>(D, St, smem, X, Ag, bg, cg, n_art);
            if (invalid) {
                status = kInvalid;
                done = true;
            } else if (n_art > 0) {
                const int st = cm_phase1<NWR, R, S, ST>(D, St, smem, X, B.lim, it1);
                if (st != kOptimal) { status = (int8_t)st; done = true; }
                else cm_price_out<NWR, R, S, ST, false>(D, St, smem, X, cg);
            } else {
                cm_candidates<NWR, R, false>(D, St, X, false, -1, 0.0);
                __syncthreads();
            }
        }
        if (!done) {
            const WlpPhase p2 = cm_run_phase<NWR, R, S, ST, false>(D, St, smem, X, B.lim);
            it2 = p2.iters;
            if (p2.state == 2) status = kIterationLimit;
            else if (p2.state == 1) status = kUnbounded;
        }

        // ---- _extract_point (simplex.py:146-151) and c @ x ----
        double *xs = reinterpret_cast<double *>(smem + C::CBV);   // n <= ROWS doubles
        double *xg = B.x + (size_t)lp * n;
        __syncthreads();
        if (D.row < n) xs[D.row] = 0.0;
        __syncthreads();
        if (status == kOptimal && D.row < m && St.basis < n) xs[St.basis] = St.rhs;
        __syncthreads();
        if (D.row < n) xg[D.row] = xs[D.row];
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
            X->lp = nxt;
        }
        __syncthreads();
        k = X->lp;
    }
}

}  // namespace blp
