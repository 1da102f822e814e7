// blp_condensed_kernel.cuh -- one warp per LP on the CONDENSED tableau:
// only the nonbasic columns (+ rhs) are stored and updated, bit-identical to
// the reference's full tableau (tableau.py:218-244 applied to every column).
//
// Why it is exact.  A basic column is a unit vector e_r, exactly: when column
// e enters at row l its new entries are a_ie - a_ie*(a_le/a_le) = a_ie - a_ie*1
// = 0 (row l: a_le/a_le = 1), its reduced cost rc_e - rc_e*1 = 0; while it
// stays basic, a later pivot on row l' != r has pivot-row entry 0, so
// r_j = 0/pe = 0 and every cell takes a - f*0 = a.  The reference rewrites
// those m columns every pivot without changing a value; skipping them leaves
// (m+1) x (n+1) cells per pivot instead of (m+1) x (n+m+1).  When variable e
// enters and w leaves, w's column (e_l before the pivot) takes e's slot: its
// new entries are exactly what the reference computes for it -- 0 - f_i*r_w
// with r_w = 1/pe (row l: r_w), reduced cost 0 - rc_e*r_w.
//
// Artificial columns (phase 1, rows with b < 0): the artificial a_i of a
// negated row and that row's slack s_i have value-equal opposite columns at
// every step (both start as +-e_i; every pivot applies sign-symmetric IEEE
// operations).  Hence never both basic, and the pair is in one of three states:
//   (A) s_i basic at row r, a_i nonbasic with column -e_r ("trivial" member);
//   (B) a_i basic at row r, s_i nonbasic with column -e_r (trivial member);
//   (C) both nonbasic: one slot holds the column of one of them (svar), the
//       other is its "partner" (spart) with the negated column.
// A trivial member's reduced cost changes only when its partner leaves (the
// pair goes to state C and takes the freed slot), so the row that holds the
// partner keeps it (ppart / prc).  Counting states shows the number of slots is
// always exactly n.  A trivial member has no positive entry, so choosing it as
// the entering column is "unbounded", as in the reference; restore_objective
// may pivot on it (|entry| = 1): that pivot negates its row and nothing else.
//
// Layout: lane L holds constraint rows L + 32k (k < RPL) as RPL register rows
// of NS slot values plus rhs; the objective row is transposed (lane q holds
// slot q + 32u's reduced cost, variable and partner).  Per pivot: entering
// from the precomputed candidates (order-preserving keys + redux); ratio test
// on the lanes' rows; the pivot row goes through shared memory, each lane
// divides its transposed slots and rebuilds their candidates; every lane
// applies a - f*r to its registers.  No CTA barrier, no shared-memory tableau.
#pragma once

#include "blp_common.cuh"
#include "blp_keys.cuh"
#include "blp_warplp_kernel.cuh"

namespace blp {

template <int RPL, int NS>
struct CtCfg {
    static constexpr int SPL = (NS + 31) / 32;          // transposed slots per lane
    static constexpr size_t ROWBUF = 0;                  // NS doubles
    static constexpr size_t RVEC = ROWBUF + (size_t)NS * 8;
    static constexpr size_t CBV = RVEC + (size_t)NS * 8; // 32*RPL doubles
    static constexpr size_t RHSV = CBV + (size_t)32 * RPL * 8;
    static constexpr size_t XS = RHSV + (size_t)32 * RPL * 8;  // NS doubles: x scatter
    static constexpr size_t BYTES = XS + (size_t)NS * 8;
    // Optional TMA staging of the next LP's A (condensed_kernel, when the launch grants
    // STG_END bytes): an mbarrier, then 32*RPL rows at a stride of NS*8 + 16 bytes (16-byte
    // aligned for cp.async.bulk; lane L's 128-bit row reads spread over 8 bank groups).
    static constexpr size_t STG_BAR = (BYTES + 15) / 16 * 16;
    static constexpr size_t STG = STG_BAR + 16;
    static constexpr size_t STG_END = STG + (size_t)32 * RPL * (NS * 8 + 16);
};

template <int RPL, int NS>
struct CtState {
    static constexpr int SPL = CtCfg<RPL, NS>::SPL;
    double a[RPL][NS];      // rows lane + 32k: slot values
    double rhs[RPL];
    int basis[RPL];         // basic variable of the row
    int ppart[RPL];         // its pair's trivial member (state A/B), or -1
    double prc[RPL];        // that member's reduced cost
    double rc[SPL], rcp[SPL];   // transposed: reduced cost of slot q = lane + 32u and of its partner
    int svar[SPL], spart[SPL];
    double obj;             // objective cell (the same in every lane)
    unsigned long long ckey;   // Dantzig winner's key and composite id (ct_cid), warp-uniform
    int cid;
};

// Composite candidate id: variable index in the high bits (so the lowest id among equal
// keys is numpy's first index), where it lives in the low 8: kind (0 the slot's variable,
// 1 the slot's partner, 2 a trivial member) and the slot q -- the reduction that picks the
// entering variable also locates it.
__device__ __forceinline__ int ct_cid(int var, int kind, int q) { return (var << 8) | (kind << 6) | q; }
constexpr int kCtSlot = 0, kCtPartner = 1, kCtTrivial = 2;

struct CtDims { int m, n, nvc, lane; };

// a[i] = v for a warp-uniform runtime index (uniform branch tree, then selp's):
// register arrays are only ever indexed statically.
template <int LO, int N, int W>
struct RegPutter {
    static __device__ __forceinline__ void put(double (&a)[W], int i, double v) {
        if constexpr (N <= 8) {
#pragma unroll
            for (int k = 0; k < N; ++k) a[LO + k] = selp_f64(v, a[LO + k], i == LO + k);
        } else {
            if (i < LO + N / 2) RegPutter<LO, N / 2, W>::put(a, i, v);
            else RegPutter<LO + N / 2, N - N / 2, W>::put(a, i, v);
        }
    }
};

template <int W>
__device__ __forceinline__ void reg_put(double (&a)[W], int i, double v) {
    RegPutter<0, W, W>::put(a, i, v);
}

__device__ __forceinline__ void ct_consider(double v, int j, unsigned long long &ck, int &ci) {
    const unsigned long long k = key_max(v);
    if (k > ck || (k == ck && j < ci)) { ck = k; ci = j; }
}

// Entering candidates over every nonbasic selectable variable: slot variables,
// slot partners, trivial members (choose_entering, Dantzig: max key, first index).
template <int RPL, int NS, bool PH1>
__device__ __forceinline__ void ct_candidates(const CtDims &D, CtState<RPL, NS> &S) {
    unsigned long long ck = kKeyEmptyMax;
    int ci = kNone;
#pragma unroll
    for (int u = 0; u < CtCfg<RPL, NS>::SPL; ++u) {
        const int q = D.lane + 32 * u;
        if (q < D.n) {
            if (PH1 || S.svar[u] < D.nvc) ct_consider(S.rc[u], ct_cid(S.svar[u], kCtSlot, q), ck, ci);
            if (S.spart[u] >= 0 && (PH1 || S.spart[u] < D.nvc))
                ct_consider(S.rcp[u], ct_cid(S.spart[u], kCtPartner, q), ck, ci);
        }
    }
#pragma unroll
    for (int k = 0; k < RPL; ++k)
        if (D.lane + 32 * k < D.m && S.ppart[k] >= 0 && (PH1 || S.ppart[k] < D.nvc))
            ct_consider(S.prc[k], ct_cid(S.ppart[k], kCtTrivial, 0), ck, ci);
    S.ckey = warp_max_key(ck);
    S.cid = warp_index_of(ck, S.ckey, ci);
}

// choose_entering_bland (tableau.py:189-197): the lowest-index candidate with rc > tol,
// as a composite id (kNone if none).  Only evaluated while Bland's rule is active.
template <int RPL, int NS, bool PH1>
__device__ __forceinline__ int ct_bland(const CtDims &D, const CtState<RPL, NS> &S) {
    int cb = kNone;
#pragma unroll
    for (int u = 0; u < CtCfg<RPL, NS>::SPL; ++u) {
        const int q = D.lane + 32 * u;
        if (q < D.n) {
            if ((PH1 || S.svar[u] < D.nvc) && S.rc[u] > kTol) cb = min(cb, ct_cid(S.svar[u], kCtSlot, q));
            if (S.spart[u] >= 0 && (PH1 || S.spart[u] < D.nvc) && S.rcp[u] > kTol)
                cb = min(cb, ct_cid(S.spart[u], kCtPartner, q));
        }
    }
#pragma unroll
    for (int k = 0; k < RPL; ++k)
        if (D.lane + 32 * k < D.m && S.ppart[k] >= 0 && (PH1 || S.ppart[k] < D.nvc) && S.prc[k] > kTol)
            cb = min(cb, ct_cid(S.ppart[k], kCtTrivial, 0));
    return (int)__reduce_min_sync(kFull, (unsigned)cb);
}

// Where variable e lives: slot s (its column) or slot s's partner (negated
// column), or a trivial member (returns s = -1).
struct CtWhere { int s; bool partner; };

template <int RPL, int NS>
__device__ __forceinline__ CtWhere ct_locate(const CtDims &D, const CtState<RPL, NS> &S, int e) {
    int hit = kNone;
    bool part = false;
#pragma unroll
    for (int u = 0; u < CtCfg<RPL, NS>::SPL; ++u) {
        const int q = D.lane + 32 * u;
        if (q < D.n && S.svar[u] == e) hit = q;
        if (q < D.n && S.spart[u] == e) { hit = q; part = true; }
    }
    CtWhere w;
    w.s = (int)__reduce_min_sync(kFull, (unsigned)hit);
    w.partner = __any_sync(kFull, part);
    if (w.s == kNone) w.s = -1;
    return w;
}

// Register row kr of the owner lane (mine) to shared memory at rb.  The row is
// picked per element with selp (a branch per row would let the compiler fold
// the rows into one dynamically indexed -- local-memory -- array).
template <int RPL, int NS>
__device__ __forceinline__ void ct_store_row(const CtState<RPL, NS> &S, bool mine, int kr, unsigned rb) {
#pragma unroll
    for (int c = 0; c < NS; c += 2) {
        double x = S.a[0][c], y = S.a[0][c + 1];
#pragma unroll
        for (int t = 1; t < RPL; ++t) {
            x = selp_f64(S.a[t][c], x, kr == t);
            y = selp_f64(S.a[t][c + 1], y, kr == t);
        }
        st_shared_v2_if(mine, rb + 8u * c, x, y);
    }
}

// Row `row` of the condensed tableau into rowbuf (its owner lane stores it).
template <int RPL, int NS>
__device__ __forceinline__ void ct_share_row(const CtDims &D, const CtState<RPL, NS> &S, unsigned char *smem,
                                             int row) {
    const unsigned rb = (unsigned)__cvta_generic_to_shared(smem + CtCfg<RPL, NS>::ROWBUF);
    __syncwarp();
    ct_store_row<RPL, NS>(S, D.lane == (row & 31), row >> 5, rb);
    __syncwarp();
}

template <int RPL>
__device__ __forceinline__ double ct_row_sel(const double (&v)[RPL], int k) {
    double r = v[0];
#pragma unroll
    for (int t = 1; t < RPL; ++t) r = selp_f64(v[t], r, k == t);
    return r;
}
template <int RPL>
__device__ __forceinline__ int ct_row_sel_i(const int (&v)[RPL], int k) {
    int r = v[0];
#pragma unroll
    for (int t = 1; t < RPL; ++t) r = k == t ? v[t] : r;
    return r;
}

// pivot (tableau.py:218-244) on the condensed tableau.  e enters from slot s
// (negated column if `partner`), row l leaves; av[k] = this lane's rows of the
// entering column, fm = its reduced cost (0 for restore pivots: the objective
// row is rebuilt by the price-out that follows), rr = rhs_l / pe (the winning
// ratio: the same IEEE division the reference applies to the rhs cell).
template <int RPL, int NS>
__device__ __forceinline__ void ct_pivot(const CtDims &D, CtState<RPL, NS> &S, unsigned char *smem, int e, int s,
                                         bool partner, int l, const double (&av)[RPL], double pe, double fm,
                                         double rr) {
    using C = CtCfg<RPL, NS>;
    constexpr int SPL = C::SPL;
    double *rowbuf = reinterpret_cast<double *>(smem + C::ROWBUF);
    double *rvec = reinterpret_cast<double *>(smem + C::RVEC);
    const unsigned rb = (unsigned)__cvta_generic_to_shared(rowbuf);
    const unsigned rv = (unsigned)__cvta_generic_to_shared(rvec);
    const int kl = l >> 5, ll = l & 31;
    const bool mine = D.lane == ll;
    const int oldvar = __shfl_sync(kFull, ct_row_sel_i<RPL>(S.basis, kl), ll);
    const int oldpart = __shfl_sync(kFull, ct_row_sel_i<RPL>(S.ppart, kl), ll);
    const double oldprc = __shfl_sync(kFull, ct_row_sel<RPL>(S.prc, kl), ll);
    __syncwarp();   // every lane is done reading rowbuf (restore's candidate scan)
    // row l into rowbuf; slot s then holds the leaving variable's column (e_l): 1 in row l
    ct_store_row<RPL, NS>(S, mine, kl, rb);
    if (mine) rowbuf[s] = 1.0;
    __syncwarp();
    // transposed: slot q's pivot-row entry r_q = a_lq / pe, its reduced cost(s), candidates
    int newtriv = -1;
    double newtriv_rc = 0.0;
#pragma unroll
    for (int u = 0; u < SPL; ++u) {
        const int q = D.lane + 32 * u;
        if (q < D.n) {
            const double r = div_entry(rowbuf[q], pe);
            rvec[q] = r;
            // branch-free (one lane is slot s): slot s restarts from the leaving variable,
            // whose column and reduced cost were e_l and 0 (partner: its trivial member's prc)
            const bool here = q == s;
            if (here) {
                // the entering variable's pair member (if any) becomes trivial at row l
                newtriv = partner ? S.svar[u] : S.spart[u];
                newtriv_rc = __dsub_rn(partner ? S.rc[u] : S.rcp[u], __dmul_rn(fm, -1.0));
            }
            const double fr = __dmul_rn(fm, r), fnr = __dmul_rn(fm, -r);
            S.rc[u] = __dsub_rn(here ? 0.0 : S.rc[u], fr);
            const int sp = here ? oldpart : S.spart[u];
            S.rcp[u] = sp >= 0 ? __dsub_rn(here ? oldprc : S.rcp[u], fnr) : 0.0;
            S.svar[u] = here ? oldvar : S.svar[u];
            S.spart[u] = sp;
        }
    }
    newtriv = (int)__reduce_min_sync(kFull, (unsigned)(newtriv < 0 ? kNone : newtriv));
    const int owner = s & 31;
    newtriv_rc = __shfl_sync(kFull, newtriv_rc, owner);
    S.obj = __dadd_rn(S.obj, __dmul_rn(fm, rr));                       // tableau.py:236-237,242
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
        if (kl == k && mine) {
            S.basis[k] = e;
            S.ppart[k] = newtriv == kNone ? -1 : newtriv;
            S.prc[k] = newtriv_rc;
        }
        const double f = (kl == k && mine) ? 0.0 : av[k];
        S.rhs[k] = (kl == k && mine) ? rr : __dsub_rn(S.rhs[k], __dmul_rn(f, rr));
        reg_put<NS>(S.a[k], s, 0.0);                                    // the leaving column: e_l
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
        const double f = av[k];
#pragma unroll
        for (int c = 0; c < NS; c += 2) {
            const double2 r2 = reinterpret_cast<const double2 *>(rvec)[c / 2];
            S.a[k][c] = __dsub_rn(S.a[k][c], __dmul_rn(f, r2.x));
            S.a[k][c + 1] = __dsub_rn(S.a[k][c + 1], __dmul_rn(f, r2.y));
        }
        // numpy: r - 0*r == r
#pragma unroll
        for (int c = 0; c < NS; c += 2) ld_shared_v2_if(mine && kl == k, rv + 8u * c, S.a[k][c], S.a[k][c + 1]);
    }
    __syncwarp();
}

// _run_phase (simplex.py:63-91); entering candidates already in S.
template <int RPL, int NS, bool PH1>
__device__ __forceinline__ WlpPhase ct_run_phase(const CtDims &D, CtState<RPL, NS> &S, unsigned char *smem,
                                                 const Limits &lim) {
    const int max_iter = lim.max_iterations > 0 ? lim.max_iterations : 50 * (D.m + D.n);
    const int trigger = lim.degenerate_limit >= 0 ? lim.degenerate_limit : (D.m > 1 ? D.m : 1);
    const unsigned long long kSent = key_max(kSentinel), kDeg = key_max(kDegenerateTol), kTolK = key_max(kTol);
    int degenerate_run = 0;
    bool use_bland = false;
    for (int it = 0;; ++it) {
        if (it == max_iter) return {2, max_iter};
        int cid;
        if (use_bland) cid = ct_bland<RPL, NS, PH1>(D, S);               // choose_entering_bland
        else cid = (S.cid == kNone || S.ckey <= kTolK) ? kNone : S.cid;  // choose_entering
        if (cid == kNone) return {0, it};
        const int e = cid >> 8;
        CtWhere w;
        w.s = cid & 63;
        w.partner = ((cid >> 6) & 3) == kCtPartner;
        if (((cid >> 6) & 3) == kCtTrivial) return {1, it};   // column -e_r: no positive entry
        double av[RPL];
        unsigned long long lk = kKeyEmptyMin;
        int lrow = kNone;
        double lratio = 0.0;
#pragma unroll
        for (int k = 0; k < RPL; ++k) {
            const int row = D.lane + 32 * k;
            double v = reg_pick<NS>(S.a[k], w.s);
            if (w.partner) v = -v;
            av[k] = row < D.m ? v : 0.0;
            const double ratio = ratio_entry(S.rhs[k], v);                 // choose_leaving
            if (row < D.m) {
                const unsigned long long key = key_min(ratio);
                if (key < lk) { lk = key; lrow = row; lratio = ratio; }
            }
        }
        const unsigned long long kmin = warp_min_key(lk);
        const int l = warp_index_of(lk, kmin, lrow);
        if (l == kNone || kmin >= kSent) return {1, it};   // unbounded (a NaN ratio keys to 0)
        const double rr = __shfl_sync(kFull, lratio, l & 31);
        const double pe = __shfl_sync(kFull, ct_row_sel<RPL>(av, l >> 5), l & 31);
        double myfm = 0.0;
#pragma unroll
        for (int u = 0; u < CtCfg<RPL, NS>::SPL; ++u)
            myfm = selp_f64(w.partner ? S.rcp[u] : S.rc[u], myfm, u == (w.s >> 5));
        const double fm = __shfl_sync(kFull, myfm, w.s & 31);
        if (kmin != 0ull && kmin <= kDeg) {                 // simplex.py:84-90
            ++degenerate_run;
            if (lim.anti_cycling && degenerate_run >= trigger) use_bland = true;
        } else {
            degenerate_run = 0;
            use_bland = false;
        }
        ct_pivot<RPL, NS>(D, S, smem, e, w.s, w.partner, l, av, pe, fm, rr);
        ct_candidates<RPL, NS, PH1>(D, S);
    }
}

// _price_out (simplex.py:133-143) for c_ext = the phase-1 objective (-1 on the
// artificials) or the original c: rows in reference order, cb == 0 skipped.
template <int RPL, int NS, bool PH1>
__device__ __forceinline__ void ct_price_out(const CtDims &D, CtState<RPL, NS> &S, unsigned char *smem,
                                             const double *cg) {
    using C = CtCfg<RPL, NS>;
    constexpr int SPL = C::SPL;
    double *cbv = reinterpret_cast<double *>(smem + C::CBV);
    double *rhsv = reinterpret_cast<double *>(smem + C::RHSV);
    const double *rowbuf = reinterpret_cast<const double *>(smem + C::ROWBUF);
    auto cext = [&](int v) -> double {
        if (PH1) return v >= D.nvc ? -1.0 : 0.0;
        return v < D.n ? cg[v] : 0.0;
    };
    double cbr[RPL];
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
        const int row = D.lane + 32 * k;
        cbr[k] = row < D.m ? cext(S.basis[k]) : 0.0;
        cbv[row] = cbr[k];
        rhsv[row] = S.rhs[k];
    }
    double racc[SPL], pacc[SPL];
#pragma unroll
    for (int u = 0; u < SPL; ++u) {
        const bool live = D.lane + 32 * u < D.n;
        racc[u] = live ? cext(S.svar[u]) : 0.0;
        pacc[u] = (live && S.spart[u] >= 0) ? cext(S.spart[u]) : 0.0;
    }
    double obj = 0.0;
    __syncwarp();
    for (int r = 0; r < D.m; ++r) {
        const double cb = cbv[r];
        if (cb == 0.0) continue;             // uniform: every lane reads the same cbv[r]
        ct_share_row<RPL, NS>(D, S, smem, r);
#pragma unroll
        for (int u = 0; u < SPL; ++u) {
            const int q = D.lane + 32 * u;
            if (q < D.n) {
                const double v = rowbuf[q];
                racc[u] = __dsub_rn(racc[u], __dmul_rn(cb, v));
                if (S.spart[u] >= 0) pacc[u] = __dsub_rn(pacc[u], __dmul_rn(cb, -v));
            }
        }
        obj = __dadd_rn(obj, __dmul_rn(cb, rhsv[r]));
    }
#pragma unroll
    for (int u = 0; u < SPL; ++u) {
        S.rc[u] = racc[u];
        S.rcp[u] = pacc[u];
    }
    // a trivial member's column is -e_row: only its own row's cb contributes
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
        if (S.ppart[k] >= 0) {
            const double c0 = cext(S.ppart[k]);
            S.prc[k] = cbr[k] != 0.0 ? __dsub_rn(c0, __dmul_rn(cbr[k], -1.0)) : c0;
        }
    }
    S.obj = obj;
    __syncwarp();
    ct_candidates<RPL, NS, PH1>(D, S);
}

// restore_objective pivot-outs (simplex.py:109-126), uncounted: for each row
// whose basic variable is artificial, the first largest |entry| over the
// selectable (non-artificial) columns.
template <int RPL, int NS>
__device__ __forceinline__ void ct_restore(const CtDims &D, CtState<RPL, NS> &S, unsigned char *smem) {
    using C = CtCfg<RPL, NS>;
    constexpr int SPL = C::SPL;
    const double *rowbuf = reinterpret_cast<const double *>(smem + C::ROWBUF);
    const unsigned long long kRed = key_max(kRedundantTol);
    for (int row = 0; row < D.m; ++row) {
        const int kr = row >> 5, lr = row & 31;
        const int bv = __shfl_sync(kFull, ct_row_sel_i<RPL>(S.basis, kr), lr);
        if (bv < D.nvc) continue;
        ct_share_row<RPL, NS>(D, S, smem, row);
        unsigned long long bk = kKeyEmptyMax;
        int bj = kNone;
#pragma unroll
        for (int u = 0; u < SPL; ++u) {
            const int q = D.lane + 32 * u;
            if (q < D.n) {
                const double v = fabs(rowbuf[q]);
                if (S.svar[u] < D.nvc) ct_consider(v, S.svar[u], bk, bj);
                if (S.spart[u] >= 0 && S.spart[u] < D.nvc) ct_consider(v, S.spart[u], bk, bj);
            }
        }
        // the basic artificial's slack: column -e_row, |entry| = 1
        const int pp = ct_row_sel_i<RPL>(S.ppart, kr);
        if (D.lane == lr && pp >= 0 && pp < D.nvc) ct_consider(1.0, pp, bk, bj);
        const unsigned long long kb = warp_max_key(bk);
        const int j = warp_index_of(bk, kb, bj);
        // entries[j] > REDUNDANT_ROW_TOL; a NaN entry compares False in numpy
        if (j == kNone || kb <= kRed || kb == ~0ull) continue;
        const CtWhere w = ct_locate<RPL, NS>(D, S, j);
        if (w.s < 0) {
            // pivot on the trivial slack: pe = -1, f_i = 0 off row `row`: the row is negated
            // (x / -1 is exactly -x in IEEE arithmetic)
#pragma unroll
            for (int k = 0; k < RPL; ++k) {
                const bool here = D.lane == lr && k == kr;
#pragma unroll
                for (int c = 0; c < NS; ++c) S.a[k][c] = selp_f64(-S.a[k][c], S.a[k][c], here);
                S.rhs[k] = selp_f64(-S.rhs[k], S.rhs[k], here);
                if (here) {
                    S.ppart[k] = S.basis[k];
                    S.basis[k] = j;
                }
            }
            __syncwarp();
            continue;
        }
        double av[RPL];
#pragma unroll
        for (int k = 0; k < RPL; ++k) {
            double v = reg_pick<NS>(S.a[k], w.s);
            if (w.partner) v = -v;
            av[k] = D.lane + 32 * k < D.m ? v : 0.0;
        }
        const double pe = __shfl_sync(kFull, ct_row_sel<RPL>(av, kr), lr);
        const double rr = __shfl_sync(kFull, div_entry(ct_row_sel<RPL>(S.rhs, kr), pe), lr);
        ct_pivot<RPL, NS>(D, S, smem, j, w.s, w.partner, row, av, pe, 0.0, rr);
    }
}

// build_tableau (tableau.py:139-172): rows straight into their lane, validation fused
// (a non-finite A, b or c entry sets `nonfinite`); slot q starts as structural x_q with
// reduced cost c_q (0 without c: the shared phase-1 prologue).  Returns n_art.
template <int RPL, int NS, bool V2 = false>
__device__ __forceinline__ int ct_build(const CtDims &D, CtState<RPL, NS> &S, const double *Ag, const double *bg,
                                        const double *cg, bool &nonfinite, int lda = -1) {
    if (lda < 0) lda = D.n;
    constexpr int SPL = CtCfg<RPL, NS>::SPL;
    const int m = D.m, n = D.n, nvc = D.nvc;
    unsigned negm[RPL];
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
        const int row = D.lane + 32 * k;
        const bool live = row < m;
        const double bi = live ? bg[row] : 0.0;
        nonfinite |= !isfinite(bi);
        const bool neg = live && bi < 0.0;
        negm[k] = __ballot_sync(kFull, neg);
        const double sgn = neg ? -1.0 : 1.0;
        S.rhs[k] = live ? __dmul_rn(bi, sgn) : 0.0;
        const double *arow = Ag + (size_t)(live ? row : 0) * lda;
        if constexpr (V2) {     // n even, 16-byte aligned rows (the TMA-staged copy)
#pragma unroll
            for (int c = 0; c < NS; c += 2) {
                double v0 = 0.0, v1 = 0.0;
                if (live && c < n) {
                    const double2 x = *reinterpret_cast<const double2 *>(arow + c);
                    nonfinite |= !(isfinite(x.x) && isfinite(x.y));
                    v0 = __dmul_rn(x.x, sgn);
                    v1 = __dmul_rn(x.y, sgn);
                }
                S.a[k][c] = v0;
                if (c + 1 < NS) S.a[k][c + 1] = v1;
            }
        } else {
#pragma unroll
            for (int c = 0; c < NS; ++c) {
                double v = 0.0;
                if (live && c < n) {
                    const double x = arow[c];
                    nonfinite |= !isfinite(x);
                    v = __dmul_rn(x, sgn);
                }
                S.a[k][c] = v;
            }
        }
    }
    int n_art = 0;
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
        const int row = D.lane + 32 * k;
        const bool neg = (negm[k] >> D.lane) & 1u;
        const int art = n_art + __popc(negm[k] & ((1u << D.lane) - 1u));
        S.basis[k] = neg ? nvc + art : n + row;
        S.ppart[k] = neg ? n + row : -1;      // the negated row's slack: column -e_row
        S.prc[k] = 0.0;
        n_art += __popc(negm[k]);
    }
#pragma unroll
    for (int u = 0; u < SPL; ++u) {
        const int q = D.lane + 32 * u;
        S.svar[u] = q;                         // slot q: structural x_q
        S.spart[u] = -1;
        S.rc[u] = (cg && q < n) ? cg[q] : 0.0;
        S.rcp[u] = 0.0;
        if (cg && q < n) nonfinite |= !isfinite(S.rc[u]);
    }
    S.obj = 0.0;
    return n_art;
}

// Phase 1 (simplex.py:168-178): build_auxiliary, _run_phase, the infeasibility test and
// restore_objective.  c-independent: the objective is -1 on the artificials.  Returns
// the status if the LP ends here (else kOptimal) and the phase-1 iterations in it1.
template <int RPL, int NS>
__device__ __forceinline__ int ct_phase1(const CtDims &D, CtState<RPL, NS> &S, unsigned char *smem,
                                         const Limits &lim, int &it1) {
    ct_price_out<RPL, NS, true>(D, S, smem, nullptr);
    const WlpPhase p1 = ct_run_phase<RPL, NS, true>(D, S, smem, lim);
    it1 = p1.iters;
    if (p1.state == 2) return kIterationLimit;
    if (p1.state == 1) return kErrPhase1Unbounded;
    if (fabs(S.obj) > kPhase1ZeroTol) return kInfeasible;
    ct_restore<RPL, NS>(D, S, smem);
    return kOptimal;
}

// Shared phase 1 (support-function mode, one A and b for every direction): phase 1 and
// restore_objective depend only on A and b, so the prologue runs them
// once and every direction starts from the restored condensed tableau (L2-resident, read
// coalesced: field-major, lane-minor) with its own price-out of c.
template <int RPL, int NS>
struct CtP1 {
    static constexpr int SPL = CtCfg<RPL, NS>::SPL;
    static constexpr int ND = RPL * NS + 2 * RPL;          // a, rhs, prc
    static constexpr int NI = 2 * RPL + 2 * SPL;           // basis, ppart, svar, spart
    static constexpr size_t BYTES = 32 * (ND * 8 + NI * 4) + 16;
    // info (4 ints after the state): [0] status of phase 1 (kOptimal = continue),
    // [1] phase-1 iterations, [2] mode (0: no b < 0 -- directions build as usual, 1: shared)
};

template <int RPL, int NS>
__device__ __forceinline__ void ct_dump(const CtDims &D, const CtState<RPL, NS> &S, double *st) {
    using P = CtP1<RPL, NS>;
    int *si = reinterpret_cast<int *>(st + 32 * P::ND);
    const int l = D.lane;
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
#pragma unroll
        for (int c = 0; c < NS; ++c) st[(k * NS + c) * 32 + l] = S.a[k][c];
        st[(RPL * NS + k) * 32 + l] = S.rhs[k];
        st[(RPL * NS + RPL + k) * 32 + l] = S.prc[k];
        si[k * 32 + l] = S.basis[k];
        si[(RPL + k) * 32 + l] = S.ppart[k];
    }
#pragma unroll
    for (int u = 0; u < P::SPL; ++u) {
        si[(2 * RPL + u) * 32 + l] = S.svar[u];
        si[(2 * RPL + P::SPL + u) * 32 + l] = S.spart[u];
    }
}

template <int RPL, int NS>
__device__ __forceinline__ void ct_load(const CtDims &D, CtState<RPL, NS> &S, const double *st) {
    using P = CtP1<RPL, NS>;
    const int *si = reinterpret_cast<const int *>(st + 32 * P::ND);
    const int l = D.lane;
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
#pragma unroll
        for (int c = 0; c < NS; ++c) S.a[k][c] = st[(k * NS + c) * 32 + l];
        S.rhs[k] = st[(RPL * NS + k) * 32 + l];
        S.prc[k] = st[(RPL * NS + RPL + k) * 32 + l];
        S.basis[k] = si[k * 32 + l];
        S.ppart[k] = si[(RPL + k) * 32 + l];
    }
#pragma unroll
    for (int u = 0; u < P::SPL; ++u) {
        S.svar[u] = si[(2 * RPL + u) * 32 + l];
        S.spart[u] = si[(2 * RPL + P::SPL + u) * 32 + l];
    }
    S.obj = 0.0;
}

// One warp: the shared polytope's phase 1 into `st` (support mode only).
template <int RPL, int NS>
__global__ void __launch_bounds__(32, 1) condensed_phase1_kernel(Batch B, double *st) {
    extern __shared__ __align__(16) unsigned char smem[];
    using C = CtCfg<RPL, NS>;
    int *info = reinterpret_cast<int *>(st + 32 * CtP1<RPL, NS>::ND) + 32 * CtP1<RPL, NS>::NI;
    CtDims D;
    D.m = B.m; D.n = B.n; D.nvc = B.n + B.m; D.lane = threadIdx.x;
    for (int q = D.lane; q < NS; q += 32) reinterpret_cast<double *>(smem + C::RVEC)[q] = 0.0;
    CtState<RPL, NS> S;
    bool nonfinite = false;
    const int n_art = ct_build<RPL, NS>(D, S, B.A, B.b, nullptr, nonfinite);
    const bool invalid = __any_sync(kFull, nonfinite);
    int status = kOptimal, it1 = 0;
    if (invalid) status = kInvalid;
    else if (n_art > 0) status = ct_phase1<RPL, NS>(D, S, smem, B.lim, it1);
    ct_dump<RPL, NS>(D, S, st);
    if (D.lane == 0) {
        info[0] = status;
        info[1] = it1;
        info[2] = (invalid || n_art > 0) ? 1 : 0;
    }
}

template <int RPL, int NS, int kMinBlocks>
__global__ void __launch_bounds__(32, kMinBlocks)
condensed_kernel(Batch B) {
    using C = CtCfg<RPL, NS>;
    constexpr int SPL = C::SPL;
    extern __shared__ __align__(16) unsigned char smem[];
    CtDims D;
    D.m = B.m; D.n = B.n; D.nvc = B.n + B.m; D.lane = threadIdx.x;
    const int m = D.m, n = D.n;
    {
        double *rvec = reinterpret_cast<double *>(smem + C::RVEC);
        for (int q = D.lane; q < NS; q += 32) rvec[q] = 0.0;   // unused slots read as 0
    }
    CtState<RPL, NS> S;
    // TMA staging (the launch granted STG_END bytes): LP k+1's A is bulk-copied into shared
    // memory (one cp.async.bulk per row, completion on an mbarrier) while LP k solves; the
    // build then reads it with 128-bit shared loads instead of per-lane strided global rows.
    unsigned dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    const bool stg = dyn >= C::STG_END && !B.shared_Ab && (n & 1) == 0 &&
                     (reinterpret_cast<uintptr_t>(B.A) & 15) == 0 && m <= 32 * RPL && n <= NS;
    const unsigned sbar = (unsigned)__cvta_generic_to_shared(smem + C::STG_BAR);
    const unsigned sbuf = (unsigned)__cvta_generic_to_shared(smem + C::STG);
    const int lda = n + 2;             // staged row stride (doubles)
    unsigned sphase = 0;
    auto stage = [&](long long q) {
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // the build's reads before the overwrite
        if (D.lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"((unsigned)(m * n * 8))
                         : "memory");
        __syncwarp();
        const double *src = B.A + (size_t)q * m * n;
        for (int r = D.lane; r < m; r += 32)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(sbuf + (unsigned)(r * lda * 8)), "l"(src + (size_t)r * n), "r"((unsigned)(n * 8)), "r"(sbar)
                         : "memory");
    };
    long long lp = 0;
    if (D.lane == 0) lp = atomicAdd(B.next_lp, 1);
    lp = __shfl_sync(kFull, lp, 0);
    if (stg) {
        if (D.lane == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        if (lp < B.count) stage(lp);
    }
    for (;;) {
        if (lp >= B.count) break;
        long long nxt = 0;                 // claim the next LP and warm L2 with its inputs
        if (D.lane == 0) nxt = atomicAdd(B.next_lp, 1);
        nxt = __shfl_sync(kFull, nxt, 0);
        if (nxt < B.count) {
            if (!stg) prefetch_lp_inputs(B, nxt, D.lane);
            else if (D.lane == 0) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(B.b + (size_t)nxt * m));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(B.c + (size_t)nxt * n));
            }
        }
        const double *Ag = B.shared_Ab ? B.A : B.A + (size_t)lp * m * n;
        const double *bg = B.shared_Ab ? B.b : B.b + (size_t)lp * m;
        const double *cg = B.c + (size_t)lp * n;

        int8_t status = kOptimal;
        int it1 = 0, it2 = 0;
        bool done = false;
        // support mode with b < 0: phase 1 was solved once by condensed_phase1_kernel (its info
        // block is re-read per LP -- an L1 hit -- rather than held in registers across the solve)
        const int *p1info = B.p1state ? reinterpret_cast<const int *>(B.p1state + 32 * CtP1<RPL, NS>::ND) +
                                        32 * CtP1<RPL, NS>::NI : nullptr;
        if (p1info && p1info[2] == 1) {
            const int p1status = p1info[0], p1iters = p1info[1];
            bool nonfinite = false;
#pragma unroll
            for (int u = 0; u < SPL; ++u)
                if (D.lane + 32 * u < n) nonfinite |= !isfinite(cg[D.lane + 32 * u]);
            if (__any_sync(kFull, nonfinite) || p1status == kInvalid) {
                status = kInvalid;
                done = true;
            } else if (p1status != kOptimal) {
                status = (int8_t)p1status;
                it1 = p1iters;
                done = true;
            } else {
                it1 = p1iters;
                ct_load<RPL, NS>(D, S, B.p1state);
                ct_price_out<RPL, NS, false>(D, S, smem, cg);
            }
        } else {
            bool nonfinite = false;
            int n_art;
            if (stg) {
                unsigned done;
                do {
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                 : "=r"(done) : "r"(sbar), "r"(sphase) : "memory");
                } while (!done);
                sphase ^= 1u;
                n_art = ct_build<RPL, NS, true>(D, S, reinterpret_cast<const double *>(smem + C::STG), bg, cg, nonfinite,
                                                lda);
                if (nxt < B.count) stage(nxt);   // overlaps this LP's solve
            } else {
                n_art = ct_build<RPL, NS>(D, S, Ag, bg, cg, nonfinite);
            }
            if (__any_sync(kFull, nonfinite)) {
                status = kInvalid;
                done = true;
            } else if (n_art > 0) {
                const int st = ct_phase1<RPL, NS>(D, S, smem, B.lim, it1);
                if (st != kOptimal) { status = (int8_t)st; done = true; }
                else ct_price_out<RPL, NS, false>(D, S, smem, cg);
            } else {
                ct_candidates<RPL, NS, false>(D, S);
            }
        }
        if (!done) {
            const WlpPhase p2 = ct_run_phase<RPL, NS, false>(D, S, smem, B.lim);
            it2 = p2.iters;
            if (p2.state == 2) status = kIterationLimit;
            else if (p2.state == 1) status = kUnbounded;
        }

        // ---- _extract_point (simplex.py:146-151) and c @ x ----
        double *xs = reinterpret_cast<double *>(smem + C::XS);    // n <= NS doubles
        double *xg = B.x + (size_t)lp * n;
        __syncwarp();
        for (int j = D.lane; j < n; j += 32) xs[j] = 0.0;
        __syncwarp();
        if (status == kOptimal) {
#pragma unroll
            for (int k = 0; k < RPL; ++k)
                if (D.lane + 32 * k < m && S.basis[k] < n) xs[S.basis[k]] = S.rhs[k];
        }
        __syncwarp();
        for (int j = D.lane; j < n; j += 32) xg[j] = xs[j];
        if (D.lane == 0) {
            double obj = __longlong_as_double(0x7ff8000000000000LL);
            if (status == kOptimal) {
                obj = 0.0;
                for (int j = 0; j < n; ++j) obj = __dadd_rn(obj, __dmul_rn(cg[j], xs[j]));
            }
            B.objective[lp] = obj;
        }
        if (D.lane == 0) {
            B.status[lp] = status;
            B.it1[lp] = it1;
            B.it2[lp] = it2;
        }
        __syncwarp();
        lp = nxt;
    }
}

}  // namespace blp
