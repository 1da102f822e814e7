// blp_tableau_kernel.cuh -- persistent CTA-per-LP two-phase dense simplex.
//
// One CTA owns one LP at a time and pulls the next LP index from an atomic
// queue when it finishes (LPs finish after very different pivot counts, so
// a static split would leave SMs idle).  Inside the CTA:
//
//   * the tableau is the reference's column-major tableau (tableau.py:56-79)
//     WITHOUT the artificial columns: [x (n) | s (m) | rhs], (m+1) rows, the
//     last row holding the reduced costs.  Artificial column k is value-equal
//     to minus the slack column of its row at every step (both start as
//     -/+e_i and every pivot applies sign-symmetric IEEE ops), so only its
//     phase-1 reduced cost is kept, in art_rc[k];
//   * kSmemTab: the tableau lives in shared memory (fits up to ~227 KB),
//     otherwise in a per-CTA HBM slot (streamed each pivot);
//   * warp w owns columns j = w, w+NW, ...; lane L owns rows L, L+32, ...
//     (RPL row slots).  The rank-1 update, the pivot-row division and the
//     next entering candidate are all computed by the column's owner warp,
//     so one pivot costs two CTA barriers:
//        B2: leaving-row argmin partials + snapshot of the entering column
//        B4: updated columns + entering-column argmax partials.
//
// Reference call graph mirrored: solve (simplex.py:154-194) -> build_tableau
// (tableau.py:139-172) -> build_auxiliary/_price_out (simplex.py:94-106,
// 133-143) -> _run_phase (simplex.py:63-91: choose_entering[_bland],
// choose_leaving, pivot = tableau.py:175-244) -> restore_objective
// (simplex.py:109-130) -> _run_phase -> _extract_point (simplex.py:146-151).
#pragma once

#include "blp_common.cuh"
#include "blp_keys.cuh"

namespace blp {

// Shared-memory carve-up; identical on host (sizing) and device.
struct TabLayout {
    int ld;          // leading dimension (rows, padded to even)
    int ncols;       // n + m + 1
    size_t off_T, off_f, off_r, off_artrc, off_cbv, off_cval, off_lval;
    size_t off_cidx, off_cbl, off_lrow, off_basis, off_artrow, off_artof, off_misc, off_wcnt, off_isb;
    size_t bytes;
};

__host__ __device__ inline size_t tl_align(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline TabLayout make_tab_layout(int m, int n, int nwarps, bool smem_tab) {
    TabLayout L;
    L.ld = (m + 3) & ~1;   // >= m+2: row m+1 is a spare row (see pivot_update)
    L.ncols = n + m + 1;
    const int mm = m > 0 ? m : 1;
    size_t o = 0;
    L.off_T = o;      o += smem_tab ? (size_t)L.ncols * L.ld * sizeof(double) : 0;
    L.off_f = o;      o = tl_align(o + (size_t)L.ld * sizeof(double), 16);
    L.off_r = o;      o = tl_align(o + (size_t)L.ncols * sizeof(double), 16);
    L.off_artrc = o;  o = tl_align(o + (size_t)mm * sizeof(double), 16);
    L.off_cbv = o;    o = tl_align(o + (size_t)mm * sizeof(double), 16);
    L.off_cval = o;   o = tl_align(o + 32 * sizeof(double), 16);
    L.off_lval = o;   o = tl_align(o + 32 * sizeof(double), 16);
    L.off_cidx = o;   o = tl_align(o + 32 * sizeof(int), 16);
    L.off_cbl = o;    o = tl_align(o + 32 * sizeof(int), 16);
    L.off_lrow = o;   o = tl_align(o + 32 * sizeof(int), 16);
    L.off_basis = o;  o = tl_align(o + (size_t)mm * sizeof(int), 16);
    L.off_artrow = o; o = tl_align(o + (size_t)mm * sizeof(int), 16);
    L.off_artof = o;  o = tl_align(o + (size_t)mm * sizeof(int), 16);
    L.off_misc = o;   o = tl_align(o + 8 * sizeof(long long), 16);
    L.off_wcnt = o;   o = tl_align(o + 32 * sizeof(int), 16);
    L.off_isb = o;    o = tl_align(o + (size_t)(n + 2 * mm), 16);
    (void)nwarps;
    L.bytes = o;
    return L;
}

enum UpdateKind { kRestore = 0, kPhase1 = 1, kPhase2 = 2 };

template <int RPL>
struct TabCtx {
    // dims
    int m, n, nvc, rhs, ld, ncols, n_art;
    int tid, lane, warp, nw, nt;
    // storage
    double *T;        // tableau, column-major, ld rows per column
    double *fvec;     // snapshot of the entering column (rows 0..m)
    double *rvec;     // pivot row / pe, written and read by the owning warp only
    double *art_rc;   // phase-1 reduced costs of the artificial columns
    double *cbv;      // basic costs during price-out
    unsigned long long *ckey;  // per-warp entering candidates (key, index, Bland index)
    int *cidx, *cbl;
    unsigned long long *lkey;  // per-warp leaving candidates (ratio key, row)
    int *lrow;
    int *basis, *art_row, *art_of;
    long long *misc;
    int *wcnt;
    unsigned char *isb;
};

// ---------------------------------------------------------------------------
// Arg-reductions on numpy-order keys (blp_keys.cuh): per-warp partials are
// (key, index) pairs in smem; every warp reduces them after a barrier.

// Per-thread running best for the entering choice: Dantzig (max key, lowest
// index) and Bland (lowest index with rc > tol).
struct EnterBest {
    unsigned long long k = kKeyEmptyMax;
    int i = kNone, bl = kNone;
    __device__ __forceinline__ void add(double v, int j) {
        const unsigned long long kv = key_max(v);
        if (kv > k || (kv == k && j < i)) { k = kv; i = j; }
        if (v > kTol && j < bl) bl = j;
    }
};

template <int RPL>
__device__ __forceinline__ void publish_candidates(const TabCtx<RPL> &X, const EnterBest &b) {
    const unsigned long long kw = warp_max_key(b.k);
    const int iw = warp_index_of(b.k, kw, b.i);
    const int bw = warp_min_int(b.bl);
    if (X.lane == 0) { X.ckey[X.warp] = kw; X.cidx[X.warp] = iw; X.cbl[X.warp] = bw; }
}

// choose_entering (tableau.py:175-186) / choose_entering_bland (:189-197).
template <int RPL>
__device__ __forceinline__ int select_entering(const TabCtx<RPL> &X, bool use_bland) {
    unsigned long long k = kKeyEmptyMax;
    int i = kNone, b = kNone;
    if (X.lane < X.nw) { k = X.ckey[X.lane]; i = X.cidx[X.lane]; b = X.cbl[X.lane]; }
    const unsigned long long kw = warp_max_key(k);
    const int e = warp_index_of(k, kw, i);
    const int bl = warp_min_int(b);
    if (use_bland) return bl == kNone ? -1 : bl;
    if (e == kNone || kw <= key_max(kTol)) return -1;   // NaN keys sort above tol, as numpy
    return e;
}

// ---------------------------------------------------------------------------
// Rank-1 pivot update on the columns this warp owns (pivot, tableau.py:218-244).
// Preconditions: fvec holds column e (rows 0..m) as it was before the pivot;
// every thread knows (e, l, pe, fm = reduced cost of e, oldvar = basis[l]).
//   1. lane k divides the pivot-row entry of the warp's k-th column;
//   2. a_ij <- a_ij - f_i * r_j on every owned cell (f_l = 0 leaves row l);
//   3. lane k writes r_j into row l of its column (numpy: r_j - 0*r_j == r_j);
//   4. lane k finishes column k's objective cell: the reduced cost it now holds
//      is tested as the next entering candidate (plus, in phase 1, the paired
//      artificial's), the rhs column gets obj_before + rc_e * r_rhs (tableau.py:242).
template <int RPL, int KIND>
__device__ __forceinline__ void pivot_update(const TabCtx<RPL> &X, int e, int l, double pe,
                                             double fm, int oldvar) {
    const int m = X.m, ld = X.ld;
    double obj_before = 0.0;
    for (int k = X.lane;; k += 32) {
        const int j = X.warp + X.nw * k;
        if (j >= X.ncols) break;
        X.rvec[j] = div_entry(X.T[(size_t)j * ld + l], pe);
        if (j == X.rhs) obj_before = X.T[(size_t)j * ld + m];
    }
    __syncwarp();
    double fr[RPL];
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
        const int i = X.lane + 32 * s;
        fr[s] = (i <= m && i != l) ? X.fvec[i] : 0.0;
    }
    // Lanes past the last row all address the spare row m+1 (ld >= m+2) with
    // factor 0: a benign same-value store, and no per-slot branch in the loop.
    {
        int roff[RPL];
#pragma unroll
        for (int s = 0; s < RPL; ++s) roff[s] = min(X.lane + 32 * s, m + 1);
        double *col = X.T + (size_t)X.warp * ld;
        const size_t cstride = (size_t)ld * X.nw;
        for (int j = X.warp; j < X.ncols; j += X.nw, col += cstride) {
            const double rj = X.rvec[j];
            double a[RPL];
#pragma unroll
            for (int s = 0; s < RPL; ++s) a[s] = col[roff[s]];
#pragma unroll
            for (int s = 0; s < RPL; ++s) col[roff[s]] = __dsub_rn(a[s], __dmul_rn(fr[s], rj));
        }
    }
    __syncwarp();
    // row l <- r, one column per lane (after the update wrote row l unchanged)
    for (int k = X.lane;; k += 32) {
        const int j = X.warp + X.nw * k;
        if (j >= X.ncols) break;
        X.T[(size_t)j * ld + l] = X.rvec[j];
    }
    __syncwarp();
    EnterBest best;
    for (int k = X.lane;; k += 32) {
        const int j = X.warp + X.nw * k;
        if (j >= X.ncols) break;
        const double rj = X.rvec[j];
        if (j == X.rhs) {
            X.T[(size_t)j * ld + m] = __dadd_rn(obj_before, __dmul_rn(fm, rj));
        } else if (KIND != kRestore) {
            const bool basic = (j == e) || (j != oldvar && X.isb[j]);
            if (!basic) best.add(X.T[(size_t)j * ld + m], j);
            if (KIND == kPhase1 && j >= X.n) {
                const int k2 = X.art_of[j - X.n];
                if (k2 >= 0) {
                    // artificial k2 = -(slack column of its row): pivot-row entry -r_j exactly
                    const double nr = __dsub_rn(X.art_rc[k2], __dmul_rn(fm, -rj));
                    X.art_rc[k2] = nr;
                    const int ja = X.nvc + k2;
                    if (!((ja == e) || (ja != oldvar && X.isb[ja]))) best.add(nr, ja);
                }
            }
        }
    }
    if (KIND != kRestore) publish_candidates(X, best);
}

// ---------------------------------------------------------------------------
// _price_out (simplex.py:133-143): rebuild the objective row against the
// current basis, sequential over rows exactly as the reference, one thread
// per column.  PHASE 1: c_aux = -1 on artificials (build_auxiliary,
// simplex.py:94-106).  PHASE 2: c_ext[:n] = c (restore_objective, :127-129).
// Ends with the entering candidates published and a barrier.
template <int RPL, int PHASE>
__device__ void price_out(const TabCtx<RPL> &X, const double *cg) {
    const int m = X.m, ld = X.ld;
    for (int i = X.tid; i < m; i += X.nt) {
        const int bv = X.basis[i];
        double cb;
        if (PHASE == 1) cb = bv >= X.nvc ? -1.0 : 0.0;
        else cb = bv < X.n ? cg[bv] : 0.0;
        X.cbv[i] = cb;
    }
    __syncthreads();
    EnterBest best;
    const int nart = PHASE == 1 ? X.n_art : 0;
    const int total = X.nvc + nart + 1;
    for (int q = X.tid; q < total; q += X.nt) {
        if (q < X.nvc) {
            const double *col = X.T + (size_t)q * ld;
            double rc = (PHASE == 2 && q < X.n) ? cg[q] : 0.0;
            for (int r = 0; r < m; ++r) {
                const double cb = X.cbv[r];
                if (cb != 0.0) rc = __dsub_rn(rc, __dmul_rn(cb, col[r]));
            }
            X.T[(size_t)q * ld + m] = rc;
            if (!X.isb[q]) best.add(rc, q);
        } else if (q < X.nvc + nart) {
            const int k = q - X.nvc;
            const double *scol = X.T + (size_t)(X.n + X.art_row[k]) * ld;
            double rc = -1.0;
            for (int r = 0; r < m; ++r) {
                const double cb = X.cbv[r];
                if (cb != 0.0) rc = __dsub_rn(rc, __dmul_rn(cb, -scol[r]));
            }
            X.art_rc[k] = rc;
            if (!X.isb[q]) best.add(rc, q);
        } else {
            const double *col = X.T + (size_t)X.rhs * ld;
            double obj = 0.0;
            for (int r = 0; r < m; ++r) {
                const double cb = X.cbv[r];
                if (cb != 0.0) obj = __dadd_rn(obj, __dmul_rn(cb, col[r]));
            }
            X.T[(size_t)X.rhs * ld + m] = obj;
        }
    }
    publish_candidates(X, best);
    __syncthreads();
}

// Candidates straight from the initial objective row (feasible start: the
// reference runs phase 2 on c without a price-out, simplex.py:168,180).
template <int RPL>
__device__ void initial_candidates(const TabCtx<RPL> &X) {
    EnterBest best;
    for (int j = X.tid; j < X.nvc; j += X.nt)
        if (!X.isb[j]) best.add(X.T[(size_t)j * X.ld + X.m], j);
    publish_candidates(X, best);
    __syncthreads();
}

struct PhaseResult { int state; int iters; };  // state: 0 optimal, 1 unbounded, 2 limit

// _run_phase (simplex.py:63-91).  Entry: candidates published + barrier.
template <int RPL, int KIND>
__device__ PhaseResult run_phase(const TabCtx<RPL> &X, const Limits &lim) {
    const int m = X.m, ld = X.ld;
    const int max_iter = lim.max_iterations > 0 ? lim.max_iterations : 50 * (m + X.n);
    const int trigger = lim.degenerate_limit >= 0 ? lim.degenerate_limit : (m > 1 ? m : 1);
    const unsigned long long kSent = key_max(kSentinel), kDeg = key_max(kDegenerateTol);
    int degenerate_run = 0;
    bool use_bland = false;
    for (int it = 0;; ++it) {
        if (it == max_iter) return {2, max_iter};
        const int e = select_entering(X, use_bland);
        if (e < 0) return {0, it};
        // choose_leaving (tableau.py:200-215) + snapshot of column e
        const bool art_e = e >= X.nvc;
        const double *ecol = X.T + (size_t)(art_e ? X.n + X.art_row[e - X.nvc] : e) * ld;
        const double *rcol = X.T + (size_t)X.rhs * ld;
        unsigned long long lk = kKeyEmptyMin;
        int li = kNone;
        for (int i = X.tid; i < m; i += X.nt) {
            const double a = art_e ? -ecol[i] : ecol[i];
            X.fvec[i] = a;
            const unsigned long long k = key_min(ratio_entry(rcol[i], a));
            if (k < lk) { lk = k; li = i; }     // rows ascend per thread
        }
        if (X.tid == 0) X.fvec[m] = art_e ? X.art_rc[e - X.nvc] : ecol[m];
        {
            const unsigned long long kw = warp_min_key(lk);
            const int iw = warp_index_of(lk, kw, li);
            if (X.lane == 0) { X.lkey[X.warp] = kw; X.lrow[X.warp] = iw; }
        }
        __syncthreads();  // B2
        unsigned long long k = kKeyEmptyMin;
        int i = kNone;
        if (X.lane < X.nw) { k = X.lkey[X.lane]; i = X.lrow[X.lane]; }
        const unsigned long long kmin = warp_min_key(k);
        const int l = warp_index_of(k, kmin, i);
        if (l == kNone || kmin >= kSent) return {1, it};   // a NaN ratio keys to 0
        const int oldvar = X.basis[l];
        const double pe = X.fvec[l];
        const double fm = X.fvec[m];
        if (kmin != 0ull && kmin <= kDeg) {                 // simplex.py:84-90
            ++degenerate_run;
            if (lim.anti_cycling && degenerate_run >= trigger) use_bland = true;
        } else {
            degenerate_run = 0;
            use_bland = false;
        }
        pivot_update<RPL, KIND>(X, e, l, pe, fm, oldvar);
        __syncthreads();  // B4
        if (X.tid == 0) { X.basis[l] = e; X.isb[oldvar] = 0; X.isb[e] = 1; }
    }
}

// restore_objective pivot-outs (simplex.py:109-126); uncounted pivots.
template <int RPL>
__device__ void restore_basis(const TabCtx<RPL> &X) {
    const int m = X.m, ld = X.ld;
    const unsigned long long kRed = key_max(kRedundantTol);
    __syncthreads();
    for (int row = 0; row < m; ++row) {
        if (X.basis[row] < X.nvc) continue;   // uniform: basis is stable here
        unsigned long long bk = kKeyEmptyMax;
        int bj = kNone;
        for (int j = X.tid; j < X.nvc; j += X.nt) {
            const unsigned long long k = key_max(fabs(X.T[(size_t)j * ld + row]));
            if (k > bk) { bk = k; bj = j; }     // columns ascend per thread
        }
        {
            const unsigned long long kw = warp_max_key(bk);
            const int jw = warp_index_of(bk, kw, bj);
            if (X.lane == 0) { X.ckey[X.warp] = kw; X.cidx[X.warp] = jw; }
        }
        __syncthreads();
        unsigned long long k = kKeyEmptyMax;
        int jj = kNone;
        if (X.lane < X.nw) { k = X.ckey[X.lane]; jj = X.cidx[X.lane]; }
        const unsigned long long kbest = warp_max_key(k);
        const int j = warp_index_of(k, kbest, jj);
        // entries[j] > REDUNDANT_ROW_TOL; a NaN entry compares False in numpy
        if (j != kNone && kbest > kRed && kbest != ~0ull) {
            for (int i = X.tid; i <= m; i += X.nt) X.fvec[i] = X.T[(size_t)j * ld + i];
            __syncthreads();
            const int oldvar = X.basis[row];
            pivot_update<RPL, kRestore>(X, j, row, X.fvec[row], X.fvec[m], oldvar);
            __syncthreads();
            if (X.tid == 0) { X.basis[row] = j; X.isb[oldvar] = 0; X.isb[j] = 1; }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
template <int RPL, bool kSmemTab, int kMaxThreads>
__global__ void __launch_bounds__(kMaxThreads)
tableau_kernel(Batch B) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int m = B.m, n = B.n;
    const int nw = blockDim.x >> 5;
    const TabLayout L = make_tab_layout(m, n, nw, kSmemTab);
    TabCtx<RPL> X;
    X.m = m; X.n = n; X.nvc = n + m; X.rhs = n + m; X.ld = L.ld; X.ncols = L.ncols;
    X.tid = threadIdx.x; X.lane = threadIdx.x & 31; X.warp = threadIdx.x >> 5;
    X.nw = nw; X.nt = blockDim.x;
    X.T = kSmemTab ? reinterpret_cast<double *>(smem + L.off_T)
                   : B.gtab + (size_t)blockIdx.x * (size_t)B.gtab_stride;
    X.fvec = reinterpret_cast<double *>(smem + L.off_f);
    X.rvec = reinterpret_cast<double *>(smem + L.off_r);
    X.art_rc = reinterpret_cast<double *>(smem + L.off_artrc);
    X.cbv = reinterpret_cast<double *>(smem + L.off_cbv);
    X.ckey = reinterpret_cast<unsigned long long *>(smem + L.off_cval);
    X.lkey = reinterpret_cast<unsigned long long *>(smem + L.off_lval);
    X.cidx = reinterpret_cast<int *>(smem + L.off_cidx);
    X.cbl = reinterpret_cast<int *>(smem + L.off_cbl);
    X.lrow = reinterpret_cast<int *>(smem + L.off_lrow);
    X.basis = reinterpret_cast<int *>(smem + L.off_basis);
    X.art_row = reinterpret_cast<int *>(smem + L.off_artrow);
    X.art_of = reinterpret_cast<int *>(smem + L.off_artof);
    X.misc = reinterpret_cast<long long *>(smem + L.off_misc);
    X.wcnt = reinterpret_cast<int *>(smem + L.off_wcnt);
    X.isb = smem + L.off_isb;
    const int ld = L.ld, nvc = n + m, rhs = n + m;

    for (;;) {
        if (X.tid == 0) { X.misc[0] = atomicAdd(B.next_lp, 1); X.misc[1] = 0; }
        __syncthreads();
        const long long qi = X.misc[0];
        if (qi >= batch_count(B)) break;      // the deferred LPs when launched after the lazy kernel
        const long long lp = batch_lp(B, qi);
        const double *Ag = B.shared_Ab ? B.A : B.A + (size_t)lp * m * n;
        const double *bg = B.shared_Ab ? B.b : B.b + (size_t)lp * m;
        const double *cg = B.c + (size_t)lp * n;

        // ---- build_tableau (tableau.py:139-172) ----
        for (int j = X.tid; j < n + 2 * m; j += X.nt) X.isb[j] = 0;
        bool nonfinite = false;  // validate (model.py:263-301), fused into the load
        for (int base = 0; base < m; base += X.nt) {
            const int i = base + X.tid;
            const double bi = i < m ? bg[i] : 0.0;
            nonfinite |= !isfinite(bi);
            const bool neg = i < m && bi < 0.0;
            const unsigned bal = __ballot_sync(kFull, neg);
            if (X.lane == 0) X.wcnt[X.warp] = __popc(bal);
            __syncthreads();
            int pre = (int)X.misc[1] + __popc(bal & ((1u << X.lane) - 1u));
            for (int w = 0; w < X.warp; ++w) pre += X.wcnt[w];
            if (i < m) {
                const double s = neg ? -1.0 : 1.0;
                X.cbv[i] = s;
                X.T[(size_t)rhs * ld + i] = __dmul_rn(bi, s);
                if (neg) { X.basis[i] = nvc + pre; X.art_row[pre] = i; X.art_of[i] = pre; }
                else { X.basis[i] = n + i; X.art_of[i] = -1; }
            }
            __syncthreads();
            if (X.tid == 0) { int t = 0; for (int w = 0; w < nw; ++w) t += X.wcnt[w]; X.misc[1] += t; }
            __syncthreads();
        }
        X.n_art = (int)X.misc[1];
        for (int k = X.tid; k < m * n; k += X.nt) {
            const int i = k / n, j = k - i * n;
            const double a = Ag[k];
            nonfinite |= !isfinite(a);
            X.T[(size_t)j * ld + i] = __dmul_rn(a, X.cbv[i]);
        }
        for (int k = X.tid; k < m * (m + 1); k += X.nt) {
            const int jj = k / (m + 1), i = k - jj * (m + 1);
            X.T[(size_t)(n + jj) * ld + i] = (i == jj) ? X.cbv[i] : 0.0;
        }
        for (int j = X.tid; j <= n; j += X.nt) {
            const double cj = j < n ? cg[j] : 0.0;
            nonfinite |= !isfinite(cj);
            X.T[(size_t)(j < n ? j : rhs) * ld + m] = cj;
        }
        const bool invalid = __syncthreads_or(nonfinite);
        for (int i = X.tid; i < m; i += X.nt) X.isb[X.basis[i]] = 1;
        __syncthreads();

        int8_t status = kOptimal;
        int it1 = 0, it2 = 0;
        bool done = false;
        if (invalid) {
            status = kInvalid;
            done = true;
        } else if (X.n_art > 0) {
            price_out<RPL, 1>(X, cg);
            const PhaseResult r1 = run_phase<RPL, kPhase1>(X, B.lim);
            __syncthreads();
            it1 = r1.iters;
            if (r1.state == 2) { status = kIterationLimit; done = true; }
            else if (r1.state == 1) { status = kErrPhase1Unbounded; done = true; }
            else if (fabs(X.T[(size_t)rhs * ld + m]) > kPhase1ZeroTol) { status = kInfeasible; done = true; }
            else {
                restore_basis(X);
                price_out<RPL, 2>(X, cg);
            }
        } else {
            initial_candidates(X);
        }
        if (!done) {
            const PhaseResult r2 = run_phase<RPL, kPhase2>(X, B.lim);
            __syncthreads();
            it2 = r2.iters;
            if (r2.state == 2) status = kIterationLimit;
            else if (r2.state == 1) status = kUnbounded;
        }

        // ---- _extract_point (simplex.py:146-151) and c @ x ----
        double *xs = X.rvec;  // ncols >= n doubles of scratch
        double *xg = B.x + (size_t)lp * n;
        for (int j = X.tid; j < n; j += X.nt) xs[j] = 0.0;
        __syncthreads();
        if (status == kOptimal)
            for (int i = X.tid; i < m; i += X.nt) {
                const int bv = X.basis[i];
                if (bv < n) xs[bv] = X.T[(size_t)rhs * ld + i];
            }
        __syncthreads();
        for (int j = X.tid; j < n; j += X.nt) xg[j] = xs[j];
        if (X.tid == 0) {
            double obj = __longlong_as_double(0x7ff8000000000000LL);  // NaN
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
    }
}

}  // namespace blp
