// blp_regtile_kernel.cuh -- register-resident two-phase simplex for LPs with
// m <= 32*RPL constraint rows (the afiro-class C1/C2 shapes and C4's 64 rows).
//
// One CTA of NW warps owns one LP at a time (persistent grid, atomic LP
// queue).  The compact tableau (reference tableau.py:56-79 minus the
// artificial columns, see blp_tableau_kernel.cuh) is split three ways:
//
//   * constraint rows live in REGISTERS: warp w owns column positions
//     [w*CPW, (w+1)*CPW), lane L owns rows L, L+32, ... (RPL slots), so a
//     lane holds an RPL x CPW tile and the rank-1 update is pure DMUL/DADD on
//     registers -- no shared-memory traffic for the O(m*(n+m)) part;
//   * the objective (reduced-cost) row is TRANSPOSED: lane q of warp w holds
//     the reduced cost of position w*CPW+q.  The lane that divides a column's
//     pivot-row entry (r_q = a_lq / pe) is the lane that updates that
//     column's reduced cost and tests it as the next entering candidate, so
//     the argmax is lane-parallel (keyed redux.sync, blp_keys.cuh);
//   * position 0 is the rhs column (warp 0, register slot 0, static), its
//     transposed slot holds the objective value; variable j sits at position j+1.
//
// Per pivot: B4 (updates + per-warp entering candidates) -> every warp
// reduces the candidates -> the owner warp of the entering column runs the
// ratio test and snapshots the column into smem -> B2 -> every warp divides
// its slice of the pivot row and updates its tile.  The pivot row itself is
// produced branch-free: its lane zeroes its registers and uses factor -1, so
// 0 - (-1)*r = r, value-equal to numpy's r - 0*r for every finite r.
//
// Arithmetic: __dmul_rn/__dsub_rn/__dadd_rn/__ddiv_rn only (numpy parity).
#pragma once

#include "blp_common.cuh"
#include "blp_keys.cuh"

namespace blp {

struct RtLayout {
    int nw, cpw, rows, ldg;  // warps, columns per warp, 32*RPL, stage leading dim (odd)
    size_t off_fvec, off_rhs, off_cbv, off_rowbuf, off_rvec, off_ckey, off_cidx, off_cbl, off_basis,
        off_artrow, off_artof, off_wcnt, off_sh, off_stage, bytes;
};

__host__ __device__ inline size_t rt_align(size_t x) { return (x + 15) / 16 * 16; }

__host__ __device__ inline RtLayout make_rt_layout(int rpl, int cpw, int nw) {
    RtLayout L;
    L.nw = nw; L.cpw = cpw; L.rows = 32 * rpl;
    L.ldg = nw * cpw + 1;
    size_t o = 0;
    L.off_fvec = o;   o = rt_align(o + (size_t)L.rows * 8);
    L.off_rhs = o;    o = rt_align(o + (size_t)L.rows * 8);
    L.off_cbv = o;    o = rt_align(o + (size_t)L.rows * 8);
    L.off_rowbuf = o; o = rt_align(o + (size_t)nw * cpw * 8);
    L.off_rvec = o;   o = rt_align(o + (size_t)nw * cpw * 8);
    L.off_ckey = o;   o = rt_align(o + 32 * 8);
    L.off_cidx = o;   o = rt_align(o + 32 * 4);
    L.off_cbl = o;    o = rt_align(o + 32 * 4);
    L.off_basis = o;  o = rt_align(o + (size_t)L.rows * 4);
    L.off_artrow = o; o = rt_align(o + (size_t)L.rows * 4);
    L.off_artof = o;  o = rt_align(o + (size_t)L.rows * 4);
    L.off_wcnt = o;   o = rt_align(o + 32 * 4);
    L.off_sh = o;     o = rt_align(o + 64);
    L.off_stage = o;  o = rt_align(o + (size_t)L.rows * L.ldg * 8);
    L.bytes = o;
    return L;
}

// Per-pivot scalars published by the owner warp of the entering column.
struct RtShared {
    long long lp;
    unsigned long long kmin;   // key of the minimum ratio
    double fm;                 // reduced cost of the entering column
    int e, l, oldvar, n_art;
};

template <int RPL, int CPW>
struct Rt {
    static constexpr int OPW = (CPW + 31) / 32;  // transposed objective slots per lane
    int m, n, nvc, ncols, nw, lane, warp, tid, nt;
    double *fvec, *rhsv, *cbv, *rowbuf, *rvec, *stage;
    unsigned long long *ckey;
    int *cidx, *cbl, *basis, *art_row, *art_of, *wcnt;
    RtShared *sh;
    int ldg;
};

enum { kRtRestore = 0, kRtPhase1 = 1, kRtPhase2 = 2 };

// Per-lane registers of one LP.
template <int RPL, int CPW>
struct RtRegs {
    double a[RPL][CPW];                 // constraint-row tile
    double rc[Rt<RPL, CPW>::OPW];       // transposed objective row (slot of position 0 = objective value)
    double arc[Rt<RPL, CPW>::OPW];      // phase-1 reduced cost of the artificial paired with a slack position
    int artk[Rt<RPL, CPW>::OPW];        // that artificial's index, or -1
    unsigned bas;                       // bit t: variable basic; bit 16+t: paired artificial basic
};

// Publish this warp's entering candidates: Dantzig (max key, lowest index) and Bland (lowest index > tol).
template <int RPL, int CPW, int KIND>
__device__ __forceinline__ void rt_candidates(const Rt<RPL, CPW> &X, const RtRegs<RPL, CPW> &R) {
    unsigned long long ck = kKeyEmptyMax;
    int ci = kNone, cb = kNone;
#pragma unroll
    for (int t = 0; t < Rt<RPL, CPW>::OPW; ++t) {
        const int q = X.lane + 32 * t;
        const int pos = X.warp * CPW + q;
        if (q < CPW && pos >= 1 && pos < X.ncols) {
            const int j = pos - 1;
            if (!(R.bas & (1u << t))) {
                const unsigned long long k = key_max(R.rc[t]);
                if (k > ck || (k == ck && j < ci)) { ck = k; ci = j; }
                if (R.rc[t] > kTol && j < cb) cb = j;
            }
            if (KIND == kRtPhase1 && R.artk[t] >= 0 && !(R.bas & (0x10000u << t))) {
                const int ja = X.nvc + R.artk[t];
                const unsigned long long k = key_max(R.arc[t]);
                if (k > ck || (k == ck && ja < ci)) { ck = k; ci = ja; }
                if (R.arc[t] > kTol && ja < cb) cb = ja;
            }
        }
    }
    const unsigned long long kw = warp_max_key(ck);
    const int iw = warp_index_of(ck, kw, ci);
    const int bw = (int)__reduce_min_sync(kFull, (unsigned)cb);
    if (X.lane == 0) { X.ckey[X.warp] = kw; X.cidx[X.warp] = iw; X.cbl[X.warp] = bw; }
}

// choose_entering / choose_entering_bland (tableau.py:175-197) from the per-warp candidates.
template <int RPL, int CPW>
__device__ __forceinline__ int rt_select_entering(const Rt<RPL, CPW> &X, bool use_bland) {
    unsigned long long k = kKeyEmptyMax;
    int i = kNone, b = kNone;
    if (X.lane < X.nw) { k = X.ckey[X.lane]; i = X.cidx[X.lane]; b = X.cbl[X.lane]; }
    const unsigned long long kw = warp_max_key(k);
    const int e = warp_index_of(k, kw, i);
    const int bl = (int)__reduce_min_sync(kFull, (unsigned)b);
    if (use_bland) return bl == kNone ? -1 : bl;
    if (e == kNone || kw <= key_max(kTol)) return -1;   // NaN keys are above tol: numpy returns them
    return e;
}

__device__ __forceinline__ void rt_barrier(int nw) {
    if (nw > 1) __syncthreads(); else __syncwarp();
}

// Owner warp of position `epos`: snapshot the column into fvec (negated for an
// artificial) and, if want_ratio, run choose_leaving (tableau.py:200-215).
template <int RPL, int CPW>
__device__ __forceinline__ void rt_owner_column(const Rt<RPL, CPW> &X, const RtRegs<RPL, CPW> &R, int e,
                                                int epos, bool art_e, int given_l) {
    const int ce = epos - X.warp * CPW;
    unsigned long long lk = kKeyEmptyMin;
    int lr = kNone;
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
        double av = reg_pick<CPW>(R.a[s], ce);
        if (art_e) av = -av;
        const int r = X.lane + 32 * s;
        if (r < X.m) {
            X.fvec[r] = av;
            if (given_l < 0) {
                const double ratio = ratio_entry(X.rhsv[r], av);
                const unsigned long long k = key_min(ratio);
                if (k < lk) { lk = k; lr = r; }
            }
        }
    }
    double myfm = 0.0;
#pragma unroll
    for (int t = 0; t < Rt<RPL, CPW>::OPW; ++t)
        myfm = selp_f64(art_e ? R.arc[t] : R.rc[t], myfm, X.lane + 32 * t == ce);
    const double fm = __shfl_sync(kFull, myfm, ce & 31);
    int l = given_l;
    unsigned long long kmin = 0;
    if (given_l < 0) {
        kmin = warp_min_key(lk);
        l = warp_index_of(lk, kmin, lr);
    }
    if (X.lane == 0) {
        X.sh->e = e;
        X.sh->l = l;
        X.sh->kmin = kmin;
        X.sh->fm = fm;
        X.sh->oldvar = l != kNone ? X.basis[l] : -1;
    }
}

// pivot (tableau.py:218-244) on this warp's tile and transposed objective slots.
template <int RPL, int CPW, int KIND>
__device__ __forceinline__ void rt_update(const Rt<RPL, CPW> &X, RtRegs<RPL, CPW> &R, int e, int l, double pe,
                                          double fm, int oldvar) {
    const int lL = l & 31, lS = l >> 5;
    double *rb = X.rowbuf + X.warp * CPW;
    double *rv = X.rvec + X.warp * CPW;
    if (X.lane == lL) {
#pragma unroll
        for (int s = 0; s < RPL; ++s)
            if (s == lS) {
#pragma unroll
                for (int c = 0; c < CPW; c += 2) {
                    reinterpret_cast<double2 *>(rb)[c / 2] = make_double2(R.a[s][c], R.a[s][c + 1]);
                    R.a[s][c] = 0.0;
                    R.a[s][c + 1] = 0.0;
                }
            }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < Rt<RPL, CPW>::OPW; ++t) {
        const int q = X.lane + 32 * t;
        const int pos = X.warp * CPW + q;
        if (q < CPW && pos < X.ncols) {
            const double r = div_entry(rb[q], pe);
            rv[q] = r;
            if (pos == 0) {
                R.rc[t] = __dadd_rn(R.rc[t], __dmul_rn(fm, r));   // tableau.py:242
            } else {
                R.rc[t] = __dsub_rn(R.rc[t], __dmul_rn(fm, r));
                const int j = pos - 1;
                if (j == e) R.bas |= (1u << t);
                if (j == oldvar) R.bas &= ~(1u << t);
                if (KIND == kRtPhase1 && R.artk[t] >= 0) {
                    R.arc[t] = __dsub_rn(R.arc[t], __dmul_rn(fm, -r));
                    const int ja = X.nvc + R.artk[t];
                    if (ja == e) R.bas |= (0x10000u << t);
                    if (ja == oldvar) R.bas &= ~(0x10000u << t);
                }
            }
        }
    }
    if (KIND != kRtRestore) rt_candidates<RPL, CPW, KIND>(X, R);
    __syncwarp();
    double f[RPL];
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
        const int r = X.lane + 32 * s;
        f[s] = r == l ? -1.0 : (r < X.m ? X.fvec[r] : 0.0);
    }
#pragma unroll
    for (int c = 0; c < CPW; c += 2) {
        const double2 r2 = reinterpret_cast<const double2 *>(rv)[c / 2];
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
            R.a[s][c] = __dsub_rn(R.a[s][c], __dmul_rn(f[s], r2.x));
            R.a[s][c + 1] = __dsub_rn(R.a[s][c + 1], __dmul_rn(f[s], r2.y));
        }
    }
    if (X.warp == 0) {
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
            const int r = X.lane + 32 * s;
            if (r < X.m) X.rhsv[r] = R.a[s][0];
        }
    }
}

// Write the register tile into the stage (row-major, ld = ldg) for price-out.
template <int RPL, int CPW>
__device__ __forceinline__ void rt_tile_to_stage(const Rt<RPL, CPW> &X, const RtRegs<RPL, CPW> &R) {
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
        const int r = X.lane + 32 * s;
        if (r < X.m) {
#pragma unroll
            for (int c = 0; c < CPW; ++c) X.stage[(size_t)r * X.ldg + X.warp * CPW + c] = R.a[s][c];
        }
    }
}

// _price_out (simplex.py:133-143) in the transposed layout: lane q of warp w
// rebuilds the reduced cost of its position from the stage, rows in order.
template <int RPL, int CPW, int PHASE>
__device__ __forceinline__ void rt_price_out(const Rt<RPL, CPW> &X, RtRegs<RPL, CPW> &R, const double *cg) {
    for (int r = X.tid; r < X.m; r += X.nt) {
        const int bv = X.basis[r];
        X.cbv[r] = PHASE == 1 ? (bv >= X.nvc ? -1.0 : 0.0) : (bv < X.n ? cg[bv] : 0.0);
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < Rt<RPL, CPW>::OPW; ++t) {
        const int q = X.lane + 32 * t;
        const int pos = X.warp * CPW + q;
        if (q < CPW && pos < X.ncols) {
            const double *col = X.stage + pos;
            if (pos == 0) {
                double obj = 0.0;
                for (int r = 0; r < X.m; ++r) {
                    const double cb = X.cbv[r];
                    if (cb != 0.0) obj = __dadd_rn(obj, __dmul_rn(cb, col[(size_t)r * X.ldg]));
                }
                R.rc[t] = obj;
            } else {
                const int j = pos - 1;
                double rc = (PHASE == 2 && j < X.n) ? cg[j] : 0.0;
                double ac = -1.0;
                const bool art = PHASE == 1 && R.artk[t] >= 0;
                for (int r = 0; r < X.m; ++r) {
                    const double cb = X.cbv[r];
                    if (cb != 0.0) {
                        const double v = col[(size_t)r * X.ldg];
                        rc = __dsub_rn(rc, __dmul_rn(cb, v));
                        if (art) ac = __dsub_rn(ac, __dmul_rn(cb, -v));
                    }
                }
                R.rc[t] = rc;
                if (art) R.arc[t] = ac;
            }
        }
    }
    rt_candidates<RPL, CPW, PHASE == 1 ? kRtPhase1 : kRtPhase2>(X, R);
    __syncthreads();
}

struct RtPhase { int state, iters; };

// _run_phase (simplex.py:63-91).  Entry: candidates published + barrier.
template <int RPL, int CPW, int KIND>
__device__ RtPhase rt_run_phase(const Rt<RPL, CPW> &X, RtRegs<RPL, CPW> &R, const Limits &lim) {
    const int max_iter = lim.max_iterations > 0 ? lim.max_iterations : 50 * (X.m + X.n);
    const int trigger = lim.degenerate_limit >= 0 ? lim.degenerate_limit : (X.m > 1 ? X.m : 1);
    const unsigned long long kSent = key_max(kSentinel), kDeg = key_max(kDegenerateTol);
    int degenerate_run = 0;
    bool use_bland = false;
    for (int it = 0;; ++it) {
        if (it == max_iter) return {2, max_iter};
        const int e = rt_select_entering(X, use_bland);
        if (e < 0) return {0, it};
        const bool art_e = e >= X.nvc;
        const int epos = art_e ? 1 + X.n + X.art_row[e - X.nvc] : e + 1;
        if (X.warp == epos / CPW) rt_owner_column(X, R, e, epos, art_e, -1);
        rt_barrier(X.nw);  // B2
        const int l = X.sh->l;
        const unsigned long long kmin = X.sh->kmin;
        if (l == kNone || kmin >= kSent) return {1, it};   // unbounded (a NaN ratio keys to 0)
        const double pe = X.fvec[l];
        const double fm = X.sh->fm;
        const int oldvar = X.sh->oldvar;
        if (kmin != 0ull && kmin <= kDeg) {                // simplex.py:84-90
            ++degenerate_run;
            if (lim.anti_cycling && degenerate_run >= trigger) use_bland = true;
        } else {
            degenerate_run = 0;
            use_bland = false;
        }
        if (X.tid == 0) X.basis[l] = e;
        rt_update<RPL, CPW, KIND>(X, R, e, l, pe, fm, oldvar);
        rt_barrier(X.nw);  // B4
    }
}

// restore_objective pivot-outs (simplex.py:109-126), uncounted.
template <int RPL, int CPW>
__device__ void rt_restore(const Rt<RPL, CPW> &X, RtRegs<RPL, CPW> &R) {
    const unsigned long long kRed = key_max(kRedundantTol);
    for (int row = 0; row < X.m; ++row) {
        if (X.basis[row] < X.nvc) continue;   // uniform; basis is stable between barriers
        const int rL = row & 31, rS = row >> 5;
        unsigned long long bk = kKeyEmptyMax;
        int bj = kNone;
        if (X.lane == rL) {
#pragma unroll
            for (int s = 0; s < RPL; ++s)
                if (s == rS) {
#pragma unroll
                    for (int c = 0; c < CPW; ++c) {
                        const int pos = X.warp * CPW + c;
                        if (pos >= 1 && pos < X.ncols) {
                            const unsigned long long k = key_max(fabs(R.a[s][c]));
                            if (k > bk) { bk = k; bj = pos - 1; }
                        }
                    }
                }
        }
        const unsigned long long kw = warp_max_key(bk);
        const int jw = warp_index_of(bk, kw, bj);
        if (X.lane == 0) { X.ckey[X.warp] = kw; X.cidx[X.warp] = jw; }
        __syncthreads();
        unsigned long long k = kKeyEmptyMax;
        int i = kNone;
        if (X.lane < X.nw) { k = X.ckey[X.lane]; i = X.cidx[X.lane]; }
        const unsigned long long kbest = warp_max_key(k);
        const int j = warp_index_of(k, kbest, i);
        // entries[j] > REDUNDANT_ROW_TOL; a NaN entry compares False in numpy
        if (j != kNone && kbest > kRed && kbest != ~0ull) {
            const int epos = j + 1;
            if (X.warp == epos / CPW) rt_owner_column(X, R, j, epos, false, row);
            __syncthreads();
            const double pe = X.fvec[row];
            const int oldvar = X.sh->oldvar;
            __syncthreads();
            if (X.tid == 0) X.basis[row] = j;
            rt_update<RPL, CPW, kRtRestore>(X, R, j, row, pe, 0.0, oldvar);
        }
        __syncthreads();
    }
}

template <int RPL, int CPW, int kMaxThreads, int kMinBlocks>
__global__ void __launch_bounds__(kMaxThreads, kMinBlocks)
regtile_kernel(Batch B) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int nw = blockDim.x >> 5;
    const RtLayout L = make_rt_layout(RPL, CPW, nw);
    Rt<RPL, CPW> X;
    X.m = B.m; X.n = B.n; X.nvc = B.n + B.m; X.ncols = B.n + B.m + 1;
    X.nw = nw; X.lane = threadIdx.x & 31; X.warp = threadIdx.x >> 5; X.tid = threadIdx.x; X.nt = blockDim.x;
    X.fvec = reinterpret_cast<double *>(smem + L.off_fvec);
    X.rhsv = reinterpret_cast<double *>(smem + L.off_rhs);
    X.cbv = reinterpret_cast<double *>(smem + L.off_cbv);
    X.rowbuf = reinterpret_cast<double *>(smem + L.off_rowbuf);
    X.rvec = reinterpret_cast<double *>(smem + L.off_rvec);
    X.stage = reinterpret_cast<double *>(smem + L.off_stage);
    X.ckey = reinterpret_cast<unsigned long long *>(smem + L.off_ckey);
    X.cidx = reinterpret_cast<int *>(smem + L.off_cidx);
    X.cbl = reinterpret_cast<int *>(smem + L.off_cbl);
    X.basis = reinterpret_cast<int *>(smem + L.off_basis);
    X.art_row = reinterpret_cast<int *>(smem + L.off_artrow);
    X.art_of = reinterpret_cast<int *>(smem + L.off_artof);
    X.wcnt = reinterpret_cast<int *>(smem + L.off_wcnt);
    X.sh = reinterpret_cast<RtShared *>(smem + L.off_sh);
    X.ldg = L.ldg;
    const int m = X.m, n = X.n, nvc = X.nvc;

    // padding positions of the pivot-row buffer stay zero forever
    for (int q = X.tid; q < nw * CPW; q += X.nt) { X.rvec[q] = 0.0; X.rowbuf[q] = 0.0; }

    RtRegs<RPL, CPW> R;
    for (;;) {
        if (X.tid == 0) { X.sh->lp = atomicAdd(B.next_lp, 1); X.sh->n_art = 0; }
        __syncthreads();
        const long long lp = X.sh->lp;
        if (lp >= B.count) break;
        const double *Ag = B.shared_Ab ? B.A : B.A + (size_t)lp * m * n;
        const double *bg = B.shared_Ab ? B.b : B.b + (size_t)lp * m;
        const double *cg = B.c + (size_t)lp * n;

        // ---- build_tableau (tableau.py:139-172) into the stage; validate on the fly ----
        bool nonfinite = false;
        for (int base = 0; base < m; base += X.nt) {
            const int i = base + X.tid;
            const double bi = i < m ? bg[i] : 0.0;
            nonfinite |= !isfinite(bi);
            const bool neg = i < m && bi < 0.0;
            const unsigned bal = __ballot_sync(kFull, neg);
            if (X.lane == 0) X.wcnt[X.warp] = __popc(bal);
            __syncthreads();
            int pre = X.sh->n_art + __popc(bal & ((1u << X.lane) - 1u));
            for (int w = 0; w < X.warp; ++w) pre += X.wcnt[w];
            if (i < m) {
                const double s = neg ? -1.0 : 1.0;
                X.cbv[i] = s;
                X.stage[(size_t)i * X.ldg] = __dmul_rn(bi, s);
                if (neg) { X.basis[i] = nvc + pre; X.art_row[pre] = i; X.art_of[i] = pre; }
                else { X.basis[i] = n + i; X.art_of[i] = -1; }
            }
            __syncthreads();
            if (X.tid == 0) { int t = 0; for (int w = 0; w < nw; ++w) t += X.wcnt[w]; X.sh->n_art += t; }
            __syncthreads();
        }
        const int n_art = X.sh->n_art;
        for (int k = X.tid; k < m * n; k += X.nt) {
            const int i = k / n, j = k - i * n;
            const double a = Ag[k];
            nonfinite |= !isfinite(a);
            X.stage[(size_t)i * X.ldg + 1 + j] = __dmul_rn(a, X.cbv[i]);
        }
        for (int k = X.tid; k < m * m; k += X.nt) {
            const int i = k / m, q = k - i * m;
            X.stage[(size_t)i * X.ldg + 1 + n + q] = i == q ? X.cbv[i] : 0.0;
        }
        for (int j = X.tid; j < n; j += X.nt) nonfinite |= !isfinite(cg[j]);
        const bool invalid = __syncthreads_or(nonfinite);

        // stage -> registers; objective row transposed
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
            const int r = X.lane + 32 * s;
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                const int pos = X.warp * CPW + c;
                R.a[s][c] = (r < m && pos < X.ncols) ? X.stage[(size_t)r * X.ldg + pos] : 0.0;
            }
            if (X.warp == 0 && r < m) X.rhsv[r] = R.a[s][0];
        }
        R.bas = 0;
#pragma unroll
        for (int t = 0; t < Rt<RPL, CPW>::OPW; ++t) {
            const int q = X.lane + 32 * t;
            const int pos = X.warp * CPW + q;
            const int j = pos - 1;
            R.rc[t] = (q < CPW && pos >= 1 && j < n) ? cg[j] : 0.0;
            R.arc[t] = 0.0;
            R.artk[t] = -1;
            if (q < CPW && j >= n && j < nvc) {
                R.artk[t] = X.art_of[j - n];
                if (R.artk[t] < 0) R.bas |= 1u << t;          // slack of a non-negated row is basic
                else R.bas |= 0x10000u << t;                  // else its row's artificial is
            }
        }

        int8_t status = kOptimal;
        int it1 = 0, it2 = 0;
        bool done = false;
        if (invalid) {
            status = kInvalid;
            done = true;
        } else if (n_art > 0) {
            rt_price_out<RPL, CPW, 1>(X, R, cg);                  // build_auxiliary
            const RtPhase p1 = rt_run_phase<RPL, CPW, kRtPhase1>(X, R, B.lim);
            __syncthreads();
            it1 = p1.iters;
            const double obj = __shfl_sync(kFull, R.rc[0], 0);     // objective value: warp 0, lane 0
            if (X.tid == 0) X.sh->fm = obj;
            __syncthreads();
            if (p1.state == 2) { status = kIterationLimit; done = true; }
            else if (p1.state == 1) { status = kErrPhase1Unbounded; done = true; }
            else if (fabs(X.sh->fm) > kPhase1ZeroTol) { status = kInfeasible; done = true; }
            else {
                rt_restore(X, R);
                rt_tile_to_stage(X, R);
                __syncthreads();
                rt_price_out<RPL, CPW, 2>(X, R, cg);
            }
            __syncthreads();
        } else {
            rt_candidates<RPL, CPW, kRtPhase2>(X, R);
            __syncthreads();
        }
        if (!done) {
            const RtPhase p2 = rt_run_phase<RPL, CPW, kRtPhase2>(X, R, B.lim);
            __syncthreads();
            it2 = p2.iters;
            if (p2.state == 2) status = kIterationLimit;
            else if (p2.state == 1) status = kUnbounded;
        }

        // ---- _extract_point (simplex.py:146-151) and c @ x ----
        double *xs = X.stage;
        for (int j = X.tid; j < n; j += X.nt) xs[j] = 0.0;
        __syncthreads();
        if (status == kOptimal && X.warp == 0) {
#pragma unroll
            for (int s = 0; s < RPL; ++s) {
                const int r = X.lane + 32 * s;
                if (r < m && X.basis[r] < n) xs[X.basis[r]] = R.a[s][0];
            }
        }
        __syncthreads();
        double *xg = B.x + (size_t)lp * n;
        for (int j = X.tid; j < n; j += X.nt) xg[j] = xs[j];
        if (X.tid == 0) {
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
    }
}

}  // namespace blp
