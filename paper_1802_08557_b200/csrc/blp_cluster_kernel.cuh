// blp_cluster_kernel.cuh -- one thread-block CLUSTER per LP, for tableaux too
// large for one SM (C5, 500 x 500: 501 x 1001 fp64 = 4 MB).
//
// The HBM-streamed variant (blp_tableau_kernel.cuh, hbm_rpl*) reads and
// writes the whole tableau from HBM on every pivot.  Here the tableau is
// split by COLUMNS over the K CTAs of a cluster (K <= 16, one CTA per SM) and
// stays on chip for the LP's whole solve.  CTA k owns sn = ceil(n/K)
// structural columns [k sn, (k+1) sn) and sm = ceil(m/K) slack columns
// n + [k sm, (k+1) sm) -- every CTA loads the same share of A -- as local
// columns 0..cpc-1 (structural first).  Thread i holds row i: local columns
// [0, RC) in registers, [RC, cpc) in a column-major shared tile tile[c][i]
// (odd row stride ld >= m).  The rhs column, the basis, the objective cell
// and the LP bookkeeping are replicated in every CTA and updated identically.
//
// Per pivot (tableau.py:175-244 on K CTAs) there is ONE cluster barrier:
//   1. every CTA publishes its local entering candidate (choose_entering over
//      its own reduced costs): the header (key, index, Bland index, rc_e) in
//      its shared memory, the candidate's column in a per-CTA global slot
//      (L2-resident; K readers of one smem port would serialise on DSMEM);
//   2. barrier.cluster arrive (release) ... wait (acquire); the candidate is
//      published right after the previous pivot's selection, before the tile
//      half of that pivot's update, so the barrier and the CTAs' skew hide
//      behind it;
//   3. warp 0 reads the K headers through DSMEM and reduces them in numpy
//      order; every row thread reads its entry f_i of the winning column;
//   4. the ratio test (choose_leaving) runs redundantly in every CTA on its
//      replicated rhs column -- identical inputs, identical l;
//   5. each CTA divides its own part of row l by pe and applies the rank-1
//      update to its own columns (registers: DMUL + DSUB; tile: LDS, DMUL,
//      DSUB, STS -- 4-column batches whose pivot-row entries are all zero are
//      skipped: a - f*0 == a, and slack columns stay sparse for many pivots).
// The slot a CTA writes at pivot k+1 was last read at pivot k-1; the barrier
// of pivot k separates them, so no second barrier is needed.
//
// Artificial columns are elided as in every other variant (art_rc per owned
// slack column); price-out (simplex.py:133-143) streams the rows in order
// through a small staging buffer so the per-column sums keep the reference's
// sequential order; restore_objective (simplex.py:109-130) reduces each
// artificial row's |entry| argmax over the cluster like an entering choice.
// The arithmetic is the other variants' (separately rounded products and
// differences, IEEE divisions), so results equal theirs and the reference's.
//
// The objective value c @ x (simplex.py:190, BLAS ddot in the reference,
// summation order unpinned) is summed left to right here, as in every kernel and the
// oracle (a near-zero optimum is ill-conditioned: any other order can miss 1e-9 relative).
#pragma once

#include "blp_common.cuh"
#include "blp_keys.cuh"

namespace blp {

constexpr int kClRB = 8;        // rows per price-out staging batch
constexpr int kClMaxK = 16;     // largest (non-portable) cluster
constexpr int kClSG = 16;       // register-half columns staged per build pass
constexpr int kClMaxCols = 256; // owned columns per CTA (register + tile)
constexpr int kClMaxRows = 512;

enum ClKind { kClRestore = 0, kClPhase1 = 1, kClPhase2 = 2 };

// ---------------------------------------------------------------------------
// Cluster / DSMEM / async-copy primitives (PTX ISA).
__device__ __forceinline__ unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cl_size() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cl_id() {
    unsigned r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_sync() { cl_arrive(); cl_wait(); }
__device__ __forceinline__ unsigned cl_map(unsigned saddr, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ double cl_ld_f64(unsigned a) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ int cl_ld_s32(unsigned a) {
    int v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ long long cl_ld_s64(unsigned a) {
    long long v;
    asm volatile("ld.shared::cluster.s64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned smem_addr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async8(unsigned saddr, const void *g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2(const void *g) { asm volatile("prefetch.global.L2 [%0];" ::"l"(g)); }
__device__ __forceinline__ void cl_st_v2_if(bool p, unsigned addr, double x, double y) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.shared.v2.f64 [%1], {%2, %3}; }"
                 ::"r"((unsigned)p), "r"(addr), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void cl_ld_v2_if(bool p, unsigned addr, double &x, double &y) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q ld.volatile.shared.v2.f64 {%0, %1}, [%3]; }"
                 : "+d"(x), "+d"(y) : "r"((unsigned)p), "r"(addr) : "memory");
}

// ---------------------------------------------------------------------------
struct ClPubHdr {                 // one CTA's entering candidate (16-byte aligned: two loads)
    unsigned long long key;       // Dantzig: numpy max-order key of its reduced cost
    int idx;                      // Dantzig: lowest index with that key
    int bl;                       // Bland: lowest index with rc > tol
    double rce;                   // reduced cost of the published column
    double pad;
};

struct ClPart {                   // per-warp partials inside one CTA
    unsigned long long ckey[32];
    int cidx[32], cbl[32];
    unsigned long long lkey[32];
    int lrow[32];
    int wneg[32];
};

// Fixed-size state in static shared memory (compile-time addresses: no
// registers spent on pointers); the tile and the staging buffer, sized by m,
// are dynamic.
template <int RC>
struct ClStatic {
    double rowbuf[RC];                 // register half of the pivot row
    double rvec[kClMaxCols];           // pivot row / pe, owned columns (zero past cpc)
    double rcv[kClMaxCols];            // objective row, owned columns
    double arc[kClMaxCols];            // phase-1 reduced cost of the artificial paired with an owned slack
    double cbv[kClMaxRows];            // basic costs during price-out; row signs during the build
    double bpre[kClMaxRows];           // b of the LP being built (copied in asynchronously)
    double stg[kClRB * RC];            // price-out staging: register halves of kClRB rows
    double stgr[kClRB];
    int artk[kClMaxCols];              // artificial index of an owned slack column, or -1
    int basis[kClMaxRows];             // replicated basis
    int art_row[kClMaxRows];           // row of artificial k
    ClPart P;
    ClPubHdr hdr[2];                   // this CTA's published candidate, by parity (read via DSMEM)
    long long nxt[2];                  // rank 0: the LP after the current one, by LP parity (read via DSMEM)
    double pe, rrhs, obj;
    int inv[2];                        // this CTA's validation flag, by LP parity (read via DSMEM)
    int sel_e, sel_owner;              // the cluster-wide entering column, as reduced by warp 0
    double sel_rce;
#ifdef BLP_CL_PROF
    unsigned long long prof[16];
    long long prof_t;
#endif
    unsigned char isb[kClMaxCols * kClMaxK + kClMaxRows];   // replicated "is basic" flags
};

template <int RC>
__device__ __forceinline__ ClStatic<RC> &cl_static() {
    __shared__ __align__(16) ClStatic<RC> s;
    return s;
}

// Optional segment timers (-DBLP_CL_PROF builds only; the product build has none):
// thread 0 of every CTA accumulates clock64 deltas per segment.
#ifdef BLP_CL_PROF
__device__ unsigned long long g_cl_prof[16];
#define CL_PROF_MARK(k)                                                                    \
    do {                                                                                   \
        if (threadIdx.x == 0) {                                                            \
            const long long _t = clock64();                                                \
            cl_static<RC>().prof[k] += (unsigned long long)(_t - cl_static<RC>().prof_t); \
            cl_static<RC>().prof_t = _t;                                                   \
        }                                                                                  \
    } while (0)
#else
#define CL_PROF_MARK(k) do { } while (0)
#endif

struct ClLayout {
    int ld, sn, sm, cpc, sc4;     // row stride, structural / slack / all columns per CTA, tile columns
    size_t off_stage;             // kClSG staging columns after the tile
    size_t bytes;                 // dynamic shared memory
};

__host__ __device__ inline size_t cl_align(size_t x) { return (x + 15) / 16 * 16; }

__host__ __device__ inline ClLayout make_cl_layout(int m, int n, int K, int RC) {
    ClLayout L;
    L.ld = m | 1;                                         // odd: staging writes conflict-free
    L.sn = (n + K - 1) / K;
    L.sm = (m + K - 1) / K;
    L.cpc = L.sn + L.sm;
    const int sc = L.cpc > RC ? L.cpc - RC : 0;
    L.sc4 = (sc + 3) & ~3;
    L.off_stage = (size_t)L.sc4 * L.ld * 8;
    L.bytes = cl_align(L.off_stage + (size_t)kClSG * L.ld * 8);
    return L;
}

// ---------------------------------------------------------------------------
struct ClCtx {
    int m, n, nv, ld, sn, sm, cpc, sc4, s0, q0, ns, K, rank;
    int tid, lane, warp, nw, nwc;  // nwc: warps holding the column threads t < cpc
    bool live;                     // tid < m: this thread holds a constraint row
    double *tile;                  // [sc4][ld] then [kClSG][ld] staging, dynamic shared memory
    double *gcol;                  // this cluster's published columns in global memory: [2][K][ld]
    int par;                       // parity of the next publication slot
};

// Global column of local column c (structural first), or -1 if not owned.
__device__ __forceinline__ int cl_gcol(const ClCtx &X, int c) {
    if (c < X.sn) return c < X.ns ? X.s0 + c : -1;
    const int q = X.q0 + c - X.sn;
    return (c < X.cpc && q < X.m) ? X.n + q : -1;
}
// Local column of an owned global column j < nv.
__device__ __forceinline__ int cl_lcol(const ClCtx &X, int j) {
    return j < X.n ? j - X.s0 : X.sn + (j - X.n - X.q0);
}

__device__ __forceinline__ double *cl_gslot(const ClCtx &X, int par, int rank) {
    return X.gcol + (size_t)(par * X.K + rank) * X.ld;
}

struct ClBest {
    unsigned long long k = kKeyEmptyMax;
    int i = kNone, bl = kNone;
    __device__ __forceinline__ void add(double v, int j) {
        const unsigned long long kv = key_max(v);
        if (kv > k || (kv == k && j < i)) { k = kv; i = j; }
        if (v > kTol && j < bl) bl = j;
    }
};

// Entering candidates of this CTA's columns (choose_entering / _bland,
// tableau.py:175-197), reduced per warp into P.  Called by warps < nwc only.
// Basic test as of the pivot being applied: (j == e) || (j != oldvar && isb[j]).
template <int RC, int KIND>
__device__ __forceinline__ void cl_candidates(const ClCtx &X, int e, int oldvar) {
    ClStatic<RC> &S = cl_static<RC>();
    ClBest b;
    const int t = X.tid, j = cl_gcol(X, t);
    if (j >= 0) {
        if (!((j == e) || (j != oldvar && S.isb[j]))) b.add(S.rcv[t], j);
        if (KIND == kClPhase1 && S.artk[t] >= 0) {       // phase 1: the paired artificial column
            const int ja = X.nv + S.artk[t];
            if (!((ja == e) || (ja != oldvar && S.isb[ja]))) b.add(S.arc[t], ja);
        }
    }
    const unsigned long long kw = warp_max_key(b.k);
    const int iw = warp_index_of(b.k, kw, b.i);
    const int bw = warp_min_int(b.bl);
    if (X.lane == 0) { S.P.ckey[X.warp] = kw; S.P.cidx[X.warp] = iw; S.P.cbl[X.warp] = bw; }
}

template <int RC>
__device__ __forceinline__ void cl_local_best(const ClCtx &X, unsigned long long &k, int &i, int &bl) {
    ClStatic<RC> &S = cl_static<RC>();
    k = kKeyEmptyMax; i = kNone; bl = kNone;
    for (int w = 0; w < X.nwc; ++w) {
        const unsigned long long kw = S.P.ckey[w];
        const int iw = S.P.cidx[w];
        if (kw > k || (kw == k && iw < i)) { k = kw; i = iw; }
        bl = min(bl, S.P.cbl[w]);
    }
}

// Publish this CTA's candidate `cand` (global column, nv + k for an
// artificial): its column into the global slot (row i by thread i), the
// header into shared memory.  With l >= 0 the column is published as it will
// be after the pivot at row l (this row's entry f, pivot row in rvec): the
// same two roundings the bulk update performs, so the value is the final one.
template <int RC>
__device__ __forceinline__ void cl_publish(const ClCtx &X, const double (&a)[RC], int cand,
                                           unsigned long long key, int idx, int bl, int l = -1, double f = 0.0) {
    ClStatic<RC> &S = cl_static<RC>();
    double rce = 0.0;
    if (cand != kNone) {                                   // CTA-uniform
        const bool art = cand >= X.nv;
        const int c = cl_lcol(X, art ? X.n + S.art_row[cand - X.nv] : cand);
        if (X.live) {
            double v = c < RC ? reg_pick<RC>(a, c) : X.tile[(size_t)(c - RC) * X.ld + X.tid];
            if (l >= 0) {
                const double r = S.rvec[c];
                v = X.tid == l ? r : __dsub_rn(v, __dmul_rn(f, r));
            }
            __stcg(cl_gslot(X, X.par, X.rank) + X.tid, art ? -v : v);
        }
        rce = art ? S.arc[c] : S.rcv[c];
    }
    if (X.tid == 0) {
        ClPubHdr &h = S.hdr[X.par];
        h.key = key;
        h.idx = idx;
        h.bl = bl;
        h.rce = rce;
    }
}

// After the cluster barrier: warp 0 reads the K headers through DSMEM (two
// loads per CTA) and reduces them in numpy order -- MODE 0 Dantzig: largest
// key, then lowest index, nothing above tol = optimal (choose_entering);
// MODE 1 Bland: lowest index; MODE 2 restore: largest |entry| key, lowest
// index, only above REDUNDANT_ROW_TOL (NaN compares False).  Result in S.sel_*.
template <int RC, int MODE>
__device__ __forceinline__ void cl_reduce_headers(const ClCtx &X) {
    ClStatic<RC> &S = cl_static<RC>();
    if (X.warp != 0) return;
    unsigned long long k = kKeyEmptyMax, ib = ((unsigned long long)(unsigned)kNone << 32) | (unsigned)kNone;
    double rc = 0.0;
    if (X.lane < X.K) {
        const unsigned h = cl_map(smem_addr(&S.hdr[X.par]), (unsigned)X.lane);
        asm volatile("ld.shared::cluster.v2.u64 {%0, %1}, [%2];" : "=l"(k), "=l"(ib) : "r"(h) : "memory");
        rc = cl_ld_f64(h + 16);
    }
    const int i = (int)(unsigned)ib, b = (int)(unsigned)(ib >> 32);
    int e;
    if (MODE == 1) {
        e = warp_min_int(b);
    } else {
        const unsigned long long kw = warp_max_key(k);
        e = warp_index_of(k, kw, i);
        if (MODE == 0 && e != kNone && kw <= key_max(kTol)) e = kNone;   // NaN keys sort above tol, as numpy
        if (MODE == 2 && !(e != kNone && kw > key_max(kRedundantTol) && kw != ~0ull)) e = kNone;
    }
    int owner = 0;
    if (e != kNone) owner = __ffs(__ballot_sync(kFull, X.lane < X.K && (MODE == 1 ? b : i) == e)) - 1;
    const double r = __shfl_sync(kFull, rc, owner);
    if (X.lane == 0) { S.sel_e = e == kNone ? -1 : e; S.sel_owner = owner; S.sel_rce = r; }
}

// This thread's entry of the column CTA `owner` published (slot par), from L2.
__device__ __forceinline__ double cl_fetch_col(const ClCtx &X, int owner) {
    if (!X.live) return 0.0;
    return __ldcg(cl_gslot(X, X.par, owner) + X.tid);
}

// Rank-1 update of this row's tile columns in batches of 4: two 16-byte
// loads of r (the same for every lane), then -- unless all four are zero,
// where a - f*0 == a -- four column loads and four stores (volatile: program
// order; the tile and rvec are both shared memory, nothing could be hoisted).
__device__ __forceinline__ void cl_update_tile(unsigned col, unsigned rv, int sc4, int ld, double fs) {
    const unsigned cs = 8u * ld;
    for (int b = 0; b < sc4; b += 4, col += 4u * cs, rv += 32u) {
        double t[4], r[4];
        lds_v2_f64(rv, r[0], r[1]);
        lds_v2_f64(rv + 16u, r[2], r[3]);
        if (r[0] == 0.0 && r[1] == 0.0 && r[2] == 0.0 && r[3] == 0.0) continue;   // CTA-uniform
#pragma unroll
        for (int k = 0; k < 4; ++k) t[k] = lds_f64(col + cs * k);
#pragma unroll
        for (int k = 0; k < 4; ++k) sts_f64(col + cs * k, __dsub_rn(t[k], __dmul_rn(fs, r[k])));
    }
}

// pivot (tableau.py:218-244) at (l, e) on this CTA's columns.  f = this row's
// entry of column e (row l: pe), rce = the entering reduced cost.
//
// publish_next: the next pivot's candidate (mode next_bland) is published
// right after S3 and the cluster barrier arrived on after the register half
// of the update (by then the global stores are performed, so the release is
// cheap); the tile half then overlaps the barrier.
template <int RC, int KIND>
__device__ __forceinline__ void cl_pivot(ClCtx &X, double (&a)[RC], double &rhs, double &obj,
                                         int e, int l, double f, double rce,
                                         bool publish_next = false, bool next_bland = false) {
    ClStatic<RC> &S = cl_static<RC>();
    const bool mine = X.tid == l;
    if ((l >> 5) == X.warp) {                   // warp-uniform: the row's warp stores its register half
        const unsigned rb = smem_addr(S.rowbuf);
#pragma unroll
        for (int c = 0; c < RC; c += 2) cl_st_v2_if(mine, rb + 8u * c, a[c], a[c + 1]);
    }
    if (mine) { S.pe = f; S.rrhs = div_entry(rhs, f); }
    __syncthreads();  // S2
    const double pe = S.pe, rrhs = S.rrhs;
    const int oldvar = S.basis[l];
    if (X.warp < X.nwc) {
        const int t = X.tid;
        if (t < X.cpc) {
            double *src = t < RC ? S.rowbuf + t : X.tile + (size_t)(t - RC) * X.ld + l;
            const double r = div_entry(*src, pe);
            S.rvec[t] = r;
            if (t >= RC) *src = r;              // row l of a tile column is final (numpy: r - 0*r)
            if (KIND != kClRestore) {
                S.rcv[t] = __dsub_rn(S.rcv[t], __dmul_rn(rce, r));
                // artificial = -(its row's slack column): pivot-row entry -r exactly
                if (KIND == kClPhase1 && S.artk[t] >= 0) S.arc[t] = __dsub_rn(S.arc[t], __dmul_rn(rce, -r));
            }
        }
        if (KIND != kClRestore) cl_candidates<RC, KIND>(X, e, oldvar);
    }
    __syncthreads();  // S3
    CL_PROF_MARK(5);
    const bool pub = KIND != kClRestore && publish_next;
    if (pub) {
        unsigned long long kD;
        int iD, bl;
        cl_local_best<RC>(X, kD, iD, bl);
        cl_publish<RC>(X, a, next_bland ? bl : iD, kD, iD, bl, l, f);
    }
    if (X.live) {
        const double2 *r2 = reinterpret_cast<const double2 *>(S.rvec);
#pragma unroll
        for (int c = 0; c < RC; c += 2) {
            const double2 r = r2[c / 2];
            a[c] = __dsub_rn(a[c], __dmul_rn(f, r.x));
            a[c + 1] = __dsub_rn(a[c + 1], __dmul_rn(f, r.y));
        }
        rhs = mine ? rrhs : __dsub_rn(rhs, __dmul_rn(f, rrhs));
    }
    if ((l >> 5) == X.warp) {                   // row l <- r (register half)
        const unsigned rv = smem_addr(S.rvec);
#pragma unroll
        for (int c = 0; c < RC; c += 2) cl_ld_v2_if(mine, rv + 8u * c, a[c], a[c + 1]);
    }
#ifndef CL_ARRIVE_LATE
    if (pub) cl_arrive();
#endif
    CL_PROF_MARK(6);
    if (X.live) cl_update_tile(smem_addr(X.tile + X.tid), smem_addr(S.rvec + RC), X.sc4, X.ld, mine ? 0.0 : f);
#ifdef CL_ARRIVE_LATE
    if (pub) cl_arrive();
#endif
    if (KIND != kClRestore) obj = __dadd_rn(obj, __dmul_rn(rce, rrhs));   // tableau.py:242
    if (X.tid == 0) { S.basis[l] = e; S.isb[oldvar] = 0; S.isb[e] = 1; }
}

struct ClPhase { int state, iters; };  // 0 optimal, 1 unbounded, 2 iteration limit

// _run_phase (simplex.py:63-91).  Entry: candidates in P + a CTA barrier.
template <int RC, int KIND>
__device__ ClPhase cl_run_phase(ClCtx &X, double (&a)[RC], double &rhs, double &obj, const Limits &lim) {
    ClStatic<RC> &S = cl_static<RC>();
    const int max_iter = lim.max_iterations > 0 ? lim.max_iterations : 50 * (X.m + X.n);
    const int trigger = lim.degenerate_limit >= 0 ? lim.degenerate_limit : (X.m > 1 ? X.m : 1);
    const unsigned long long kSent = key_max(kSentinel), kDeg = key_max(kDegenerateTol);
    int degenerate_run = 0;
    bool use_bland = false;
    {
        unsigned long long kD;
        int iD, bl;
        cl_local_best<RC>(X, kD, iD, bl);
        cl_publish<RC>(X, a, iD, kD, iD, bl);
        cl_arrive();
    }
    // loop invariant: this pivot's candidates are published and the barrier arrived on
    for (int it = 0;; ++it) {
        CL_PROF_MARK(8);
        cl_wait();
        CL_PROF_MARK(3);
        if (use_bland) cl_reduce_headers<RC, 1>(X);
        else cl_reduce_headers<RC, 0>(X);
        __syncthreads();  // S0
        const int e = S.sel_e;
        const double rce = S.sel_rce;
        if (e < 0) { X.par ^= 1; return {0, it}; }
        const double f = cl_fetch_col(X, S.sel_owner);
        X.par ^= 1;
        // choose_leaving (tableau.py:200-215), redundantly in every CTA
        unsigned long long lk = kKeyEmptyMin;
        if (X.live) lk = key_min(ratio_entry(rhs, f));
        {
            const unsigned long long kw = warp_min_key(lk);
            const int lw = warp_index_of(lk, kw, X.tid);
            if (X.lane == 0) { S.P.lkey[X.warp] = kw; S.P.lrow[X.warp] = lw; }
        }
        __syncthreads();  // S1
        unsigned long long kmin;
        int l;
        {                                      // rows ascend with the warp: lowest row among the minima
            const unsigned long long k = X.lane < X.nw ? S.P.lkey[X.lane] : kKeyEmptyMin;
            const int r = X.lane < X.nw ? S.P.lrow[X.lane] : kNone;
            kmin = warp_min_key(k);
            l = warp_index_of(k, kmin, r);
        }
        if (l == kNone || kmin >= kSent) return {1, it};   // unbounded (a NaN ratio keys to 0)
        if (kmin != 0ull && kmin <= kDeg) {                 // simplex.py:84-90
            ++degenerate_run;
            if (lim.anti_cycling && degenerate_run >= trigger) use_bland = true;
        } else {
            degenerate_run = 0;
            use_bland = false;
        }
        const bool more = it + 1 < max_iter;
        CL_PROF_MARK(4);
        cl_pivot<RC, KIND>(X, a, rhs, obj, e, l, f, rce, more, use_bland);
        if (!more) return {2, max_iter};
    }
}

// _price_out (simplex.py:133-143): rows streamed in order through the
// staging buffer, one thread per owned column (plus thread cpc for the
// objective cell).  PHASE 1: c_aux = -1 on artificials; PHASE 2: original c.
template <int RC, int PHASE>
__device__ void cl_price_out(ClCtx &X, const double (&a)[RC], double rhs, double &obj, const double *cg) {
    ClStatic<RC> &S = cl_static<RC>();
    if (X.live) {
        const int bv = S.basis[X.tid];
        S.cbv[X.tid] = PHASE == 1 ? (bv >= X.nv ? -1.0 : 0.0) : (bv < X.n ? cg[bv] : 0.0);
    }
    const int t = X.tid, j = X.tid < X.cpc ? cl_gcol(X, t) : -1;
    const bool col = j >= 0;
    const bool art = PHASE == 1 && col && S.artk[t] >= 0;
    double rc = (PHASE == 2 && col && j < X.n) ? cg[j] : 0.0, ac = -1.0, ob = 0.0;
    __syncthreads();
    for (int rb = 0; rb < X.m; rb += kClRB) {
        if (X.live && X.tid >= rb && X.tid < rb + kClRB) {
            const unsigned s = smem_addr(S.stg + (X.tid - rb) * RC);
#pragma unroll
            for (int c = 0; c < RC; c += 2) cl_st_v2_if(true, s + 8u * c, a[c], a[c + 1]);
            S.stgr[X.tid - rb] = rhs;
        }
        __syncthreads();
        if (col || t == X.cpc) {
            const int qe = min(kClRB, X.m - rb);
            for (int q = 0; q < qe; ++q) {
                const int r = rb + q;
                const double cb = S.cbv[r];
                if (cb == 0.0) continue;
                if (!col) { ob = __dadd_rn(ob, __dmul_rn(cb, S.stgr[q])); continue; }
                const double v = t < RC ? S.stg[q * RC + t] : X.tile[(size_t)(t - RC) * X.ld + r];
                rc = __dsub_rn(rc, __dmul_rn(cb, v));
                if (art) ac = __dsub_rn(ac, __dmul_rn(cb, -v));
            }
        }
        __syncthreads();
    }
    if (col) {
        S.rcv[t] = rc;
        if (PHASE == 1) S.arc[t] = art ? ac : 0.0;
    }
    if (t == X.cpc) S.obj = ob;
    __syncthreads();
    obj = S.obj;
    if (X.warp < X.nwc) cl_candidates<RC, PHASE == 1 ? kClPhase1 : kClPhase2>(X, -1, -1);
    __syncthreads();
}

// restore_objective pivot-outs (simplex.py:109-126): for each row whose basic
// variable is artificial, the first max |entry| over the structural + slack
// columns of the whole cluster; pivot there if > REDUNDANT_ROW_TOL.  Uncounted.
template <int RC>
__device__ void cl_restore(ClCtx &X, double (&a)[RC], double &rhs, double &obj) {
    ClStatic<RC> &S = cl_static<RC>();
    __syncthreads();
    for (int row = 0; row < X.m; ++row) {
        if (S.basis[row] < X.nv) continue;     // CTA- and cluster-uniform
        const bool mine = X.tid == row;
        if ((row >> 5) == X.warp) {
            const unsigned rb = smem_addr(S.rowbuf);
#pragma unroll
            for (int c = 0; c < RC; c += 2) cl_st_v2_if(mine, rb + 8u * c, a[c], a[c + 1]);
        }
        __syncthreads();
        if (X.warp < X.nwc) {
            unsigned long long bk = kKeyEmptyMax;
            int bj = kNone;
            const int t = X.tid, j = cl_gcol(X, t);
            if (j >= 0) {
                const double v = t < RC ? S.rowbuf[t] : X.tile[(size_t)(t - RC) * X.ld + row];
                bk = key_max(fabs(v));
                bj = j;
            }
            const unsigned long long kw = warp_max_key(bk);
            const int jw = warp_index_of(bk, kw, bj);
            if (X.lane == 0) { S.P.ckey[X.warp] = kw; S.P.cidx[X.warp] = jw; S.P.cbl[X.warp] = kNone; }
        }
        __syncthreads();
        unsigned long long kb;
        int jb, bl;
        cl_local_best<RC>(X, kb, jb, bl);
        cl_publish<RC>(X, a, jb, kb, jb, kNone);
        cl_sync();
        cl_reduce_headers<RC, 2>(X);
        __syncthreads();
        const int j = S.sel_e;
        if (j >= 0) {
            const double f = cl_fetch_col(X, S.sel_owner);
            X.par ^= 1;
            cl_pivot<RC, kClRestore>(X, a, rhs, obj, j, row, f, 0.0);
        } else {
            X.par ^= 1;
        }
        __syncthreads();
    }
}

// First staging pass of an LP's register half (its first kClSG structural
// columns of this CTA) and its b, as one asynchronous copy group.
template <int RC, int NT>
__device__ __forceinline__ void cl_issue_pass0(const ClCtx &X, const double *Ag, const double *bg, unsigned sb) {
    ClStatic<RC> &S = cl_static<RC>();
    const int w = min(kClSG, min(RC, X.ns));
    for (int i = X.warp; i < X.m; i += NT / 32)
        for (int c = X.lane; c < w; c += 32)
            cp_async8(sb + 8u * (unsigned)(c * X.ld + i), Ag + (size_t)i * X.n + X.s0 + c);
    if (X.live) cp_async8(smem_addr(&S.bpre[X.tid]), bg + X.tid);
    cp_async_commit();
}

// ---------------------------------------------------------------------------
template <int RC, int NT>
__global__ void __launch_bounds__(NT, 1)
cluster_kernel(Batch B) {
    extern __shared__ __align__(16) unsigned char smem[];
    // launched as a programmatic dependent of the lazy kernel (blp_cluster.cu cluster_fire):
    // nothing it reads (the deferral list, the LP queue) is valid before that grid completes;
    // a no-op for a plain launch
    asm volatile("griddepcontrol.wait;" ::: "memory");
    ClStatic<RC> &S = cl_static<RC>();
    const int m = B.m, n = B.n, nv = n + m;
    ClCtx X;
    X.K = (int)cl_size();
    X.rank = (int)cl_rank();
    const ClLayout L = make_cl_layout(m, n, X.K, RC);
    X.m = m; X.n = n; X.nv = nv; X.ld = L.ld; X.sn = L.sn; X.sm = L.sm; X.cpc = L.cpc; X.sc4 = L.sc4;
    X.s0 = X.rank * L.sn;
    X.q0 = X.rank * L.sm;
    X.ns = max(0, min(L.sn, n - X.s0));
    X.tid = threadIdx.x; X.lane = threadIdx.x & 31; X.warp = threadIdx.x >> 5; X.nw = NT / 32;
    X.nwc = (L.cpc + 31) >> 5;
    X.live = X.tid < m;
    X.tile = reinterpret_cast<double *>(smem);
    X.gcol = B.gtab + (size_t)cl_id() * 2 * X.K * L.ld;
    X.par = 0;
    const int ld = L.ld, sn = L.sn, ns = X.ns, s0 = X.s0, ncol4 = RC + L.sc4;
    double *stage = reinterpret_cast<double *>(smem + L.off_stage);
    const unsigned tb = smem_addr(X.tile), sb = tb + (unsigned)L.off_stage;
    // columns past the owned ones read as zero pivot-row entries: never written again
    for (int t = X.tid; t < ncol4; t += NT) S.rvec[t] = 0.0;
#ifdef BLP_CL_PROF
    if (X.tid == 0) { for (int k = 0; k < 16; ++k) S.prof[k] = 0; S.prof_t = clock64(); }
#endif
    // LP queue: rank 0 claims LP t+1 while the cluster builds LP t and publishes it
    // (by LP parity) before the build's cluster barrier: one barrier per LP.
    const long long count = batch_count(B);   // the deferred LPs when launched after the lazy kernel
    if (X.rank == 0 && X.tid == 0) S.nxt[0] = atomicAdd(B.next_lp, 1);
    cl_sync();
    long long qi = cl_ld_s64(cl_map(smem_addr(&S.nxt[0]), 0u));
    double a[RC];
    // the staging buffer holds the next LP's first pass during a solve unless rank 0
    // needs it as x scratch (the tile alone is too small for x)
    const bool prefetch_stage = (size_t)L.sc4 * ld >= (size_t)n;
    bool pre = false;

    for (int t = 0;; ++t) {
        if (qi >= count) break;                // cluster-uniform
        const long long lp = batch_lp(B, qi);
        CL_PROF_MARK(0);
        const double *Ag = B.shared_Ab ? B.A : B.A + (size_t)lp * m * n;
        const double *bg = B.shared_Ab ? B.b : B.b + (size_t)lp * m;
        const double *cg = B.c + (size_t)lp * n;
        if (X.rank == 0 && X.tid == 0) S.nxt[(t + 1) & 1] = atomicAdd(B.next_lp, 1);

        // ---- build_tableau (tableau.py:139-172): this CTA's columns, replicated rhs ----
        // Structural columns: the register half in passes of kClSG columns through the
        // staging buffer, the tile half straight into the tile; every copy an
        // asynchronous, coalesced 8-byte global->shared copy (row segments across a warp).
        const int wr = min(RC, ns), wt = max(0, ns - RC);
        if (!pre) cl_issue_pass0<RC, NT>(X, Ag, bg, sb);   // else prefetched during the previous LP
        for (int i = X.warp; i < m; i += NT / 32)
            for (int c = X.lane; c < wt; c += 32)
                cp_async8(tb + 8u * (unsigned)(c * ld + i), Ag + (size_t)i * n + s0 + RC + c);
        cp_async_commit();
        asm volatile("cp.async.wait_group 1;" ::: "memory");   // pass 0 and b landed
        __syncthreads();
        const double bi = X.live ? S.bpre[X.tid] : 0.0;
        bool nonfinite = !isfinite(bi);
        const bool neg = X.live && bi < 0.0;
        const unsigned nm = __ballot_sync(kFull, neg);
        if (X.lane == 0) S.P.wneg[X.warp] = __popc(nm);
        __syncthreads();
        int before = __popc(nm & ((1u << X.lane) - 1u));
        for (int w = 0; w < X.warp; ++w) before += S.P.wneg[w];
        const double sgn = neg ? -1.0 : 1.0;
        double rhs = X.live ? __dmul_rn(bi, sgn) : 0.0;
        if (X.live) {
            S.cbv[X.tid] = sgn;
            S.basis[X.tid] = neg ? nv + before : n + X.tid;
            if (neg) S.art_row[before] = X.tid;
        }
        CL_PROF_MARK(10);
#pragma unroll
        for (int p = 0; p < RC; p += kClSG) {
            if (p > 0) {                        // next pass into the staging buffer
                __syncthreads();
                for (int i = X.warp; i < m; i += NT / 32)
                    for (int c = X.lane; c < min(kClSG, wr - p); c += 32)
                        cp_async8(sb + 8u * (unsigned)(c * ld + i), Ag + (size_t)i * n + s0 + p + c);
                cp_async_commit();
                cp_async_wait_all();
                __syncthreads();
            }
#pragma unroll
            for (int c = p; c < p + kClSG && c < RC; ++c) {
                double v = 0.0;
                if (X.live) {
                    if (c < wr) {
                        const double g = stage[(size_t)(c - p) * ld + X.tid];
                        nonfinite |= !isfinite(g);
                        v = __dmul_rn(g, sgn);
                    } else if (c >= sn && c < L.cpc && X.q0 + c - sn == X.tid) {
                        v = sgn;                // this row's slack entry
                    }
                }
                a[c] = v;
            }
        }
        CL_PROF_MARK(11);
        // tile slack / unowned columns: the identity part of [A | I] (tableau.py:157-170),
        // signs from cbv (published by the pass barrier above)
        for (int tc = wt + X.warp; tc < L.sc4; tc += NT / 32) {
            const int c = RC + tc, q = X.q0 + c - sn;
            const bool slack = c >= sn && c < L.cpc && q < m;
            for (int i = X.lane; i < m; i += 32) X.tile[(size_t)tc * ld + i] = (slack && i == q) ? S.cbv[i] : 0.0;
        }
        cp_async_wait_all();
        __syncthreads();
        if (X.live) {                           // A * sign (tableau.py:157-158) and validation, tile half
            double *p = X.tile + X.tid;
            for (int c = 0; c < wt; ++c, p += ld) {
                const double v = *p;
                nonfinite |= !isfinite(v);
                if (neg) *p = __dmul_rn(v, -1.0);
            }
        }
        CL_PROF_MARK(12);
        for (int tt = X.tid; tt < ncol4; tt += NT) {
            const int j = cl_gcol(X, tt);
            S.rcv[tt] = (j >= 0 && j < n) ? cg[j] : 0.0;   // phase 2 runs on c directly when feasible
            S.arc[tt] = 0.0;
            S.artk[tt] = (j >= n && S.basis[j - n] >= nv) ? S.basis[j - n] - nv : -1;
        }
        for (int j = X.tid; j < n; j += NT) nonfinite |= !isfinite(cg[j]);
        for (int j = X.tid; j < nv + m; j += NT) S.isb[j] = 0;
        const int n_art = __syncthreads_count(neg);
        if (X.live) S.isb[S.basis[X.tid]] = 1;
        const int inv_local = __syncthreads_or(nonfinite);
        if (X.tid == 0) S.inv[t & 1] = inv_local;
        CL_PROF_MARK(13);
        cl_sync();                              // the build's only cluster barrier
        CL_PROF_MARK(14);
        int inv = 0;
        if (X.lane < X.K) inv = cl_ld_s32(cl_map(smem_addr(&S.inv[t & 1]), (unsigned)X.lane));
        const bool invalid = __any_sync(kFull, inv != 0);
        const long long qn = cl_ld_s64(cl_map(smem_addr(&S.nxt[(t + 1) & 1]), 0u));
        const long long lpn = qn < count ? batch_lp(B, qn) : B.count;
        // next LP: its first staging pass and b straight into shared memory (the staging
        // buffer is idle until then), the rest of its rows of this CTA's columns into L2
        pre = lpn < B.count && prefetch_stage;
        if (pre) {
            __syncthreads();                    // everyone is done with the staging buffer
            cl_issue_pass0<RC, NT>(X, B.shared_Ab ? B.A : B.A + (size_t)lpn * m * n,
                                   B.shared_Ab ? B.b : B.b + (size_t)lpn * m, sb);
        }
        if (lpn < B.count && !B.shared_Ab && X.live && ns > 0) {
            const char *g0 = reinterpret_cast<const char *>(B.A + ((size_t)lpn * m + X.tid) * n + s0);
            const char *g1 = reinterpret_cast<const char *>(B.A + ((size_t)lpn * m + X.tid) * n + s0 + ns);
            for (const char *g = reinterpret_cast<const char *>((size_t)g0 & ~(size_t)127); g < g1; g += 128)
                prefetch_l2(g);
            if ((X.tid & 15) == 0) prefetch_l2(B.b + (size_t)lpn * m + X.tid);
        }
        CL_PROF_MARK(1);

        int8_t status = kOptimal;
        int it1 = 0, it2 = 0;
        bool done = false;
        double obj = 0.0;
        if (invalid) {
            status = kInvalid;
            done = true;
        } else if (n_art > 0) {
            cl_price_out<RC, 1>(X, a, rhs, obj, cg);                        // build_auxiliary
            const ClPhase p1 = cl_run_phase<RC, kClPhase1>(X, a, rhs, obj, B.lim);
            it1 = p1.iters;
            if (p1.state == 2) { status = kIterationLimit; done = true; }
            else if (p1.state == 1) { status = kErrPhase1Unbounded; done = true; }
            else if (fabs(obj) > kPhase1ZeroTol) { status = kInfeasible; done = true; }
            else {
                cl_restore<RC>(X, a, rhs, obj);
                cl_price_out<RC, 2>(X, a, rhs, obj, cg);
            }
        } else {
            if (X.warp < X.nwc) cl_candidates<RC, kClPhase2>(X, -1, -1);
            __syncthreads();
        }
        if (!done) {
            const ClPhase p2 = cl_run_phase<RC, kClPhase2>(X, a, rhs, obj, B.lim);
            it2 = p2.iters;
            if (p2.state == 2) status = kIterationLimit;
            else if (p2.state == 1) status = kUnbounded;
        }
        CL_PROF_MARK(2);

        // ---- _extract_point (simplex.py:146-151) and c @ x, by rank 0 ----
        __syncthreads();
        if (X.rank == 0) {
            double *xs = X.tile;                // tile + staging: >= n doubles (planner); the tile alone when prefetching
            for (int j = X.tid; j < n; j += NT) xs[j] = 0.0;
            __syncthreads();
            if (status == kOptimal && X.live && S.basis[X.tid] < n) xs[S.basis[X.tid]] = rhs;
            __syncthreads();
            double *xg = B.x + (size_t)lp * n;
            for (int j = X.tid; j < n; j += NT) {   // x out; products c_j x_j in place (parallel)
                const double xj = xs[j];
                xg[j] = xj;
                xs[j] = __dmul_rn(cg[j], xj);
            }
            __syncthreads();
            if (X.warp == 0) {
                // c @ x left to right (the oracle's order; see blp_lazy_kernel.cuh)
                double s = 0.0;
                if (status == kOptimal && X.lane == 0)
                    for (int j = 0; j < n; ++j) {
                        const double p = xs[j];
                        if (p != 0.0) s = __dadd_rn(s, p);
                    }
                if (X.lane == 0) {
                    B.objective[lp] = status == kOptimal ? s : __longlong_as_double(0x7ff8000000000000LL);
                    B.status[lp] = status;
                    B.it1[lp] = it1;
                    B.it2[lp] = it2;
                }
            }
        }
        __syncthreads();
        CL_PROF_MARK(7);
        qi = qn;
    }
    cl_sync();                                  // no CTA leaves while its shared memory may still be read
#ifdef BLP_CL_PROF
    if (X.tid == 0)
        for (int k = 0; k < 16; ++k) atomicAdd(&g_cl_prof[k], S.prof[k]);
#endif
}

}  // namespace blp
