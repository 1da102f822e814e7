/*
 * blp_oracle.c -- CPU restatement of the reference two-phase dense tableau
 * simplex (batchlp 0.1.0, /root/reference/pkg/src/batchlp/{tableau,simplex}.py).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path and the CPU baseline timed by bench.py; the product path
 * (paper_1802_08557_b200/) never links, imports or calls it.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.
 *
 * Deliberately NOT the GPU algorithm: it keeps the reference's full tableau
 * (structural | slack | artificial | rhs columns, column-major, element
 * (i,j) at j*p+i -- tableau.py:56-79) including the artificial columns the
 * GPU kernel elides, so it checks the elision independently.
 *
 * Arithmetic follows numpy's IEEE-754 elementwise semantics: every
 * multiply and subtract is rounded separately (build with
 * -ffp-contract=off), divisions are IEEE, arg-reductions take the FIRST
 * max/min with NaN treated as the extreme value (numpy argmax/argmin).
 * The one non-elementwise op of the reference, the objective c @ x
 * (simplex.py:190, BLAS ddot with implementation-defined order), is a
 * left-to-right sum here; callers compare it at 1e-9 relative.
 *
 * Parity pinned against the reference itself: the fixtures in tests/golden/ were
 * produced by running the imported reference (tests/golden/make_golden.py).
 */
#include <math.h>
#include <pthread.h>
#include <unistd.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_SENTINEL 1e308          /* tableau.py:37 */
#define OR_TOL 1e-9                /* tableau.py:38 DEFAULT_TOL */
#define OR_PHASE1_ZERO_TOL 1e-7    /* simplex.py:26 */
#define OR_DEGENERATE_TOL 1e-9     /* simplex.py:27 */
#define OR_REDUNDANT_TOL 1e-7      /* simplex.py:31 */

enum { OR_OPTIMAL = 0, OR_UNBOUNDED = 1, OR_INFEASIBLE = 2, OR_ITERATION_LIMIT = 3,
       OR_ERR_PHASE1_UNBOUNDED = 4, OR_ERR_NOMEM = 5 };

typedef struct {
    int32_t max_iterations;   /* <= 0: 50*(m+n)     (simplex.py:52-55) */
    int32_t anti_cycling;     /* 0/1                (simplex.py:45)    */
    int32_t degenerate_limit; /* < 0: max(m,1)      (simplex.py:57-60) */
    int32_t reserved;
} or_limits;

typedef struct {
    int n, m, n_art;
    int p, nv, q;          /* rows, variable columns, total columns (tableau.py:61-65) */
    double *v;             /* p*q, column-major */
    int *basis;            /* m basic-variable indices (the reference stores them as floats in column nv+1) */
    unsigned char *sel;    /* nv selectable flags (tableau.py:71) */
    unsigned char *isb;    /* nv "is basic" flags, derived from basis */
} tab;

#define CELL(t, i, j) ((t)->v[(size_t)(j) * (size_t)(t)->p + (size_t)(i)])

/* numpy argmax: first maximum, NaN counts as maximal (first NaN wins). */
static int np_better_max(double a, double b) {
    if (isnan(b)) return 0;
    if (isnan(a)) return 1;
    return a > b;
}
/* numpy argmin: first minimum, NaN counts as minimal. */
static int np_better_min(double a, double b) {
    if (isnan(b)) return 0;
    if (isnan(a)) return 1;
    return a < b;
}

static void tab_free(tab *t) {
    free(t->v); free(t->basis); free(t->sel); free(t->isb);
}

/* build_tableau, tableau.py:139-172 */
static int tab_build(tab *t, const double *A, const double *b, const double *c, int m, int n) {
    int n_art = 0;
    for (int i = 0; i < m; ++i) n_art += (b[i] < 0);
    t->n = n; t->m = m; t->n_art = n_art;
    t->p = m + 1; t->nv = n + m + n_art; t->q = t->nv + 2;
    t->v = (double *)calloc((size_t)t->p * t->q, sizeof(double));
    t->basis = (int *)malloc(sizeof(int) * (m > 0 ? m : 1));
    t->sel = (unsigned char *)malloc(t->nv > 0 ? t->nv : 1);
    t->isb = (unsigned char *)calloc(t->nv > 0 ? t->nv : 1, 1);
    if (!t->v || !t->basis || !t->sel || !t->isb) { tab_free(t); return -1; }
    memset(t->sel, 1, t->nv);
    int rhs = t->nv, k = 0;
    for (int i = 0; i < m; ++i) {
        double s = b[i] < 0 ? -1.0 : 1.0;
        for (int j = 0; j < n; ++j) CELL(t, i, j) = A[(size_t)i * n + j] * s;
        CELL(t, i, rhs) = b[i] * s;
        CELL(t, i, n + i) = s;
        if (b[i] < 0) { CELL(t, i, n + m + k) = 1.0; t->basis[i] = n + m + k; ++k; }
        else t->basis[i] = n + i;
        t->isb[t->basis[i]] = 1;
    }
    for (int j = 0; j < n; ++j) CELL(t, m, j) = c[j];
    return 0;
}

/* choose_entering, tableau.py:175-186 (Dantzig, first max, <= tol means optimal) */
static int tab_enter_dantzig(const tab *t) {
    int best = -1; double bv = -INFINITY; int any = 0;
    for (int j = 0; j < t->nv; ++j) {
        if (!t->sel[j] || t->isb[j]) continue;
        any = 1;
        double v = CELL(t, t->m, j);
        if (best < 0 || np_better_max(v, bv)) { best = j; bv = v; }
    }
    if (!any) return -1;
    /* masked columns are -inf in the reference; an all -inf row leaves the
     * first index selected and still fails the tol test below */
    if (bv <= OR_TOL) return -1;
    return best;
}

/* choose_entering_bland, tableau.py:189-197 */
static int tab_enter_bland(const tab *t) {
    for (int j = 0; j < t->nv; ++j)
        if (t->sel[j] && !t->isb[j] && CELL(t, t->m, j) > OR_TOL) return j;
    return -1;
}

/* choose_leaving, tableau.py:200-215; *ratio_out gets the ratio of the chosen row */
static int tab_leave(const tab *t, int e, double *ratio_out) {
    if (t->m == 0) return -1;
    int best = 0; double bv = 0.0;
    for (int i = 0; i < t->m; ++i) {
        double a = CELL(t, i, e);
        double r = (a > OR_TOL) ? CELL(t, i, t->nv) / a : OR_SENTINEL;
        if (i == 0 || np_better_min(r, bv)) { best = i; bv = r; }
    }
    if (bv >= OR_SENTINEL) return -1;
    *ratio_out = bv;
    return best;
}

/* pivot, tableau.py:218-244.  scratch holds p doubles. */
static void tab_pivot(tab *t, int e, int l, double *f) {
    const int p = t->p, width = t->nv + 1;
    const double pe = CELL(t, l, e);
    for (int i = 0; i < p; ++i) f[i] = CELL(t, i, e);
    f[l] = 0.0;
    const double obj_before = CELL(t, t->m, t->nv);
    const double rc_e = f[t->m];
    for (int j = 0; j < width; ++j) {
        double *col = &t->v[(size_t)j * p];
        double r = col[l] / pe;
        col[l] = r;
        for (int i = 0; i < p; ++i) {
            double prod = f[i] * r;
            col[i] = col[i] - prod;
        }
    }
    double rhs_new = CELL(t, l, t->nv);
    double inc = rc_e * rhs_new;
    CELL(t, t->m, t->nv) = obj_before + inc;
    t->isb[t->basis[l]] = 0;
    t->basis[l] = e;
    t->isb[e] = 1;
}

/* _run_phase, simplex.py:63-91.  Returns 0 optimal, 1 unbounded, 2 iteration limit. */
static int tab_run_phase(tab *t, const or_limits *lim, int *iters, double *f) {
    const int max_iter = lim->max_iterations > 0 ? lim->max_iterations : 50 * (t->m + t->n);
    const int trigger = lim->degenerate_limit >= 0 ? lim->degenerate_limit : (t->m > 1 ? t->m : 1);
    int degenerate_run = 0, use_bland = 0;
    for (int it = 0; it < max_iter; ++it) {
        int e = use_bland ? tab_enter_bland(t) : tab_enter_dantzig(t);
        if (e < 0) { *iters = it; return 0; }
        double ratio = 0.0;
        int l = tab_leave(t, e, &ratio);
        if (l < 0) { *iters = it; return 1; }
        tab_pivot(t, e, l, f);
        if (ratio <= OR_DEGENERATE_TOL) {
            ++degenerate_run;
            if (lim->anti_cycling && degenerate_run >= trigger) use_bland = 1;
        } else {
            degenerate_run = 0;
            use_bland = 0;
        }
    }
    *iters = max_iter;
    return 2;
}

/* _price_out, simplex.py:133-143: rebuild the last row from c_ext (length nv) */
static void tab_price_out(tab *t, const double *c_ext) {
    const int m = t->m, nv = t->nv;
    double *rc = (double *)malloc(sizeof(double) * (nv > 0 ? nv : 1));
    memcpy(rc, c_ext, sizeof(double) * nv);
    double obj = 0.0;
    for (int row = 0; row < m; ++row) {
        double cb = c_ext[t->basis[row]];
        if (cb != 0.0) {
            for (int j = 0; j < nv; ++j) { double prod = cb * CELL(t, row, j); rc[j] = rc[j] - prod; }
            double prod = cb * CELL(t, row, nv);
            obj = obj + prod;
        }
    }
    for (int j = 0; j < nv; ++j) CELL(t, m, j) = rc[j];
    CELL(t, m, nv) = obj;
    free(rc);
}

/* build_auxiliary, simplex.py:94-106 */
static void tab_build_auxiliary(tab *t) {
    double *c_aux = (double *)calloc(t->nv > 0 ? t->nv : 1, sizeof(double));
    for (int j = t->n + t->m; j < t->nv; ++j) c_aux[j] = -1.0;
    tab_price_out(t, c_aux);
    free(c_aux);
}

/* restore_objective, simplex.py:109-130 */
static void tab_restore(tab *t, const double *c, double *f) {
    const int first_art = t->n + t->m;
    for (int j = first_art; j < t->nv; ++j) t->sel[j] = 0;
    for (int row = 0; row < t->m; ++row) {
        if (t->basis[row] < first_art) continue;
        int best = 0; double bv = 0.0;
        for (int j = 0; j < t->nv; ++j) {
            double v = t->sel[j] ? fabs(CELL(t, row, j)) : 0.0;
            if (j == 0 || np_better_max(v, bv)) { best = j; bv = v; }
        }
        if (bv > OR_REDUNDANT_TOL) tab_pivot(t, best, row, f);
    }
    double *c_ext = (double *)calloc(t->nv > 0 ? t->nv : 1, sizeof(double));
    for (int j = 0; j < t->n; ++j) c_ext[j] = c[j];
    tab_price_out(t, c_ext);
    free(c_ext);
}

/* solve, simplex.py:154-194 (validation is the caller's job, model.py:263-301) */
static int or_solve_one(const double *A, const double *b, const double *c, int m, int n,
                        const or_limits *lim, double *objective, double *x,
                        int32_t *it1, int32_t *it2) {
    tab t;
    *it1 = 0; *it2 = 0; *objective = NAN;
    for (int j = 0; j < n; ++j) x[j] = 0.0;
    if (tab_build(&t, A, b, c, m, n)) return OR_ERR_NOMEM;
    double *f = (double *)malloc(sizeof(double) * t.p);
    int status;
    if (t.n_art > 0) {
        tab_build_auxiliary(&t);
        int iters = 0;
        int st = tab_run_phase(&t, lim, &iters, f);
        *it1 = iters;
        if (st == 2) { status = OR_ITERATION_LIMIT; goto done; }
        if (st == 1) { status = OR_ERR_PHASE1_UNBOUNDED; goto done; }
        if (fabs(CELL(&t, t.m, t.nv)) > OR_PHASE1_ZERO_TOL) { status = OR_INFEASIBLE; goto done; }
        tab_restore(&t, c, f);
    }
    {
        int iters = 0;
        int st = tab_run_phase(&t, lim, &iters, f);
        *it2 = iters;
        if (st == 2) { status = OR_ITERATION_LIMIT; goto done; }
        if (st == 1) { status = OR_UNBOUNDED; goto done; }
    }
    /* _extract_point, simplex.py:146-151 */
    for (int i = 0; i < t.m; ++i)
        if (t.basis[i] < n) x[t.basis[i]] = CELL(&t, i, t.nv);
    {
        double s = 0.0;
        for (int j = 0; j < n; ++j) { double prod = c[j] * x[j]; s = s + prod; }
        *objective = s;
    }
    status = OR_OPTIMAL;
done:
    free(f);
    tab_free(&t);
    return status;
}

typedef struct {
    const double *A, *b, *c;
    int64_t count, next;
    int32_t m, n, shared_Ab;
    const or_limits *lim;
    int8_t *status; double *objective, *x; int32_t *it1, *it2;
    pthread_mutex_t mu;
} or_job;

static void *or_worker(void *arg) {
    or_job *J = (or_job *)arg;
    const int64_t grain = 16;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        int64_t k0 = J->next;
        J->next += grain;
        pthread_mutex_unlock(&J->mu);
        if (k0 >= J->count) break;
        int64_t k1 = k0 + grain < J->count ? k0 + grain : J->count;
        for (int64_t k = k0; k < k1; ++k) {
            const size_t m = (size_t)J->m, n = (size_t)J->n;
            const double *Ak = J->shared_Ab ? J->A : J->A + (size_t)k * m * n;
            const double *bk = J->shared_Ab ? J->b : J->b + (size_t)k * m;
            int st = or_solve_one(Ak, bk, J->c + (size_t)k * n, J->m, J->n, J->lim,
                                  &J->objective[k], J->x + (size_t)k * n, &J->it1[k], &J->it2[k]);
            J->status[k] = (int8_t)st;
            if (st != OR_OPTIMAL) {
                J->objective[k] = NAN;
                for (size_t j = 0; j < n; ++j) J->x[(size_t)k * n + j] = 0.0;
            }
        }
    }
    return NULL;
}

/*
 * Batched entry: A [count][m][n] row-major, b [count][m], c [count][n]
 * (shared_Ab != 0: A [m][n] and b [m] shared by all, c per LP).
 * Outputs status [count], objective [count] (NaN unless optimal),
 * x [count][n] (zero unless optimal), it1/it2 [count].
 * nthreads <= 0: all online cores.  Returns the thread count used.
 */
int oracle_solve_batch(const double *A, const double *b, const double *c, int64_t count,
                       int32_t m, int32_t n, int32_t shared_Ab, const or_limits *lim,
                       int8_t *status, double *objective, double *x,
                       int32_t *it1, int32_t *it2, int32_t nthreads) {
    int nt = nthreads > 0 ? nthreads : (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nt < 1) nt = 1;
    if ((int64_t)nt > count) nt = count > 0 ? (int)count : 1;
    or_job J = {A, b, c, count, 0, m, n, shared_Ab, lim, status, objective, x, it1, it2,
                PTHREAD_MUTEX_INITIALIZER};
    if (nt == 1) { or_worker(&J); return 1; }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nt);
    for (int i = 0; i < nt; ++i) pthread_create(&th[i], NULL, or_worker, &J);
    for (int i = 0; i < nt; ++i) pthread_join(th[i], NULL);
    free(th);
    return nt;
}
