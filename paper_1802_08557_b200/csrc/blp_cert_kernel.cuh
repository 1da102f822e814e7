// blp_cert_kernel.cuh -- batched from-scratch optimality certificates
// (reference oracle.py:168-223 check_certificate).
//
// For every LP whose status is OPTIMAL, nothing is read from the solver
// except the primal point x:
//   max_violation  = max(0, max_i (A x - b)_i)
//   max_negativity = max(0, max_j -x_j)
//   a basis of [A | I] is rebuilt greedily from the point's support -- the
//   columns with level > tol first (x_j, then the slacks b - A x), then the
//   rest, each in index order -- keeping a column iff it raises the rank;
//   duals solve B^T y = c_B; max_reduced_cost = max(c_ext - [A | I]^T y).
// The rank test is classical Gram-Schmidt with one re-orthogonalisation
// (CGS2): a column is independent iff its residual norm exceeds
// |trial|_F * max(m, k) * eps, the SVD-rank threshold numpy's matrix_rank
// applies (with the Frobenius norm bounding the largest singular value).
// B = QR is then used directly: R^T z = c_B, y = Q z.
// When the basis route leaves max_reduced_cost > tol on a primal-feasible
// point, the LP is flagged (needs_prices): the reference then searches for
// complementary-slackness prices with an auxiliary LP (oracle.py:226-242);
// the host layer solves that LP with the batched simplex itself and
// re-prices with cert_prices_kernel.
//
// One CTA per LP (grid-stride), threads over rows / columns; Q and R live in
// a per-CTA global workspace (2 m^2 doubles, L2-resident at these sizes).
#pragma once

#include <cfloat>

#include "blp_common.cuh"

namespace blp {

struct CertBatch {
    const double *A, *b, *c, *x;   // A [count][m][n] (or [m][n] when shared_Ab), b [count][m], c/x [count][n]
    long long count;
    int m, n, shared_Ab;
    const int8_t *status;          // solver status; only OPTIMAL (0) LPs are certified
    double tol;
    double *max_rc, *max_viol, *max_neg;
    int8_t *needs_prices;
    double *work;                  // [gridDim.x][2 m m]
};

constexpr int kCertThreads = 128;

__device__ __forceinline__ double cert_warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

__device__ __forceinline__ double cert_warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

// Block-wide sum / max; every thread gets the result.  `red` holds 32 doubles.
__device__ __forceinline__ double cert_block_sum(double v, double *red) {
    v = cert_warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s = __dadd_rn(s, red[k]);
    return s;
}

__device__ __forceinline__ double cert_block_max(double v, double *red) {
    v = cert_warp_max(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = -INFINITY;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s = fmax(s, red[k]);
    return s;
}

__global__ void __launch_bounds__(kCertThreads) cert_kernel(CertBatch B) {
    extern __shared__ __align__(16) double csm[];
    const int m = B.m, n = B.n, t = threadIdx.x, NT = blockDim.x;
    double *xs = csm;              // n
    double *lev = xs + n;          // n + m: [x | b - A x]
    double *ax = lev + n + m;      // m
    double *v = ax + m;            // m   candidate column / residual
    double *coef = v + m;          // m   projections of one CGS pass
    double *racc = coef + m;       // m   accumulated projections (R column)
    double *w = racc + m;          // m   forward-substitution right-hand side
    double *z = w + m;             // m
    double *y = z + m;             // m
    double *cB = y + m;            // m
    double *red = cB + m;          // 32
    double *Q = B.work + (size_t)blockIdx.x * 2 * m * m;   // Q[i*m + k], column k = k-th basis direction
    double *R = Q + (size_t)m * m;                          // R[k*m + j], upper triangle
    const double nan = __longlong_as_double(0x7ff8000000000000LL);

    for (long long lp = blockIdx.x; lp < B.count; lp += gridDim.x) {
        if (B.status[lp] != 0) {
            if (t == 0) {
                B.max_rc[lp] = nan; B.max_viol[lp] = nan; B.max_neg[lp] = nan; B.needs_prices[lp] = 0;
            }
            continue;
        }
        const double *A = B.shared_Ab ? B.A : B.A + (size_t)lp * m * n;
        const double *b = B.shared_Ab ? B.b : B.b + (size_t)lp * m;
        const double *c = B.c + (size_t)lp * n;
        const double *x = B.x + (size_t)lp * n;
        __syncthreads();
        for (int j = t; j < n; j += NT) { xs[j] = x[j]; lev[j] = x[j]; }
        __syncthreads();
        // A x: one warp per row, lanes over columns
        for (int i = t >> 5; i < m; i += NT >> 5) {
            double s = 0.0;
            for (int j = t & 31; j < n; j += 32) s = __dadd_rn(s, __dmul_rn(A[(size_t)i * n + j], xs[j]));
            s = cert_warp_sum(s);
            if ((t & 31) == 0) ax[i] = s;
        }
        __syncthreads();
        double vmax = 0.0, nmax = 0.0;
        for (int i = t; i < m; i += NT) {
            const double r = __dsub_rn(ax[i], b[i]);
            vmax = fmax(vmax, r);
            lev[n + i] = -r;                          // b - A x
        }
        for (int j = t; j < n; j += NT) nmax = fmax(nmax, -xs[j]);
        const double viol = cert_block_max(vmax, red);
        const double negv = cert_block_max(nmax, red);
        double maxrc;
        if (m == 0) {
            double cm = 0.0;
            for (int j = t; j < n; j += NT) cm = fmax(cm, c[j]);
            maxrc = cert_block_max(cm, red);
        } else {
            // ---- greedy basis of [A | I]: support columns first, then the rest
            int rank = 0;
            double frob2 = 0.0;
            for (int pass = 0; pass < 2 && rank < m; ++pass) {
                for (int j = 0; j < n + m && rank < m; ++j) {
                    const bool pos = lev[j] > B.tol;
                    if (pos != (pass == 0)) continue;        // uniform: lev is in smem
                    double part = 0.0;
                    for (int i = t; i < m; i += NT) {
                        const double a = j < n ? A[(size_t)i * n + j] : (i == j - n ? 1.0 : 0.0);
                        v[i] = a;
                        part = __dadd_rn(part, __dmul_rn(a, a));
                    }
                    const double cn2 = cert_block_sum(part, red);
                    for (int k = t; k < rank; k += NT) racc[k] = 0.0;
                    for (int rep = 0; rep < 2 && rank > 0; ++rep) {
                        __syncthreads();
                        for (int k = t; k < rank; k += NT) {
                            double s = 0.0;
                            for (int i = 0; i < m; ++i) s = __dadd_rn(s, __dmul_rn(Q[(size_t)i * m + k], v[i]));
                            coef[k] = s;
                            racc[k] = __dadd_rn(racc[k], s);
                        }
                        __syncthreads();
                        for (int i = t; i < m; i += NT) {
                            double s = v[i];
                            for (int k = 0; k < rank; ++k) s = __dsub_rn(s, __dmul_rn(Q[(size_t)i * m + k], coef[k]));
                            v[i] = s;
                        }
                    }
                    part = 0.0;
                    for (int i = t; i < m; i += NT) part = __dadd_rn(part, __dmul_rn(v[i], v[i]));
                    const double nrm = sqrt(cert_block_sum(part, red));
                    const double thr = sqrt(__dadd_rn(frob2, cn2)) * (double)max(m, rank + 1) * DBL_EPSILON;
                    if (nrm > thr) {
                        for (int i = t; i < m; i += NT) Q[(size_t)i * m + rank] = __ddiv_rn(v[i], nrm);
                        for (int k = t; k < rank; k += NT) R[(size_t)k * m + rank] = racc[k];
                        if (t == 0) {
                            R[(size_t)rank * m + rank] = nrm;
                            cB[rank] = j < n ? c[j] : 0.0;
                        }
                        frob2 = __dadd_rn(frob2, cn2);
                        ++rank;
                    }
                    __syncthreads();
                }
            }
            if (rank < m) {
                maxrc = nan;                                 // singular basis (np.linalg.solve raises)
            } else {
                // R^T z = c_B (forward substitution), then y = Q z
                for (int k = t; k < m; k += NT) w[k] = cB[k];
                __syncthreads();
                for (int k = 0; k < m; ++k) {
                    const double zk = __ddiv_rn(w[k], R[(size_t)k * m + k]);
                    for (int i = k + 1 + t; i < m; i += NT) w[i] = __dsub_rn(w[i], __dmul_rn(R[(size_t)k * m + i], zk));
                    if (t == 0) z[k] = zk;
                    __syncthreads();
                }
                for (int i = t; i < m; i += NT) {
                    double s = 0.0;
                    for (int k = 0; k < m; ++k) s = __dadd_rn(s, __dmul_rn(Q[(size_t)i * m + k], z[k]));
                    y[i] = s;
                }
                __syncthreads();
                double rmax = -INFINITY;
                for (int j = t; j < n; j += NT) {
                    double s = 0.0;
                    for (int i = 0; i < m; ++i) s = __dadd_rn(s, __dmul_rn(A[(size_t)i * n + j], y[i]));
                    rmax = fmax(rmax, __dsub_rn(c[j], s));
                }
                for (int i = t; i < m; i += NT) rmax = fmax(rmax, -y[i]);
                maxrc = cert_block_max(rmax, red);
            }
        }
        if (t == 0) {
            B.max_rc[lp] = maxrc;
            B.max_viol[lp] = viol;
            B.max_neg[lp] = negv;
            B.needs_prices[lp] = (maxrc > B.tol && viol <= B.tol && negv <= B.tol) ? 1 : 0;
        }
    }
}

// Re-price flagged LPs with complementary prices y [count][m] (solved by the
// batched simplex): max(c - A^T y, -y), one warp per LP.
struct CertPrices {
    const double *A, *c, *y;
    long long count;
    int m, n, shared_Ab;
    const int8_t *mask;            // 1 = replace max_rc[k]
    double *max_rc;
};

__global__ void __launch_bounds__(256) cert_prices_kernel(CertPrices P) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long k = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < P.count; k += warps) {
        if (!P.mask[k]) continue;
        const double *A = P.shared_Ab ? P.A : P.A + (size_t)k * P.m * P.n;
        const double *c = P.c + (size_t)k * P.n;
        const double *y = P.y + (size_t)k * P.m;
        double r = -INFINITY;
        for (int j = lane; j < P.n; j += 32) {
            double s = 0.0;
            for (int i = 0; i < P.m; ++i) s = __dadd_rn(s, __dmul_rn(A[(size_t)i * P.n + j], y[i]));
            r = fmax(r, __dsub_rn(c[j], s));
        }
        for (int i = lane; i < P.m; i += 32) r = fmax(r, -y[i]);
        r = cert_warp_max(r);
        if (lane == 0) P.max_rc[k] = r;
    }
}

}  // namespace blp
