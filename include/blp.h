/*
 * blp.h -- C ABI of the B200 batched two-phase dense simplex (libblp.so).
 *
 * The reference (batchlp 0.1.0, /root/reference/pkg/src/batchlp) is a pure
 * Python package with no C ABI.  Its drop-in boundary for the hot path is the
 * Python pair re-exported from batchlp/__init__.py:3-12,37:
 *
 *   batch_solve(lps, config) -> BatchReport      batch.py:134-179
 *   solve(lp, limits)        -> SolveOutcome     simplex.py:154-194
 *
 * Every entry point below replaces the per-LP body of those functions
 * (validate -> build_tableau -> phase 1 -> restore_objective -> phase 2 ->
 * _extract_point) for a whole packed batch; the Python package
 * paper_1802_08557_b200 keeps the reference's object API on top of it
 * (INTEGRATION.md shows the ctypes binding).  Plain pointers and sizes only.
 *
 * Input layout (packed, same shape (m, n) for the whole batch, as
 * batch.py:141-144 requires):
 *   A  [count][m][n] fp64 row-major   (StandardFormLP.A, model.py:105-107)
 *   b  [count][m]    fp64
 *   c  [count][n]    fp64
 * With shared_Ab != 0 (support-function mode) A is [m][n] and b is [m],
 * shared by every LP; only c differs per LP.
 *
 * Output layout:
 *   status     [count] int8   BLP_STATUS_* (model.py:29-33 order)
 *   objective  [count] fp64   c.x when OPTIMAL, NaN otherwise (simplex.py:187-194)
 *   x          [count][n] fp64 primal point when OPTIMAL, zeros otherwise
 *   iters1/2   [count] int32  pivots in phase 1 / phase 2 (SolveOutcome, model.py:137-138)
 *
 * Results are bit-identical to the reference's pivot sequence: status, x and
 * iteration counts equal the reference's exactly; objective agrees to 1e-9
 * relative (the reference sums c.x with BLAS ddot, whose order is unpinned).
 * Finiteness validation (model.py:263-301) is fused into the kernels' tableau
 * build: an LP with a non-finite entry gets BLP_STATUS_INVALID and is not
 * solved; the caller turns it into the reference's ValueError.
 */
#ifndef BLP_H_
#define BLP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BLP_ABI_VERSION 1

/* Per-LP status codes.  0-3 mirror Status (model.py:29-33). */
#define BLP_STATUS_OPTIMAL 0
#define BLP_STATUS_UNBOUNDED 1
#define BLP_STATUS_INFEASIBLE 2
#define BLP_STATUS_ITERATION_LIMIT 3
/* phase 1 reported unbounded: the reference raises RuntimeError (simplex.py:173-175) */
#define BLP_STATUS_ERR_PHASE1_UNBOUNDED 4
/* a non-finite entry in A, b or c: the reference's solve raises
 * ValueError("invalid LP: ...") from validate() (simplex.py:162-164) */
#define BLP_STATUS_INVALID 5

/* Return codes of the entry points. */
#define BLP_OK 0
#define BLP_ERR_INVALID -1     /* bad argument (negative sizes, null pointers) */
#define BLP_ERR_CUDA -2        /* CUDA runtime error; see blp_last_error() */
#define BLP_ERR_TOO_LARGE -3   /* the LP shape exceeds every kernel variant */

/* SolverLimits, simplex.py:34-60.  Tolerances are the reference's module
 * constants (tableau.py:37-39, simplex.py:26-31) compiled into the kernels. */
typedef struct blp_limits {
    int32_t max_iterations;   /* <= 0: 50*(m+n) per phase (SolverLimits.iterations_for) */
    int32_t anti_cycling;     /* 0 or 1 (SolverLimits.anti_cycling)                    */
    int32_t degenerate_limit; /* < 0: max(m,1) (SolverLimits.bland_trigger)             */
    int32_t reserved;         /* must be 0                                              */
} blp_limits;

/*
 * Device-resident batch solve.  All array pointers are device pointers on
 * `device`'s current context; work is enqueued on `cuda_stream` (a
 * cudaStream_t, NULL = legacy default stream) and the call returns without
 * synchronising.  Replaces the per-LP loop of batch.py:162-173 / simplex.py:154-194.
 */
int blp_solve_batch_device(const double *A, const double *b, const double *c,
                           int64_t count, int32_t m, int32_t n, int32_t shared_Ab,
                           const blp_limits *limits,
                           int8_t *status, double *objective, double *x,
                           int32_t *iters1, int32_t *iters2,
                           void *cuda_stream);

/*
 * Host-buffer batch solve (the reference-facing call: batch_solve's
 * Sequence[StandardFormLP] packed into host arrays).  Copies inputs to
 * `device`, solves, copies results back, and returns when the host output
 * buffers are filled.  Large batches are pipelined in sub-batches over
 * several streams so host<->device copies overlap the kernels.  Pinned host
 * buffers give full PCIe bandwidth; pageable ones work but copy slower.
 */
int blp_solve_batch_host(const double *A, const double *b, const double *c,
                         int64_t count, int32_t m, int32_t n, int32_t shared_Ab,
                         const blp_limits *limits,
                         int8_t *status, double *objective, double *x,
                         int32_t *iters1, int32_t *iters2,
                         int32_t device);

/*
 * Host batch solve from one pointer per LP array -- the reference's object API
 * (batch_solve(lps: Sequence[StandardFormLP]), batch.py:134-179) without packing:
 * A[k] -> that LP's m x n row-major fp64 matrix, b[k] -> m values, c[k] -> n
 * values (StandardFormLP.A / .b / .c, model.py:103-105).  The library copies
 * them with host threads straight into its pinned staging ring, overlapped with
 * the H2D / kernel / D2H of earlier sub-batches; outputs as blp_solve_batch_host.
 * The caller keeps the arrays alive and unmodified until the call returns.
 */
int blp_solve_batch_gather(const double *const *A, const double *const *b, const double *const *c,
                           int64_t count, int32_t m, int32_t n,
                           const blp_limits *limits,
                           int8_t *status, double *objective, double *x,
                           int32_t *iters1, int32_t *iters2,
                           int32_t device);

/*
 * Batched hyper-rectangle LPs (the paper's Eq. 7 kernel; reference
 * boxlp.py:44-83 solve_box / solve_box_batch): maximise direction.x over
 * lower <= x <= upper for `count` boxes of dimension n, row-major [count][n].
 * value [count] (NaN if invalid), point [count][n] (zeros if invalid),
 * status [count]: 0 valid; -1 a non-finite bound ("box bounds must be
 * finite"); k+1 lower[k] > upper[k] at the first such k (boxlp.py:57-61).
 * _device: device pointers, async on cuda_stream; _host: host buffers, synchronous.
 */
int blp_box_solve_device(const double *lower, const double *upper, const double *direction,
                         int64_t count, int32_t n, double *value, double *point, int32_t *status,
                         void *cuda_stream);
int blp_box_solve_host(const double *lower, const double *upper, const double *direction,
                       int64_t count, int32_t n, double *value, double *point, int32_t *status,
                       int32_t device);

/*
 * Batched from-scratch optimality certificates (
 * replaces the reference's per-LP oracle.py:168-223 check_certificate).
 * For each LP k with status[k] == 0 (OPTIMAL), from A, b, c and the point
 * x [count][n] only: max_violation = max(0, max(A x - b)), max_negativity =
 * max(0, max(-x)), and max_reduced_cost = max(c_ext - [A|I]^T y) with y the
 * duals of a basis rebuilt greedily from the point's support (levels > tol
 * first, then the rest, index order, rank test at numpy's SVD threshold).
 * needs_prices[k] = 1 when max_reduced_cost > tol on a primal-feasible point:
 * the reference then looks for complementary-slackness prices with an
 * auxiliary LP (oracle.py:226-242), which the caller solves with
 * blp_solve_batch_* and applies through blp_certify_reprice_*.
 * Non-OPTIMAL LPs get NaN outputs and needs_prices 0.
 */
int blp_certify_batch_device(const double *A, const double *b, const double *c, const double *x,
                             int64_t count, int32_t m, int32_t n, int32_t shared_Ab,
                             const int8_t *status, double tol,
                             double *max_reduced_cost, double *max_violation, double *max_negativity,
                             int8_t *needs_prices, void *cuda_stream);
int blp_certify_batch_host(const double *A, const double *b, const double *c, const double *x,
                           int64_t count, int32_t m, int32_t n, int32_t shared_Ab,
                           const int8_t *status, double tol,
                           double *max_reduced_cost, double *max_violation, double *max_negativity,
                           int8_t *needs_prices, int32_t device);

/* max_reduced_cost[k] = max(c - A^T y_k, -y_k) for every k with mask[k] != 0
 * (y [count][m]: complementary prices; oracle.py:220-222). */
int blp_certify_reprice_device(const double *A, const double *c, const double *y, int64_t count,
                               int32_t m, int32_t n, int32_t shared_Ab, const int8_t *mask,
                               double *max_reduced_cost, void *cuda_stream);
int blp_certify_reprice_host(const double *A, const double *c, const double *y, int64_t count,
                             int32_t m, int32_t n, int32_t shared_Ab, const int8_t *mask,
                             double *max_reduced_cost, int32_t device);

/* Largest (m, n) the library accepts: 1 if supported, 0 otherwise. */
int blp_shape_supported(int32_t m, int32_t n);

/* Name of the kernel variant blp_solve_* would use for (m, n) (static string). */
const char *blp_kernel_variant(int32_t m, int32_t n);

/* The same for a batch in the given mode (shared_Ab = 1: support function, one A and b). */
const char *blp_kernel_variant_mode(int32_t m, int32_t n, int32_t shared_Ab);

/* Number of CUDA kernels this library has launched since load (monotonic). */
int64_t blp_launch_count(void);

/* Text of the last error on the calling thread ("" if none). */
const char *blp_last_error(void);

/* Measured shared-memory bandwidth of `device` in GB/s (LDS+STS bytes, all
 * SMs), the roofline denominator of the smem-resident kernels; < 0 on error. */
double blp_probe_smem_gbs(int32_t device);

/* Measured unfused FP64 rate of `device` in GFLOP/s (independent DMUL+DADD
 * chains: one flop each), the roofline denominator of the register-resident
 * kernels whose rank-1 update is exactly that instruction pair; < 0 on error. */
double blp_probe_fp64_gflops(int32_t device);

/* BLP_ABI_VERSION of the loaded library. */
int blp_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* BLP_H_ */
