// blp_cluster.h -- host side of the cluster-resident variant (blp_cluster.cu),
// called by the C ABI's planner/launcher in blp_capi.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

#include "blp_common.cuh"

namespace blp_cluster {

// Shape check without a device: some cluster size K <= 16 holds the tableau on
// chip (one row per thread, m <= threads; the per-CTA tile within 227 KB).
bool shape_fits(int m, int n);

// Kernel name as reported by blp_kernel_variant.
const char *variant_name(int m, int n);

// Launch the persistent cluster grid (K chosen from the occupancy calculator:
// the most SMs in use, then the smallest K).  K and the cluster count used are
// returned for diagnostics.
cudaError_t launch(const blp::Batch &B, cudaStream_t stream, int *K_used, int *clusters_used);

// The lazy-tableau kernel (blp_lazy_kernel.cuh) over the whole batch, then the
// cluster kernel over the LPs it deferred (phase 1 needed, or more than
// kLazyMaxPivots pivots); both stream-ordered, no host synchronisation.
cudaError_t launch_lazy_then_cluster(const blp::Batch &B, cudaStream_t stream);

// Whether the lazy path is used for this shape (BLP_LAZY=0 disables it).
bool lazy_enabled(int m, int n);

// The lazy kernel alone: on return *defer_list / *defer_count (device) name the
// LPs a dense kernel must still solve; *ws is the workspace to cudaFreeAsync
// after that dense launch.
cudaError_t launch_lazy(const blp::Batch &B, cudaStream_t stream, int **defer_list, int **defer_count, void **ws);

// After the dense launch: support-mode validation of the shared polytope, then
// the workspace is released (stream-ordered).
cudaError_t finish_lazy(const blp::Batch &B, cudaStream_t stream, void *ws);

// Kernels finish_lazy launches for this batch (support-mode validate + finalize, or the
// split mode's finalize), for blp_launch_count.
int finish_lazy_launches(const blp::Batch &B);

}  // namespace blp_cluster
