// blp_condensed.h -- host side of the condensed-tableau kernels (blp_condensed.cu):
// instance selection by shape, used by the C ABI's planner in blp_capi.cu.
#pragma once

#include <cstddef>

#include "blp_common.cuh"

namespace blp_condensed {

using KernelFn = void (*)(blp::Batch);

struct Instance {
    KernelFn fn;
    const char *name;
    size_t smem;       // dynamic shared memory per CTA (one warp)
};

// The smallest instance holding m rows (lane L owns rows L + 32k) and n nonbasic
// slots, or false.
bool select(int m, int n, Instance *out);

}  // namespace blp_condensed
