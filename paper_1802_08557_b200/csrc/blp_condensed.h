// blp_condensed.h -- host side of the condensed-tableau kernels (blp_condensed.cu):
// instance selection by shape, used by the C ABI's planner in blp_capi.cu.
#pragma once

#include <cstddef>

#include "blp_common.cuh"

namespace blp_condensed {

using KernelFn = void (*)(blp::Batch);
using Phase1Fn = void (*)(blp::Batch, double *);

struct Instance {
    KernelFn fn;
    const char *name;
    size_t smem;       // dynamic shared memory per CTA
    Phase1Fn phase1;   // support mode: the shared phase-1 prologue (one warp, same smem)
    size_t p1_bytes;   // its state + info block
    int threads = 32;  // one warp, or 32 x NWR for the multi-warp (cmulti) form
};

// The instance for m rows and n nonbasic slots, or false: one warp (lane L owns rows
// L + 32k) up to 32 rows, and for 33..128 rows either the one-warp form (rows per lane
// 2 or 4) or the multi-warp form (thread = row; BLP_CMULTI=0 disables it).
bool select(int m, int n, Instance *out);

}  // namespace blp_condensed
