// blp_box_kernel.cuh -- batched hyper-rectangle LPs (the paper's Eq. 7 kernel,
// PAPER.md:272-285; reference boxlp.py:44-83): maximise d.x over
// lower <= x <= upper, coordinate-wise: x_i = lower_i where d_i < 0, else
// upper_i; value = sum_i d_i x_i.
//
// One thread per box; the row of each array a thread walks is contiguous and
// the warp's rows are adjacent, so every 128-byte line is fully consumed out
// of L1 over the n iterations.  Pure streaming: 3*8n bytes in, 8n+12 out.
//
// Validation mirrors boxlp.py:51-52,57-61: a box is valid iff every
// lower <= upper and lower + upper is finite; an invalid box reports
// status -1 when some bound is non-finite, else 1 + the first index with
// lower > upper (0 + 1 when none, as the reference's argmax of all-False).
#pragma once

#include "blp_common.cuh"

namespace blp {

struct BoxBatch {
    const double *lower, *upper, *dir;  // [count][n] row-major
    long long count;
    int n;
    double *value;                      // [count] (NaN when invalid)
    double *point;                      // [count][n] (zeros when invalid)
    int *status;                        // [count]
};

__global__ void __launch_bounds__(256) box_kernel(BoxBatch B) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < B.count; k += stride) {
        const size_t base = (size_t)k * B.n;
        const double *lo = B.lower + base, *hi = B.upper + base, *d = B.dir + base;
        double *p = B.point + base;
        bool valid = true, nonfinite = false;
        int first_gt = -1;
        double v = 0.0;
        for (int i = 0; i < B.n; ++i) {
            const double l = lo[i], h = hi[i], di = d[i];
            const bool ok = (l <= h) && isfinite(__dadd_rn(l, h));
            valid &= ok;
            nonfinite |= !isfinite(l) || !isfinite(h);
            if (first_gt < 0 && l > h) first_gt = i;
            const double xi = di < 0.0 ? l : h;       // np.where(direction < 0, lo, hi)
            p[i] = xi;
            v = __dadd_rn(v, __dmul_rn(di, xi));
        }
        if (!valid) {
            for (int i = 0; i < B.n; ++i) p[i] = 0.0;
            v = __longlong_as_double(0x7ff8000000000000LL);
        }
        B.value[k] = v;
        B.status[k] = valid ? 0 : (nonfinite ? -1 : 1 + (first_gt < 0 ? 0 : first_gt));
    }
}

}  // namespace blp
