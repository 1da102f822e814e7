// blp_condensed.cu -- instances of the condensed-tableau warp-per-LP kernel
// (blp_condensed_kernel.cuh), in their own translation unit so they compile in
// parallel with the rest of the library.
#include "blp_condensed.h"

#include <cstdlib>

#include "blp_condensed_kernel.cuh"

namespace blp_condensed {

namespace {
struct Row { int rpl, ns; Instance inst; };
// kMinBlocks = resident LPs per SM the register budget is tuned for (C2, ctab_r1_s32:
// 16 -> 128 registers, 5.05 ms per 1e5; 20 -> 96 registers + spills, 6.37 ms)
const Row kInstances[] = {
    {1, 8, {blp::condensed_kernel<1, 8, 24>, "ctab_r1_s8", blp::CtCfg<1, 8>::BYTES}},
    {1, 16, {blp::condensed_kernel<1, 16, 20>, "ctab_r1_s16", blp::CtCfg<1, 16>::BYTES}},
    {1, 32, {blp::condensed_kernel<1, 32, 16>, "ctab_r1_s32", blp::CtCfg<1, 32>::BYTES}},
    {1, 64, {blp::condensed_kernel<1, 64, 8>, "ctab_r1_s64", blp::CtCfg<1, 64>::BYTES}},
    {2, 8, {blp::condensed_kernel<2, 8, 12>, "ctab_r2_s8", blp::CtCfg<2, 8>::BYTES}},
    {2, 16, {blp::condensed_kernel<2, 16, 10>, "ctab_r2_s16", blp::CtCfg<2, 16>::BYTES}},
    {2, 32, {blp::condensed_kernel<2, 32, 8>, "ctab_r2_s32", blp::CtCfg<2, 32>::BYTES}},
    {4, 8, {blp::condensed_kernel<4, 8, 10>, "ctab_r4_s8", blp::CtCfg<4, 8>::BYTES}},
    {4, 16, {blp::condensed_kernel<4, 16, 8>, "ctab_r4_s16", blp::CtCfg<4, 16>::BYTES}},
};

int rows_per_lane(int m) { return m <= 32 ? 1 : (m <= 64 ? 2 : (m <= 128 ? 4 : 0)); }
}  // namespace

bool select(int m, int n, Instance *out) {
    if (m < 1 || n < 1) return false;
    const int rpl = rows_per_lane(m);
    for (const Row &r : kInstances) {
        if (r.rpl != rpl || n > r.ns) continue;
        *out = r.inst;
        return true;
    }
    return false;
}

}  // namespace blp_condensed
