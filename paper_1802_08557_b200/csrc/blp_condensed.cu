// blp_condensed.cu -- instances of the condensed-tableau warp-per-LP kernel
// (blp_condensed_kernel.cuh), in their own translation unit so they compile in
// parallel with the rest of the library.
#include "blp_condensed.h"

#include <cstdlib>

#include "blp_cmulti_kernel.cuh"
#include "blp_condensed_kernel.cuh"

namespace blp_condensed {

namespace {
struct Row { int rpl, ns; Instance inst; size_t stg_end; };
// kMinBlocks = resident LPs per SM the register budget is tuned for (C2, ctab_r1_s32:
// 16 -> 128 registers, 5.05 ms per 1e5; 14 -> 5.05; 18 -> 112 registers + spills, 6.39;
// 20 -> 96 registers + spills, 6.37 ms)
const Row kInstances[] = {
    {1, 8, {blp::condensed_kernel<1, 8, 24>, "ctab_r1_s8", blp::CtCfg<1, 8>::BYTES,
              blp::condensed_phase1_kernel<1, 8>, blp::CtP1<1, 8>::BYTES}, blp::CtCfg<1, 8>::STG_END},
    {1, 16, {blp::condensed_kernel<1, 16, 20>, "ctab_r1_s16", blp::CtCfg<1, 16>::BYTES,
              blp::condensed_phase1_kernel<1, 16>, blp::CtP1<1, 16>::BYTES}, blp::CtCfg<1, 16>::STG_END},
    {1, 32, {blp::condensed_kernel<1, 32, 16>, "ctab_r1_s32", blp::CtCfg<1, 32>::BYTES,
              blp::condensed_phase1_kernel<1, 32>, blp::CtP1<1, 32>::BYTES}, blp::CtCfg<1, 32>::STG_END},
    {1, 64, {blp::condensed_kernel<1, 64, 8>, "ctab_r1_s64", blp::CtCfg<1, 64>::BYTES,
              blp::condensed_phase1_kernel<1, 64>, blp::CtP1<1, 64>::BYTES}, blp::CtCfg<1, 64>::STG_END},
    {2, 8, {blp::condensed_kernel<2, 8, 12>, "ctab_r2_s8", blp::CtCfg<2, 8>::BYTES,
              blp::condensed_phase1_kernel<2, 8>, blp::CtP1<2, 8>::BYTES}, blp::CtCfg<2, 8>::STG_END},
    {2, 16, {blp::condensed_kernel<2, 16, 10>, "ctab_r2_s16", blp::CtCfg<2, 16>::BYTES,
              blp::condensed_phase1_kernel<2, 16>, blp::CtP1<2, 16>::BYTES}, blp::CtCfg<2, 16>::STG_END},
    {2, 32, {blp::condensed_kernel<2, 32, 8>, "ctab_r2_s32", blp::CtCfg<2, 32>::BYTES,
              blp::condensed_phase1_kernel<2, 32>, blp::CtP1<2, 32>::BYTES}, blp::CtCfg<2, 32>::STG_END},
    {4, 8, {blp::condensed_kernel<4, 8, 10>, "ctab_r4_s8", blp::CtCfg<4, 8>::BYTES,
              blp::condensed_phase1_kernel<4, 8>, blp::CtP1<4, 8>::BYTES}, blp::CtCfg<4, 8>::STG_END},
    {4, 16, {blp::condensed_kernel<4, 16, 8>, "ctab_r4_s16", blp::CtCfg<4, 16>::BYTES,
              blp::condensed_phase1_kernel<4, 16>, blp::CtP1<4, 16>::BYTES}, blp::CtCfg<4, 16>::STG_END},
};

// Multi-warp condensed form (blp_cmulti_kernel.cuh): NWR row-warps, R register slots and S
// tile slots per row, tile stride ST (odd, >= m), kMinBlocks LPs per SM.
struct MRow { int nwr, ns, r, st; Instance inst; };
#define CM_INST(NWR, R, S, ST, MB)                                                                     \
    {NWR, R + S, R, ST, {blp::cmulti_kernel<NWR, R, S, ST, MB>, "cm" #NWR "_r" #R "_s" #S,                  \
                  blp::CmCfg<NWR, R, S, ST>::BYTES, blp::cmulti_phase1_kernel<NWR, R, S, ST>,                \
                  blp::CmP1<NWR, R, S, ST>::BYTES, 32 * NWR}}
// First fit in this order.  C3 (100 x 100, c3 count 2e4, device-resident): r48_s56 at 3 LPs
// per SM 74.8 ms; r88_s16 (2 per SM) 88.0; r80_s24 89.5; r64_s40 94.7; r96_s32 107.7.
// C4 (64 x 32 support, 1e6): r16_s16 at 10 LPs per SM 38.4 ms; r32_s0 (8 per SM) 39.4;
// r24_s8 39.9; afiro 64 x 32 (1e5): 16.1 / 18.3 / 18.3 ms.
const MRow kMulti[] = {
    CM_INST(2, 16, 16, 65, 10),
    CM_INST(2, 64, 0, 65, 4),
    CM_INST(4, 32, 0, 129, 4),
    CM_INST(4, 48, 16, 129, 3),
    CM_INST(4, 48, 56, 129, 3),
    CM_INST(4, 96, 32, 129, 2),
    // 129..256 rows: eight row-warps (one thread per row), below the cluster kernel's reach
    CM_INST(8, 24, 40, 257, 2),
    CM_INST(8, 64, 64, 257, 1),
    CM_INST(8, 96, 104, 257, 1),
    // 257..512 rows, n <= 72: sixteen row-warps
    CM_INST(16, 24, 48, 513, 1),
    // A/B alternatives (BLP_CM_R selects the register width)
    CM_INST(4, 88, 16, 129, 2),
    CM_INST(4, 80, 24, 129, 2),
    CM_INST(4, 64, 40, 129, 2),
    CM_INST(2, 32, 0, 65, 8),
    CM_INST(2, 24, 8, 65, 10),
};
#undef CM_INST

int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return (v && *v) ? atoi(v) : dflt;
}

int rows_per_lane(int m) { return m <= 32 ? 1 : (m <= 64 ? 2 : (m <= 128 ? 4 : 0)); }
}  // namespace

bool select(int m, int n, Instance *out) {
    if (m < 1 || n < 1) return false;
    // BLP_CMULTI: 0 never, 1 for 65..128 rows and where the one-warp form has no instance,
    // 3 for every 33..128-row shape, 2 (default) as 3 except narrow LPs, which the one-warp
    // form (2 or 4 rows per lane) solves faster.  Measured (1e5 LPs, one-warp vs multi-warp
    // incl. its lazy pre-pass): afiro recipe (two-phase) 64 x 8 5.18 vs 8.93 ms, 128 x 8 16.0
    // vs 34.8, 64 x 16 10.9 vs 11.8, 100 x 16 36.3 vs 37.0, but 40 x 16 8.33 vs 8.06; the
    // reference's random LPs (single phase, few pivots) 64 x 8 0.40 vs 0.57, 64 x 16 0.69 vs
    // 0.80, but 128 x 16 1.75 vs 1.42 (the one-warp form has no lazy pre-pass); C4 64 x 32
    // (1e6 directions) ctab_r2_s32 42.0 vs cm2_r16_s16 37.1 ms.
    const int cm = env_int("BLP_CMULTI", 2);
    const bool narrow = n <= 8 || (n <= 16 && m > 48 && m <= 64);
    if (m > 32 && m <= 512 && cm != 0) {
        const int nwr = m <= 64 ? 2 : (m <= 128 ? 4 : (m <= 256 ? 8 : 16));
        const bool one_warp_fits = (m <= 64 && n <= 32) || (m > 64 && m <= 128 && n <= 16);
        const bool multi = !one_warp_fits || cm == 3 || (cm == 2 && !narrow) || (cm == 1 && m > 64);
        if (multi) {
            const int want_r = env_int("BLP_CM_R", 0);
            for (const MRow &r : kMulti) {
                if (r.nwr != nwr || n > r.ns || m > r.st) continue;
                if (want_r && r.r != want_r) continue;
                *out = r.inst;
                return true;
            }
        }
    }
    const int rpl = rows_per_lane(m);
    for (const Row &r : kInstances) {
        if (r.rpl != rpl || n > r.ns) continue;
        *out = r.inst;
        // BLP_CT_STAGE: grant the TMA staging buffer of the next LP's A -- 1 (default) for rows
        // of >= 32 doubles, 2 always, 0 never.  Measured (1e5 LPs, staged vs direct loads): C2
        // 28 x 32 4.945 vs 4.997 ms; afiro 20 x 10 (ctab_r1_s16) 1.409 vs 1.348; 64 x 16
        // (ctab_r2_s16) 11.05 vs 10.86 -- short rows make many small bulk copies per LP.
        const int stage = env_int("BLP_CT_STAGE", 1);
        if (stage == 2 || (stage == 1 && n >= 32)) out->smem = r.stg_end;
        return true;
    }
    return false;
}

}  // namespace blp_condensed
