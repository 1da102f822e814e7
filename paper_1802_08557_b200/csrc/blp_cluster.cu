// blp_cluster.cu -- launcher of the cluster-resident simplex (blp_cluster_kernel.cuh).
//
// A separate translation unit: the cluster kernel is large and compiles in
// parallel with blp_capi.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "blp_cluster.h"
#include "blp_cluster_kernel.cuh"
#include "blp_lazy_kernel.cuh"

namespace blp_cluster {
namespace {

constexpr size_t kMaxDynSmem = 227 * 1024;
constexpr int kRC = 32;       // register columns per row
constexpr int kNT = 512;      // one row per thread: m <= 512

using KernelFn = void (*)(blp::Batch);

KernelFn kernel_fn() { return blp::cluster_kernel<kRC, kNT>; }

int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return (v && *v) ? atoi(v) : dflt;
}

// Per-CTA shared memory for cluster size K, or 0 if K cannot hold the shape.
size_t smem_for(int m, int n, int K) {
    if (m < 1 || m > kNT || K < 1 || K > blp::kClMaxK) return 0;
    const blp::ClLayout L = blp::make_cl_layout(m, n, K, kRC);
    if (L.cpc + 1 > kNT || L.cpc > blp::kClMaxCols) return 0;     // column threads + the objective thread
    if ((size_t)(L.sc4 + blp::kClSG) * L.ld < (size_t)n) return 0;  // x staging reuses the tile
    if (L.bytes + sizeof(blp::ClStatic<kRC>) > kMaxDynSmem) return 0;
    return L.bytes;
}

}  // namespace

bool shape_fits(int m, int n) {
    for (int K = 2; K <= blp::kClMaxK; ++K)
        if (smem_for(m, n, K)) return true;
    return false;
}

bool lazy_enabled(int m, int n) {
    return env_int("BLP_LAZY", 1) != 0 && blp::lazy_smem_bytes(m, n, 0, 512, 1) <= kMaxDynSmem;
}

const char *variant_name(int m, int n) {
    return lazy_enabled(m, n) ? "lazy+cluster_r32" : "cluster_r32";
}

namespace {
// A prepared cluster launch: the configuration (cluster size K from the occupancy calculator)
// and its workspace, allocated and cleared on the stream (cluster_prepare) ahead of the
// launch itself (cluster_fire), so that a programmatic dependent launch can follow the lazy
// kernel directly.
struct ClusterLaunch {
    int K = 0;
    long long clusters = 0;
    size_t smem = 0;
    void *ws = nullptr;
};

cudaError_t cluster_prepare(const blp::Batch &B, cudaStream_t stream, ClusterLaunch *CL) {
    KernelFn fn = kernel_fn();
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    const int forced = env_int("BLP_CLUSTER_K", 0);
    int bestK = 0, bestC = 0;
    size_t bestS = 0;
    for (int K = 2; K <= blp::kClMaxK; ++K) {
        if (forced && K != forced) continue;
        const size_t s = smem_for(B.m, B.n, K);
        if (!s) continue;
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s);
        if (e != cudaSuccess) return e;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = K;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(K, 1, 1);
        cfg.blockDim = dim3(kNT, 1, 1);
        cfg.dynamicSmemBytes = s;
        cfg.stream = stream;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, fn, &cfg) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if (nc * K > bestC * bestK) { bestK = K; bestC = nc; bestS = s; }
    }
    if (!bestK) return cudaErrorInvalidConfiguration;
    CL->K = bestK;
    CL->clusters = std::min<long long>(bestC, B.count);
    CL->smem = bestS;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bestS);
    if (e != cudaSuccess) return e;
    // workspace: the LP queue head + per cluster [2 parities][K CTAs][ld] published columns
    const blp::ClLayout L = blp::make_cl_layout(B.m, B.n, bestK, kRC);
    const size_t scratch = (size_t)CL->clusters * 2 * bestK * L.ld * sizeof(double);
    e = cudaMallocAsync(&CL->ws, 256 + scratch, stream);
    if (e != cudaSuccess) { CL->ws = nullptr; return e; }
    e = cudaMemsetAsync(CL->ws, 0, 256, stream);
    if (e != cudaSuccess) { cudaFreeAsync(CL->ws, stream); CL->ws = nullptr; }
    return e;
}

// pdl: a programmatic dependent launch after the lazy kernel (which triggers its dependents
// at its start): the cluster grid is scheduled onto SMs as the lazy kernel's CTAs retire and
// waits in griddepcontrol.wait for its completion, so the launch of a dense pass that is
// often empty (C5: no LP deferred) overlaps the lazy kernel's tail instead of following it.
// Measured neutral (C5 1e4: 5.331 / 5.328 ms vs 5.332 / 5.330 with BLP_PDL=0; random 300 x
// 300: 1.397 / 1.388 vs 1.397 / 1.392): the empty launch was already off the critical path.
cudaError_t cluster_fire(const blp::Batch &B, const ClusterLaunch &CL, cudaStream_t stream, bool pdl) {
    KernelFn fn = kernel_fn();
    blp::Batch Bl = B;
    Bl.next_lp = reinterpret_cast<int *>(CL.ws);
    Bl.gtab = reinterpret_cast<double *>(reinterpret_cast<char *>(CL.ws) + 256);
    Bl.gtab_stride = 0;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL.K;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3((unsigned)(CL.clusters * CL.K), 1, 1);
    cfg.blockDim = dim3(kNT, 1, 1);
    cfg.dynamicSmemBytes = CL.smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 2 : 1;
    if (env_int("BLP_VERBOSE", 0))
        fprintf(stderr, "blp cluster: m=%d n=%d K=%d clusters=%lld smem=%zu+%zu pdl=%d\n", B.m, B.n, CL.K, CL.clusters,
                CL.smem, sizeof(blp::ClStatic<kRC>), pdl ? 1 : 0);
#ifdef BLP_CL_PROF
    {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbolAsync(blp::g_cl_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, stream);
    }
#endif
    cudaError_t e = cudaLaunchKernelEx(&cfg, fn, Bl);
#ifdef BLP_CL_PROF
    {
        unsigned long long h[16];
        cudaMemcpyFromSymbolAsync(h, blp::g_cl_prof, sizeof(h), 0, cudaMemcpyDeviceToHost, stream);
        cudaStreamSynchronize(stream);
        const char *names[16] = {"claim", "build", "phase-setup", "wait", "select", "pivot-S3", "publish",
                                 "extract", "update", "lp-end", "b:head", "b:regs", "b:tile", "b:init", "b:barrier", ""};
        double tot = 0;
        for (int k = 0; k < 16; ++k) tot += (double)h[k];
        fprintf(stderr, "blp cluster prof (thread 0 of each CTA, %% of cycles):");
        for (int k = 0; k < 15; ++k) fprintf(stderr, " %s=%.1f", names[k], 100.0 * h[k] / tot);
        fprintf(stderr, "  total Gcyc=%.3f\n", tot / 1e9);
    }
#endif
    const cudaError_t ef = cudaFreeAsync(CL.ws, stream);
    return e != cudaSuccess ? e : ef;
}


}  // namespace

cudaError_t launch(const blp::Batch &B, cudaStream_t stream, int *K_used, int *clusters_used) {
    ClusterLaunch CL;
    const cudaError_t e = cluster_prepare(B, stream, &CL);
    if (e != cudaSuccess) return e;
    if (K_used) *K_used = CL.K;
    if (clusters_used) *clusters_used = (int)CL.clusters;
    return cluster_fire(B, CL, stream, false);
}

static int lazy_ws_mode(const blp::Batch &B, int nt) {
    return (nt == 512 && !B.shared_Ab && env_int("BLP_LAZY_WS", 0)) ? 1 : 0;
}

static int lazy_nt(const blp::Batch &B) {
    const int dflt = B.shared_Ab ? (B.m <= 64 ? 32 : 64) : (B.m <= 64 ? 64 : (B.m <= 128 ? 128 : 512));
    return env_int("BLP_LAZY_NT", dflt);
}

// BLP_LAZY_SPLIT=1 (opt-in, parity-tested): validation of A as its own work queue
// (independent LPs, non-WS form; blp_lazy_kernel.cuh), made BLP_STATUS_INVALID by
// lazy_finalize_kernel afterwards.  Measured slower: C5 1e4 5.54 ms vs 5.12 inline, random
// 100 x 100 2e4 0.91 vs 0.86 -- a solve is a chain of ~5 us pivots, so the CTAs that solve
// while the others stream are too few; inline, every CTA overlaps its neighbour's stream.
// BLP_LAZY_SPLIT=2 (every CTA solves first, validation after all solves, so no stream passes
// through L2 while the replay history is live): 6.09 vs 5.21 ms -- the solves alone take
// ~3 ms, latency-bound (~6 us per pivot: A and history round trips), with nothing to overlap.
static bool lazy_split(const blp::Batch &B) {
    return !B.shared_Ab && (long long)B.m * B.n > 0 && !lazy_ws_mode(B, lazy_nt(B)) &&
           env_int("BLP_LAZY_SPLIT", 0) != 0;
}

cudaError_t launch_lazy(const blp::Batch &B, cudaStream_t stream, int **defer_list, int **defer_count, void **ws_out) {
    using LazyFn = void (*)(blp::Batch);
    // BLP_LAZY_NT: threads per CTA (resident CTAs per SM follow from the register budget).
    // C5 1e4: 256 -> 6.73 ms, 512 -> 6.96, 128 -> 7.71; random 100 x 100, 2e4: 128 -> 0.95,
    // 256 -> 1.21, 64 -> 0.99; 64 x 64: 64 -> 0.42, 128 -> 0.51, 32 -> 0.48; support mode (no
    // per-LP scan of A) C4 1e6: 32 -> 65.4 ms, 64 -> 70.7, 128 -> 81.5 (dense pairlp: 77.3)
    // (after the unrolled validation scan, C5: 512 -> 5.43 ms, 256 -> 5.75)
    const int nt = lazy_nt(B);
    // BLP_LAZY_WS=1: the warp-specialised bulk-copy validation stream (measured slower on
    // C5: 6.7 vs 6.0 ms -- the solve, not the stream, bounds an LP); the staged replay
    // (RP=1) only for the shared polytope (C4 1e6: 60.2 vs 65.0 ms; C5 5.87 vs 5.43,
    // random 100 x 100 0.98 vs 0.83)
    const int ws_mode = lazy_ws_mode(B, nt);
    const int rp = env_int("BLP_LAZY_RP", B.shared_Ab ? 1 : 0) ? 1 : 0;
    LazyFn fn;
    if (ws_mode) fn = rp ? (LazyFn)blp::lazy_kernel<512, 2, 1, 1> : (LazyFn)blp::lazy_kernel<512, 2, 1, 0>;
    else if (rp)
        fn = nt == 512 ? (LazyFn)blp::lazy_kernel<512, 2, 0, 1>
           : nt == 128 ? (LazyFn)blp::lazy_kernel<128, 8, 0, 1>
           : nt == 64  ? (LazyFn)blp::lazy_kernel<64, 16, 0, 1>
           : nt == 32  ? (LazyFn)blp::lazy_kernel<32, 32, 0, 1>
                       : (LazyFn)blp::lazy_kernel<256, 4, 0, 1>;
    else if (B.m >= blp::kLazyMaxPivots && env_int("BLP_LAZY_SPARSE", 0))
        // BLP_LAZY_SPARSE=1: slack columns of rows never pivoted on are exact unit columns,
        // skipped (SPX; measured slower: C5 5.61 vs 5.34 ms -- blp_lazy_kernel.cuh)
        fn = nt == 512 ? (LazyFn)blp::lazy_kernel<512, 2, 0, 0, 0, 1>
           : nt == 128 ? (LazyFn)blp::lazy_kernel<128, 8, 0, 0, 0, 1>
           : nt == 64  ? (LazyFn)blp::lazy_kernel<64, 16, 0, 0, 0, 1>
           : nt == 32  ? (LazyFn)blp::lazy_kernel<32, 32, 0, 0, 0, 1>
                       : (LazyFn)blp::lazy_kernel<256, 4, 0, 0, 0, 1>;
    else
        fn = nt == 512 ? (LazyFn)blp::lazy_kernel<512, 2, 0, 0>
           : nt == 128 ? (LazyFn)blp::lazy_kernel<128, 8, 0, 0>
           : nt == 64  ? (LazyFn)blp::lazy_kernel<64, 16, 0, 0>
           : nt == 32  ? (LazyFn)blp::lazy_kernel<32, 32, 0, 0>
                       : (LazyFn)blp::lazy_kernel<256, 4, 0, 0>;
    const int threads = (nt == 512 || nt == 128 || nt == 64 || nt == 32) ? nt : 256;
    size_t smem = blp::lazy_smem_bytes(B.m, B.n, ws_mode, threads, rp);
    // BLP_LAZY_FSMEM=1: f^t history of the first pivots in shared memory (two CTAs per SM kept)
    // (value > 1: per-CTA shared-memory cap in KB; 1: 113 KB)
    // BLP_LAZY_RSMEM=1: the r^t history of those pivots too (same cap semantics).  Measured
    // (C5 1e4, parity-checked): default 5.39 ms; FSMEM=1 8.04; RSMEM=1 8.26, =100 6.14, =80
    // 5.94 -- the history bytes taken off L2 cost L1 capacity (the entering column's strided
    // reads of A hit there) and residency, so both stay opt-in.
    const int fsmem = env_int("BLP_LAZY_FSMEM", 0), rsmem = env_int("BLP_LAZY_RSMEM", 0);
    if (nt == 512 && !ws_mode && !rp && (fsmem || rsmem)) {
        const int capk = rsmem > 1 ? rsmem : fsmem > 1 ? fsmem : 113;
        const size_t base = (smem + 15) / 16 * 16, cap = (size_t)capk * 1024;
        const size_t per = 8 * (size_t)std::max(1, B.m) + (rsmem ? 8 * (size_t)(B.n + B.m) : 0);
        const size_t kf = base < cap ? std::min<size_t>(blp::kLazyMaxPivots, (cap - base) / per) : 0;
        if (kf >= (rsmem ? 2u : 4u)) {
            fn = rsmem ? (LazyFn)blp::lazy_kernel<512, 2, 0, 0, 2> : (LazyFn)blp::lazy_kernel<512, 2, 0, 0, 1>;
            smem = base + kf * per;
        }
    }
    *ws_out = nullptr;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // BLP_LAZY_CARVEOUT: shared-memory share of the L1/shared array in percent (-1: driver's choice)
    const int carve = env_int("BLP_LAZY_CARVEOUT", -1);
    if (carve >= 0 && (e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve)) != cudaSuccess)
        return e;
    int dev = 0, sms = 0, occ = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem)) != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    // BLP_LAZY_PER_SM: cap on resident CTAs per SM (the replay history of all resident CTAs vs L2)
    const int per_sm = std::max(1, std::min(occ, env_int("BLP_LAZY_PER_SM", occ)));
    const long long grid = std::min<long long>((long long)per_sm * sms, B.count);
    const long long stride = blp::lazy_scratch_doubles(B.m, B.n);
    // workspace: [0] LP queue, [64] deferred count | defer list | invalid flags | per-CTA replay history
    const size_t list_bytes = ((size_t)B.count * sizeof(int) + 255) / 256 * 256;
    const size_t flag_bytes = ((size_t)B.count + 255) / 256 * 256;
    char *ws = nullptr;
    e = cudaMallocAsync(reinterpret_cast<void **>(&ws), 256 + list_bytes + flag_bytes + (size_t)grid * stride * sizeof(double),
                        stream);
    if (e != cudaSuccess) return e;
    *ws_out = ws;
    unsigned char *flags = reinterpret_cast<unsigned char *>(ws + 256 + list_bytes);
    e = cudaMemsetAsync(ws, 0, 256, stream);
    blp::Batch Bl = B;
    Bl.next_lp = reinterpret_cast<int *>(ws);
    Bl.defer_count = reinterpret_cast<int *>(ws + 64);
    Bl.defer_list = reinterpret_cast<int *>(ws + 256);
    Bl.gtab = reinterpret_cast<double *>(ws + 256 + list_bytes + flag_bytes);
    Bl.gtab_stride = stride;
    const bool split = lazy_split(B);
    Bl.vq = split ? reinterpret_cast<int *>(ws + 128) : nullptr;
    Bl.vflag = split ? flags : nullptr;
    // BLP_LAZY_SPLIT=1: half the CTAs validate first; 2: every CTA solves first (the solves then
    // run while no validation stream passes through L2, the validation after them)
    Bl.vfirst = env_int("BLP_LAZY_SPLIT", 0) == 2 ? 0 : (int)(grid / 2);
    // BLP_LAZY_DISCARD (default: history rows of >= 8 KB): discard a solved LP's replay history
    // from L2 (no write-back of dead lines).  Measured: C5 1e4 5.187 / 5.187 ms vs 5.286 / 5.295,
    // DRAM 28.30 vs 29.51 GB per launch; random 300 x 300 (7.2 KB rows) 1.375 vs 1.372; random
    // 100 x 100 (2.4 KB rows) 0.884 / 0.880 vs 0.871 / 0.867 -- short LPs pay the discards.
    Bl.lazy_discard = env_int("BLP_LAZY_DISCARD", (2 * B.m + B.n) * 8 >= 8192 ? 1 : 0);
    if (split && e == cudaSuccess) e = cudaMemsetAsync(flags, 0, flag_bytes, stream);
    *defer_list = Bl.defer_list;
    *defer_count = Bl.defer_count;
    if (e == cudaSuccess) {
        // BLP_LAZY_PERSIST (pivots; default 0 = off): the first pivots' replay history of every
        // resident CTA -- one contiguous range in the pivot-major layout -- is marked persisting
        // in L2 against the validation stream of A.  Measured within noise (C5 5.19 vs 5.22 ms
        // alternating in one process; ncu: the same L2 read misses with and without), and it
        // raises the device-wide persisting-L2 limit, so it is opt-in.
        const int kp = B.shared_Ab ? 0 : env_int("BLP_LAZY_PERSIST", 0);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3((unsigned)threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cfg.numAttrs = 0;
        if (kp > 0) {
            int maxwin = 0, maxpers = 0;
            cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, dev);
            cudaDeviceGetAttribute(&maxpers, cudaDevAttrMaxPersistingL2CacheSize, dev);
            size_t want = (size_t)std::min(kp, blp::kLazyMaxPivots) * (size_t)grid * (size_t)(2 * B.m + B.n) * 8;
            want = std::min(want, (size_t)std::max(0, std::min(maxwin, maxpers)));
            if (want > 0) {
                size_t cur = 0;
                cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
                if (cur < want) {
                    const cudaError_t le = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
                    if (le != cudaSuccess) cudaGetLastError();   // not fatal: the window is a hint
                    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
                }
                if (env_int("BLP_VERBOSE", 0))
                    fprintf(stderr, "blp lazy: persisting window %zu B (limit %zu B, max %d)\n", want, cur, maxpers);
                attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
                attr[0].val.accessPolicyWindow.base_ptr = Bl.gtab;
                attr[0].val.accessPolicyWindow.num_bytes = want;
                attr[0].val.accessPolicyWindow.hitRatio = 1.0f;
                attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
                attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
            }
        }
        e = cudaLaunchKernelEx(&cfg, fn, Bl);
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    if (env_int("BLP_VERBOSE", 0))
        fprintf(stderr, "blp lazy: m=%d n=%d grid=%lld x %d (%d per SM, ws=%d rp=%d) smem=%zu scratch=%.1f MB\n", B.m, B.n,
                grid, threads, occ, ws_mode, rp, smem, grid * stride * 8.0 / 1e6);
    if (e == cudaSuccess && B.shared_Ab && (long long)B.m * B.n > 0) {
        // support mode: the shared polytope is validated once by finish_lazy, after the
        // dense launch (its flags start cleared here)
        e = cudaMemsetAsync(flags, 0, flag_bytes, stream);
    }
    return e;
}

// Support mode only: after the dense kernel, mark every LP invalid if the shared
// polytope holds a non-finite entry (the lazy kernel does not scan A then).
static cudaError_t launch_lazy_finalize(const blp::Batch &B, cudaStream_t stream, void *ws) {
    const bool split = lazy_split(B);
    if (!split && (!B.shared_Ab || (long long)B.m * B.n == 0)) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t list_bytes = ((size_t)B.count * sizeof(int) + 255) / 256 * 256;
    unsigned char *flags = reinterpret_cast<unsigned char *>(static_cast<char *>(ws) + 256 + list_bytes);
    // support mode: the shared polytope is validated here; split mode: the lazy kernel's
    // validation queue already set the flags
    if (!split) blp::lazy_validate_kernel<<<1, 256, 0, stream>>>(B.A, B.count, (long long)B.m * B.n, 1, flags);
    blp::lazy_finalize_kernel<<<(unsigned)std::max<long long>(1, std::min<long long>((B.count + 255) / 256, 4LL * sms)),
                                256, 0, stream>>>(flags, B);
    return cudaGetLastError();
}

int finish_lazy_launches(const blp::Batch &B) {
    if (lazy_split(B)) return 1;
    return (B.shared_Ab && (long long)B.m * B.n > 0) ? 2 : 0;
}

cudaError_t finish_lazy(const blp::Batch &B, cudaStream_t stream, void *ws) {
    cudaError_t e = launch_lazy_finalize(B, stream, ws);
    const cudaError_t ef = ws ? cudaFreeAsync(ws, stream) : cudaSuccess;
    return e != cudaSuccess ? e : ef;
}

cudaError_t launch_lazy_then_cluster(const blp::Batch &B, cudaStream_t stream) {
    int *dl = nullptr, *dc = nullptr;
    void *ws = nullptr;
    // the dense pass is prepared (workspace cleared) before the lazy kernel so that it can
    // follow it as a programmatic dependent launch (BLP_PDL=0: a plain stream-ordered launch;
    // support mode clears its flags after the lazy kernel, so it launches plainly)
    ClusterLaunch CL;
    cudaError_t e = cluster_prepare(B, stream, &CL);
    if (e == cudaSuccess) e = launch_lazy(B, stream, &dl, &dc, &ws);
    if (e == cudaSuccess) {
        blp::Batch Bc = B;                       // the dense kernel solves the deferred LPs
        Bc.defer_list = dl;
        Bc.defer_count = dc;
        const bool pdl = !B.shared_Ab && env_int("BLP_PDL", 1) != 0;
#ifndef BLP_AB_NODENSE   // A/B builds only: the cost of the (possibly empty) dense launch
        e = cluster_fire(Bc, CL, stream, pdl);
#else
        cudaFreeAsync(CL.ws, stream);
#endif
    } else if (CL.ws) {
        cudaFreeAsync(CL.ws, stream);
    }
    const cudaError_t ef = finish_lazy(B, stream, ws);
    return e != cudaSuccess ? e : ef;
}

}  // namespace blp_cluster
