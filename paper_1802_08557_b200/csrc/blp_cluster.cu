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

const char *variant_name(int m, int n) {
    (void)m; (void)n;
    return "cluster_r32";
}

cudaError_t launch(const blp::Batch &B, cudaStream_t stream, int *K_used, int *clusters_used) {
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
    long long clusters = std::min<long long>(bestC, B.count);
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bestS);
    if (e != cudaSuccess) return e;
    // workspace: the LP queue head + per cluster [2 parities][K CTAs][ld] published columns
    const blp::ClLayout L = blp::make_cl_layout(B.m, B.n, bestK, kRC);
    const size_t scratch = (size_t)clusters * 2 * bestK * L.ld * sizeof(double);
    void *ws = nullptr;
    e = cudaMallocAsync(&ws, 256 + scratch, stream);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(ws, 0, 256, stream);
    if (e != cudaSuccess) { cudaFreeAsync(ws, stream); return e; }
    blp::Batch Bl = B;
    Bl.next_lp = reinterpret_cast<int *>(ws);
    Bl.gtab = reinterpret_cast<double *>(reinterpret_cast<char *>(ws) + 256);
    Bl.gtab_stride = 0;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = bestK;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(clusters * bestK), 1, 1);
    cfg.blockDim = dim3(kNT, 1, 1);
    cfg.dynamicSmemBytes = bestS;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (env_int("BLP_VERBOSE", 0))
        fprintf(stderr, "blp cluster: m=%d n=%d K=%d clusters=%lld smem=%zu+%zu\n", B.m, B.n, bestK, clusters, bestS,
                sizeof(blp::ClStatic<kRC>));
    if (K_used) *K_used = bestK;
    if (clusters_used) *clusters_used = (int)clusters;
#ifdef BLP_CL_PROF
    {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbolAsync(blp::g_cl_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, stream);
    }
#endif
    e = cudaLaunchKernelEx(&cfg, fn, Bl);
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
    const cudaError_t ef = cudaFreeAsync(ws, stream);
    return e != cudaSuccess ? e : ef;
}

}  // namespace blp_cluster
