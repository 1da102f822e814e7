// blp_capi.cu -- C ABI of libblp.so (declared in include/blp.h).
//
// Host runtime around the simplex kernels: variant selection by LP shape,
// persistent-grid sizing from the occupancy calculator, stream-ordered
// workspace, and the host-buffer path that pipelines sub-batches over
// several streams so H2D / kernel / D2H overlap (the paper's multi-stream
// scheme, on B200's independent copy engines).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/blp.h"
#include "blp_common.cuh"
#include "blp_regtile_kernel.cuh"
#include "blp_warplp_kernel.cuh"
#include "blp_warplp2_kernel.cuh"
#include "blp_condensed.h"
#include "blp_pairlp_kernel.cuh"
#include "blp_tableau_kernel.cuh"
#include "blp_box_kernel.cuh"
#include "blp_cert_kernel.cuh"
#include "blp_cluster.h"

namespace {

thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};

int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

#define BLP_CUDA_TRY(expr)                                                              \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            return fail(BLP_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

constexpr size_t kMaxDynSmem = 227 * 1024;

using KernelFn = void (*)(blp::Batch);

// One launch configuration: kernel variant, CTA size, dynamic smem, HBM tableau slot.
struct Plan {
    KernelFn fn = nullptr;
    const char *name = "unsupported";
    int threads = 0;
    size_t smem = 0;
    long long slot = 0;  // doubles of global tableau per CTA (HBM-streamed variant)
    bool lazy = false;     // the exact lazy-tableau kernel runs first; this one takes its deferred LPs
    bool cluster = false;  // cluster-resident variant (blp_cluster.cu): launched by blp_cluster::launch
    blp_condensed::Phase1Fn phase1 = nullptr;   // condensed: shared phase-1 prologue (support mode)
    size_t p1_bytes = 0;
};

int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return (v && *v) ? atoi(v) : dflt;
}

// Register-tile variant for m <= 64: columns per warp CPW (BLP_RT_CPW overrides).
bool plan_regtile(int m, int n, Plan *p) {
    const int ncols = n + m + 1;
    const int rpl = m <= 32 ? 1 : (m <= 64 ? 2 : 0);
    if (rpl == 0) return false;
    int cpw = env_int("BLP_RT_CPW", rpl == 1 ? 32 : 16);
    struct Inst { int rpl, cpw, maxt; KernelFn fn; const char *name; };
    static const Inst insts[] = {
        {1, 16, 128, blp::regtile_kernel<1, 16, 128, 4>, "regtile_r1_c16"},
        {1, 32, 64, blp::regtile_kernel<1, 32, 64, 8>, "regtile_r1_c32"},
        {2, 16, 256, blp::regtile_kernel<2, 16, 256, 2>, "regtile_r2_c16"},
        {2, 32, 128, blp::regtile_kernel<2, 32, 128, 2>, "regtile_r2_c32"},
    };
    for (int attempt = 0; attempt < 2; ++attempt) {
        for (const Inst &I : insts) {
            if (I.rpl != rpl || I.cpw != cpw) continue;
            const int nw = (ncols + I.cpw - 1) / I.cpw;
            if (nw * 32 > I.maxt) break;
            const blp::RtLayout L = blp::make_rt_layout(I.rpl, I.cpw, nw);
            if (L.bytes > kMaxDynSmem) break;
            p->fn = I.fn; p->name = I.name; p->threads = nw * 32; p->smem = L.bytes; p->slot = 0;
            return true;
        }
        cpw = rpl == 1 ? 64 : 32;  // wider tiles for wide LPs
    }
    return false;
}

// Shared-memory (or HBM) tableau variant; rows per lane RPL = ceil((m+1)/32).
bool plan_tableau(int m, int n, Plan *p) {
    const int rpl = (m + 1 + 31) / 32;
    const blp::TabLayout Ls = blp::make_tab_layout(m, n, 32, true);
    bool smem_tab = Ls.bytes <= kMaxDynSmem && rpl <= 4 && env_int("BLP_FORCE_HBM", 0) == 0;
    int maxt = 1024;
    if (smem_tab) {
        switch (rpl) {
            case 1: p->fn = blp::tableau_kernel<1, true, 1024>; p->name = "smem_rpl1"; break;
            case 2: p->fn = blp::tableau_kernel<2, true, 1024>; p->name = "smem_rpl2"; break;
            case 3: p->fn = blp::tableau_kernel<3, true, 1024>; p->name = "smem_rpl3"; break;
            default: p->fn = blp::tableau_kernel<4, true, 1024>; p->name = "smem_rpl4"; break;
        }
    } else if (rpl <= 1) { p->fn = blp::tableau_kernel<1, false, 1024>; p->name = "hbm_rpl1"; }
    else if (rpl <= 2) { p->fn = blp::tableau_kernel<2, false, 1024>; p->name = "hbm_rpl2"; }
    else if (rpl <= 4) { p->fn = blp::tableau_kernel<4, false, 1024>; p->name = "hbm_rpl4"; }
    else if (rpl <= 8) { p->fn = blp::tableau_kernel<8, false, 512>; p->name = "hbm_rpl8"; maxt = 512; }
    else if (rpl <= 16) { p->fn = blp::tableau_kernel<16, false, 512>; p->name = "hbm_rpl16"; maxt = 512; }
    else if (rpl <= 32) { p->fn = blp::tableau_kernel<32, false, 256>; p->name = "hbm_rpl32"; maxt = 256; }
    else return false;
    // threads: resident CTAs of one SM hold ~32 warps (register budget ~64/thread),
    // never more warps than columns
    const int ncols = n + m + 1;
    int ctas = smem_tab ? (int)std::max<size_t>(1, (228 * 1024) / (Ls.bytes + 1024)) : 2;
    ctas = std::min(ctas, 16);
    int warps = std::max(2, std::min(16, 32 / ctas));   // C3 (1 CTA/SM): 16 beats 8 and 32
    warps = std::min(warps, std::max(1, (ncols + 1) / 2));
    warps = std::min(env_int("BLP_TAB_WARPS", warps), maxt / 32);
    p->threads = std::max(1, warps) * 32;
    const blp::TabLayout L = blp::make_tab_layout(m, n, p->threads / 32, smem_tab);
    p->smem = L.bytes;
    p->slot = smem_tab ? 0 : (long long)L.ncols * L.ld;
    return true;
}

// Warp-per-LP register variant: m <= 32 rows, n + m + 1 <= 64 columns.
bool plan_warplp(int m, int n, Plan *p) {
    const int ncols = n + m + 1;
    if (m > 32) return false;
    if (ncols <= 32) {
        p->fn = blp::warplp_kernel<32, 16>; p->name = "warplp_c32"; p->smem = blp::WlpCfg<32>::bytes(m);
    } else if (ncols <= 62 && env_int("BLP_WLP2", 38) > 0) {
        // register/smem split row (blp_warplp2_kernel.cuh); BLP_WLP2 = register columns
        // (C2 1e5: r38/s24 @16 LPs/SM 8.9 ms, r46/s16 9.8, r30/s32 10.1, all-register c62 10.3)
        switch (env_int("BLP_WLP2", 38)) {
            case 30: p->fn = blp::warplp2_kernel<30, 32, 18>; p->name = "warplp2_r30_s32";
                     p->smem = blp::Wl2Cfg<30, 32>::BYTES; break;
            case 34: p->fn = blp::warplp2_kernel<34, 28, 17>; p->name = "warplp2_r34_s28";
                     p->smem = blp::Wl2Cfg<34, 28>::BYTES; break;
            case 42: p->fn = blp::warplp2_kernel<42, 20, 15>; p->name = "warplp2_r42_s20";
                     p->smem = blp::Wl2Cfg<42, 20>::BYTES; break;
            case 46: p->fn = blp::warplp2_kernel<46, 16, 14>; p->name = "warplp2_r46_s16";
                     p->smem = blp::Wl2Cfg<46, 16>::BYTES; break;
            default: p->fn = blp::warplp2_kernel<38, 24, 16>; p->name = "warplp2_r38_s24";
                     p->smem = blp::Wl2Cfg<38, 24>::BYTES; break;
        }
    } else if (ncols <= 62) {
        p->fn = blp::warplp_kernel<62, 12>; p->name = "warplp_c62"; p->smem = blp::WlpCfg<62>::bytes(m);
    } else if (ncols <= 64) {
        // BLP_WLP_MINB trades registers (= ILP) against resident LPs per SM
        switch (env_int("BLP_WLP_MINB", 12)) {
            case 8: p->fn = blp::warplp_kernel<64, 8>; p->name = "warplp_c64_b8"; break;
            case 10: p->fn = blp::warplp_kernel<64, 10>; p->name = "warplp_c64_b10"; break;
            default: p->fn = blp::warplp_kernel<64, 12>; p->name = "warplp_c64"; break;
        }
        p->smem = blp::WlpCfg<64>::bytes(m);
    } else {
        return false;
    }
    p->threads = 32;
    p->slot = 0;
    return true;
}

// Condensed-tableau warp-per-LP variants (blp_condensed_kernel.cuh): only the n nonbasic
// columns + rhs of each row are stored and updated; lane L holds rows L + 32k (k < RPL).
// BLP_CONDENSED=0 disables the family.
bool plan_condensed(int m, int n, Plan *p) {
    if (env_int("BLP_CONDENSED", 1) == 0) return false;
    blp_condensed::Instance I;
    if (!blp_condensed::select(m, n, &I)) return false;
    p->fn = I.fn; p->name = I.name; p->threads = I.threads; p->smem = I.smem; p->slot = 0;
    p->phase1 = I.phase1; p->p1_bytes = I.p1_bytes;
    return true;
}

// Row-warp-per-LP variants (blp_pairlp_kernel.cuh): NWR warps own 32 rows each, a row's
// first R positions in registers and the next S in a [S][ST] shared tile (ST >= m).
template <int R, int S, int NWR, int ST, int MINB>
bool use_pairlp(int m, int ncols, const char *name, Plan *p) {
    if (m > ST || ncols > R + S) return false;
    p->fn = blp::pairlp_kernel<R, S, NWR, ST, MINB>;
    p->name = name;
    p->smem = blp::PairCfg<R, S, NWR, ST>::BYTES;
    p->threads = 32 * NWR;
    p->slot = 0;
    return true;
}

// 32 < m <= 64: two row-warps (C4 64 x 32); 64 < m <= 128: four (C3 100 x 100), 2 LPs per SM.
// BLP_PAIR / BLP_QUAD = register columns per row.
bool plan_pairlp(int m, int n, Plan *p) {
    const int ncols = n + m + 1;
    if (m > 64 && m <= 128) {
        if (env_int("BLP_QUAD", 96) == 80 && use_pairlp<80, 122, 4, 101, 2>(m, ncols, "quadlp_r80_s122", p))
            return true;
        return use_pairlp<96, 106, 4, 129, 2>(m, ncols, "quadlp_r96_s106", p);
    }
    if (m <= 32 || m > 64) return false;
    if (env_int("BLP_PAIR", 62) == 50) return use_pairlp<50, 48, 2, 65, 7>(m, ncols, "pairlp_r50_s48", p);
    if (use_pairlp<62, 36, 2, 65, 6>(m, ncols, "pairlp_r62_s36", p)) return true;      // C4: 97 columns
    return use_pairlp<62, 48, 2, 65, 6>(m, ncols, "pairlp_r62_s48", p);                // up to 110 (50 x 50)
}

// Cluster-resident variant: tableaux that no single-SM variant holds on chip
// (the smem tableau exceeds 227 KB), up to 512 rows.
bool plan_cluster(int m, int n, bool forced, Plan *p) {
    if (!forced) {
        if (env_int("BLP_FORCE_HBM", 0)) return false;
        if (blp::make_tab_layout(m, n, 32, true).bytes <= kMaxDynSmem) return false;
    }
    if (!blp_cluster::shape_fits(m, n)) return false;
    p->fn = nullptr;
    p->name = blp_cluster::variant_name(m, n);
    p->threads = 0;
    p->smem = 0;
    p->slot = 0;
    p->cluster = true;
    return true;
}

// BLP_KERNEL=condensed|warplp|pairlp|regtile|cluster|smem forces a family (testing / tuning).
bool plan_launch(int m, int n, Plan *p, bool shared_Ab = false) {
    const char *force = getenv("BLP_KERNEL");
    const bool any = !force || !*force;
    if ((any || strcmp(force, "condensed") == 0) && plan_condensed(m, n, p)) {
        // the multi-warp condensed form (33..128 rows) takes the lazy kernel's deferrals, as
        // the dense 33..128-row kernels do (below) -- except in support mode, where the shared
        // phase 1 applies and the lazy pass only adds work (C4 2e5: 9.18 -> 7.88 ms without it)
        p->lazy = !shared_Ab && p->threads > 32 && any && m > 32 && env_int("BLP_LAZY_SMALL", 1) != 0 &&
                  blp_cluster::lazy_enabled(m, n);
        if (p->lazy) {
            static thread_local std::string cname;
            cname = std::string("lazy+") + p->name;
            p->name = cname.c_str();
        }
        return true;
    }
    if ((any || strcmp(force, "warplp") == 0) && plan_warplp(m, n, p)) return true;
    bool dense = (any || strcmp(force, "pairlp") == 0) && plan_pairlp(m, n, p);
    if (!dense) {
        if ((any || strcmp(force, "warplp") == 0 || strcmp(force, "regtile") == 0) && plan_regtile(m, n, p)) return true;
        if ((any || strcmp(force, "cluster") == 0) && plan_cluster(m, n, !any, p)) return true;   // lazy inside
        dense = plan_tableau(m, n, p);
    }
    if (!dense) return false;
    // The exact lazy tableau first (single-phase LPs within 64 pivots), the dense kernel for
    // what it defers: always ahead of the HBM-streamed kernel; ahead of the 33..128-row and
    // shared-memory kernels unless a family is forced.  Measured
    // (scripts/lazy_vs_dense.py, device-resident): the reference's random workload 2.5x faster
    // at 50 x 50, 3.6x at 64 x 64, 4.5x at 100 x 100 (5-8 pivots); the support-function batch
    // (C4, 64 x 32, ~24 pivots) 1.18x; C3 unchanged (phase-1 LPs are handed over after one
    // look at b).
    p->lazy = blp_cluster::lazy_enabled(m, n) &&
              (p->slot != 0 ? env_int("BLP_FORCE_HBM", 0) == 0
                            : (any && m > 32 && env_int("BLP_LAZY_SMALL", 1) != 0));
    if (p->lazy) {
        static thread_local std::string name;
        name = std::string("lazy+") + p->name;
        p->name = name.c_str();
    }
    return true;
}

struct DeviceInfo {
    int sms = 0;
    bool init = false;
};
std::mutex g_mu;
DeviceInfo g_dev[64];

int device_sms(int dev, int *sms) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (dev < 0 || dev >= 64) return fail(BLP_ERR_INVALID, "device index out of range");
    if (!g_dev[dev].init) {
        BLP_CUDA_TRY(cudaDeviceGetAttribute(&g_dev[dev].sms, cudaDevAttrMultiProcessorCount, dev));
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            unsigned long long thr = ~0ull;  // keep freed blocks cached between calls
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        g_dev[dev].init = true;
    }
    *sms = g_dev[dev].sms;
    return BLP_OK;
}

void fill_batch(blp::Batch &B, const double *A, const double *b, const double *c, long long count, int m, int n,
                int shared_Ab, const blp_limits *lim, int8_t *status, double *objective, double *x, int32_t *it1,
                int32_t *it2) {
    B.A = A; B.b = b; B.c = c; B.count = count; B.m = m; B.n = n; B.shared_Ab = shared_Ab;
    B.status = status; B.objective = objective; B.x = x; B.it1 = it1; B.it2 = it2;
    B.next_lp = nullptr;
    B.gtab = nullptr;
    B.gtab_stride = 0;
    B.defer_list = nullptr;
    B.defer_count = nullptr;
    B.p1state = nullptr;
    B.vq = nullptr;
    B.vflag = nullptr;
    B.vfirst = 0;
    B.lim.max_iterations = lim ? lim->max_iterations : 0;
    B.lim.anti_cycling = lim ? lim->anti_cycling : 1;
    B.lim.degenerate_limit = lim ? lim->degenerate_limit : -1;
    B.lim.reserved = 0;
}

blp::Batch Bproto(const double *A, const double *b, const double *c, long long count, int m, int n, int shared_Ab,
                  const blp_limits *lim, int8_t *status, double *objective, double *x, int32_t *it1, int32_t *it2) {
    blp::Batch B;
    fill_batch(B, A, b, c, count, m, n, shared_Ab, lim, status, objective, x, it1, it2);
    return B;
}

int launch_cluster(const double *A, const double *b, const double *c, long long count, int m, int n,
                   int shared_Ab, const blp_limits *lim, int8_t *status, double *objective, double *x,
                   int32_t *it1, int32_t *it2, cudaStream_t stream) {
    blp::Batch B;
    fill_batch(B, A, b, c, count, m, n, shared_Ab, lim, status, objective, x, it1, it2);
    int K = 0, clusters = 0;
    const cudaError_t e = blp_cluster::lazy_enabled(m, n) ? blp_cluster::launch_lazy_then_cluster(B, stream)
                                                           : blp_cluster::launch(B, stream, &K, &clusters);
    if (e != cudaSuccess) return fail(BLP_ERR_CUDA, std::string("cluster launch: ") + cudaGetErrorString(e));
    // lazy, cluster (+ validate and/or finalize)
    g_launches.fetch_add(blp_cluster::lazy_enabled(m, n) ? 2 + blp_cluster::finish_lazy_launches(B) : 1,
                         std::memory_order_relaxed);
    return BLP_OK;
}

int launch_solve(const double *A, const double *b, const double *c, long long count, int m, int n,
                 int shared_Ab, const blp_limits *lim, int8_t *status, double *objective, double *x,
                 int32_t *it1, int32_t *it2, cudaStream_t stream) {
    if (count == 0) return BLP_OK;
    int dev = 0;
    BLP_CUDA_TRY(cudaGetDevice(&dev));
    int sms = 0;
    int rc = device_sms(dev, &sms);
    if (rc) return rc;
    Plan P;
    if (!plan_launch(m, n, &P, shared_Ab != 0)) return fail(BLP_ERR_TOO_LARGE, "LP shape exceeds every kernel variant");
    if (P.cluster) return launch_cluster(A, b, c, count, m, n, shared_Ab, lim, status, objective, x, it1, it2, stream);
    BLP_CUDA_TRY(cudaFuncSetAttribute(P.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem));
    int occ = 0;
    BLP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, P.fn, P.threads, P.smem));
    if (occ < 1) return fail(BLP_ERR_TOO_LARGE, "kernel variant cannot be resident on an SM");
    long long grid = (long long)occ * sms;
    if (grid > count) grid = count;
    int *defer_list = nullptr, *defer_count = nullptr;
    void *lazy_ws = nullptr;
    if (P.lazy) {   // the lazy kernel over the batch; this kernel then solves only what it defers
        const cudaError_t le = blp_cluster::launch_lazy(Bproto(A, b, c, count, m, n, shared_Ab, lim, status, objective,
                                                               x, it1, it2), stream, &defer_list, &defer_count, &lazy_ws);
        if (le != cudaSuccess) return fail(BLP_ERR_CUDA, std::string("lazy launch: ") + cudaGetErrorString(le));
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }

    const size_t slot_bytes = (size_t)P.slot * sizeof(double) * (size_t)grid;
    const bool p1 = shared_Ab && P.phase1 != nullptr;
    const size_t ws_bytes = 256 + slot_bytes + (p1 ? P.p1_bytes : 0);
    void *ws = nullptr;
    BLP_CUDA_TRY(cudaMallocAsync(&ws, ws_bytes, stream));
    BLP_CUDA_TRY(cudaMemsetAsync(ws, 0, 256, stream));

    blp::Batch B;
    B.A = A; B.b = b; B.c = c; B.count = count; B.m = m; B.n = n; B.shared_Ab = shared_Ab;
    B.status = status; B.objective = objective; B.x = x; B.it1 = it1; B.it2 = it2;
    B.next_lp = reinterpret_cast<int *>(ws);
    B.gtab = P.slot ? reinterpret_cast<double *>(reinterpret_cast<char *>(ws) + 256) : nullptr;
    B.gtab_stride = P.slot;
    B.defer_list = defer_list;
    B.defer_count = defer_count;
    B.p1state = nullptr;
    B.vq = nullptr;
    B.vflag = nullptr;
    B.vfirst = 0;
    B.lim.max_iterations = lim ? lim->max_iterations : 0;
    B.lim.anti_cycling = lim ? lim->anti_cycling : 1;
    B.lim.degenerate_limit = lim ? lim->degenerate_limit : -1;
    B.lim.reserved = 0;

    if (p1) {   // support mode: phase 1 + restore_objective once for the shared A, b
        double *st = reinterpret_cast<double *>(reinterpret_cast<char *>(ws) + 256 + slot_bytes);
        BLP_CUDA_TRY(cudaFuncSetAttribute(P.phase1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem));
        P.phase1<<<1, P.threads, P.smem, stream>>>(B, st);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        BLP_CUDA_TRY(cudaGetLastError());
        B.p1state = st;
    }
    P.fn<<<(unsigned)grid, P.threads, P.smem, stream>>>(B);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    BLP_CUDA_TRY(cudaGetLastError());
    BLP_CUDA_TRY(cudaFreeAsync(ws, stream));
    if (P.lazy) {
        BLP_CUDA_TRY(blp_cluster::finish_lazy(B, stream, lazy_ws));
        g_launches.fetch_add(blp_cluster::finish_lazy_launches(B), std::memory_order_relaxed);
    }
    return BLP_OK;
}

bool bad_args(const double *A, const double *b, const double *c, long long count, int m, int n,
              const int8_t *status, const double *objective, const double *x, const int32_t *it1,
              const int32_t *it2) {
    if (count < 0 || m < 0 || n < 0) return true;
    if (count == 0) return false;
    if ((m > 0 && (!b || (n > 0 && !A))) || (n > 0 && (!c || !x))) return true;
    return !status || !objective || !it1 || !it2;
}

// Shared-memory bandwidth probe: every thread streams 16-byte LDS/STS pairs
// over a conflict-free slice for `iters` rounds (the roofline denominator of
// the smem-resident kernels; BASELINE.md §2 asks for it to be measured).
__global__ void __launch_bounds__(1024) smem_probe_kernel(double *sink, int iters) {
    extern __shared__ __align__(16) unsigned char probe_smem[];
    const unsigned base = (unsigned)__cvta_generic_to_shared(probe_smem);
    const int slots = blockDim.x * 4;
    for (int s = threadIdx.x; s < slots; s += blockDim.x) {
        const unsigned a = base + 16u * s;
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"((double)s), "d"(1.0) : "memory");
    }
    __syncthreads();
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const unsigned a = base + 16u * (threadIdx.x + q * blockDim.x);
            double x, y;
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a) : "memory");
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(y), "d"(x) : "memory");
            acc += x;
        }
    }
    if (acc == -1.0) sink[0] = acc;  // keep the loop observable
}

// FP64 pipe probe: independent DMUL -> DADD chains (unfused, like the tableau
// update), the roofline denominator of the register-resident kernels.
__global__ void __launch_bounds__(256) fp64_probe_kernel(double *sink, int iters, double s, double t) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __dadd_rn(__dmul_rn(x[k], s), t);
    }
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += x[k];
    if (acc == -1.0) sink[0] = acc;
}

// Restores the caller's current device on every return from a host entry point
// (they cudaSetDevice to the requested GPU; the caller's torch/CUDA state must not move).
struct DeviceGuard {
    int saved = -1;
    DeviceGuard() {
        if (cudaGetDevice(&saved) != cudaSuccess) { cudaGetLastError(); saved = -1; }
    }
    ~DeviceGuard() {
        if (saved >= 0) cudaSetDevice(saved);
    }
};

struct StreamSet {
    std::vector<cudaStream_t> s;
};
StreamSet g_streams[64];

// ---------------------------------------------------------------------------
// Pageable host buffers (plain numpy arrays through the reference API): copies
// from/to them are staged by the driver and synchronous, which serialises the
// sub-batch pipeline (C2 1e5: 70 ms pageable vs 14.9 ms pinned).  The staged
// path copies them through a per-device ring of pinned slots with a small
// pool of host threads (parallel memcpy), overlapped with the H2D / kernel /
// D2H of earlier sub-batches.

class CopyPool {
  public:
    explicit CopyPool(int n) {
        for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : workers_) t.join();
    }
    // f(0) .. f(parts-1) over the pool (the caller runs f(0)); returns when all are done
    void parallel_for(int parts, const std::function<void(int)> &f) {
        parts = std::max(1, std::min(parts, (int)workers_.size() + 1));
        if (parts == 1) { f(0); return; }
        {
            std::lock_guard<std::mutex> lk(m_);
            for (int k = 1; k < parts; ++k) {
                ++pending_;
                tasks_.push_back([&f, k] { f(k); });
            }
        }
        cv_.notify_all();
        f(0);
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [&] { return pending_ == 0; });
    }
    int threads() const { return (int)workers_.size() + 1; }
    // memcpy of n bytes split over the pool (and the caller)
    void copy(void *dst, const void *src, size_t n) {
        constexpr size_t kMin = 1 << 20;
        const int parts = (int)std::min<size_t>((size_t)workers_.size() + 1, std::max<size_t>(1, n / kMin));
        if (parts <= 1) { std::memcpy(dst, src, n); return; }
        const size_t step = (n + parts - 1) / parts;
        {
            std::lock_guard<std::mutex> lk(m_);
            for (int k = 1; k < parts; ++k) {
                const size_t off = step * k;
                if (off >= n) break;
                ++pending_;
                tasks_.push_back([=] { std::memcpy((char *)dst + off, (const char *)src + off, std::min(step, n - off)); });
            }
        }
        cv_.notify_all();
        std::memcpy(dst, src, std::min(step, n));
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [&] { return pending_ == 0; });
    }

  private:
    void loop() {
        for (;;) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || !tasks_.empty(); });
                if (stop_ && tasks_.empty()) return;
                f = std::move(tasks_.back());
                tasks_.pop_back();
            }
            f();
            {
                std::lock_guard<std::mutex> lk(m_);
                if (--pending_ == 0) done_.notify_all();
            }
        }
    }
    std::vector<std::thread> workers_;
    std::vector<std::function<void()>> tasks_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    int pending_ = 0;
    bool stop_ = false;
};

CopyPool &copy_pool() {
    static CopyPool pool(std::max(1, env_int("BLP_COPY_THREADS",
                                             std::min(8, (int)std::thread::hardware_concurrency() - 1))));
    return pool;
}

bool is_pinned(const void *p) {
    if (!p) return true;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

struct Staging {
    char *in[4] = {}, *out[4] = {};
    size_t in_bytes = 0, out_bytes = 0;
    char *poly = nullptr;          // pinned copy of a shared polytope (support mode), reused
    size_t poly_bytes = 0;
};
Staging g_staging[64];
std::mutex g_staging_mu[64];

// Where a staged sub-batch's inputs come from: three contiguous packed arrays, or
// (blp_solve_batch_gather) one pointer per LP for each of A, b, c.
struct InputSource {
    const double *A = nullptr, *b = nullptr, *c = nullptr;
    const double *const *Ap = nullptr, *const *bp = nullptr, *const *cp = nullptr;
    bool gather() const { return Ap != nullptr; }
};

// Host-buffer solve through the pinned staging ring (see above).
int solve_host_staged(const InputSource &src, long long count, int m, int n,
                      int shared_Ab, const blp_limits *lim, int8_t *status, double *objective, double *x,
                      int32_t *it1, int32_t *it2, int device, const std::vector<cudaStream_t> &ss) {
    const double *A = src.A, *b = src.b, *c = src.c;
    constexpr int kSlots = 4;
    const size_t szA = (size_t)m * n, szb = (size_t)m;
    const size_t in_lp = (shared_Ab ? 0 : (szA + szb) * 8) + (size_t)n * 8;
    const size_t out_lp = (size_t)n * 8 + 8 + 4 + 4 + 1;
    // Slot size: room for >= 2048 LPs (or a 16th of the batch), between 64 and 256 MB
    // (BLP_STAGE_MB overrides).  Large LPs need it: C3 (81 KB of inputs per LP) through the
    // list API in 64 MB slots ran 792-LP sub-batches, too small to fill the GPU: 600 ms per
    // 1e5; 256 MB: 376 ms.
    const size_t want_slot = in_lp * (size_t)std::max<long long>(2048, (count + 15) / 16);
    const size_t dflt_mb = std::min<size_t>(256, std::max<size_t>(64, (want_slot + (1 << 20) - 1) >> 20));
    const size_t slot = (size_t)std::max(1, env_int("BLP_STAGE_MB", (int)dflt_mb)) << 20;
    long long chunk = std::max<long long>(1, (long long)(slot / std::max<size_t>(1, in_lp)));
    chunk = std::min<long long>(chunk, std::max<long long>(2048, (count + 15) / 16));   // keep a pipeline
    chunk = std::min<long long>(chunk, count);
    const size_t in_bytes = (size_t)chunk * in_lp + 64, out_bytes = (size_t)chunk * out_lp + 64;
    std::lock_guard<std::mutex> lk(g_staging_mu[device]);   // one staged call per device at a time
    Staging &st = g_staging[device];
    if (st.in_bytes < in_bytes || st.out_bytes < out_bytes) {
        for (int k = 0; k < kSlots; ++k) {
            if (st.in[k]) cudaFreeHost(st.in[k]);
            if (st.out[k]) cudaFreeHost(st.out[k]);
            st.in[k] = st.out[k] = nullptr;
        }
        st.in_bytes = st.out_bytes = 0;
        for (int k = 0; k < kSlots; ++k) {
            BLP_CUDA_TRY(cudaMallocHost(reinterpret_cast<void **>(&st.in[k]), in_bytes));
            BLP_CUDA_TRY(cudaMallocHost(reinterpret_cast<void **>(&st.out[k]), out_bytes));
        }
        st.in_bytes = in_bytes;
        st.out_bytes = out_bytes;
    }
    // Shared polytope: uploaded once on ss[0] through pinned slot 0 (a pageable source
    // would let cudaMemcpy return before the DMA lands), and every stream waits for it.
    // The pinned copy is a per-device buffer reused across calls (pinning pages per call cost
    // ~ms: the reference's list API makes one call per planned chunk, 49 for C4), and the
    // device copy is stream-ordered (cudaMallocAsync / cudaFreeAsync on ss[0]): calls on a
    // device are serialised by the staging mutex and drain every stream before returning.
    double *dA_shared = nullptr, *db_shared = nullptr;
    if (shared_Ab) {
        const size_t pbytes = (szA + szb) * 8 + 16;
        if (st.poly_bytes < pbytes) {
            if (st.poly) cudaFreeHost(st.poly);
            st.poly = nullptr;
            st.poly_bytes = 0;
            BLP_CUDA_TRY(cudaMallocHost(reinterpret_cast<void **>(&st.poly), pbytes));
            st.poly_bytes = pbytes;
        }
        char *hp = st.poly;
        BLP_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&dA_shared), (std::max<size_t>(1, szA) + std::max<size_t>(1, szb)) * 8,
                                     ss[0]));
        db_shared = dA_shared + std::max<size_t>(1, szA);
        if (szA) std::memcpy(hp, A, szA * 8);
        if (szb) std::memcpy(hp + szA * 8, b, szb * 8);
        cudaError_t e = cudaSuccess;
        if (szA) e = cudaMemcpyAsync(dA_shared, hp, szA * 8, cudaMemcpyHostToDevice, ss[0]);
        if (e == cudaSuccess && szb) e = cudaMemcpyAsync(db_shared, hp + szA * 8, szb * 8, cudaMemcpyHostToDevice, ss[0]);
        cudaEvent_t up;
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&up, cudaEventDisableTiming);
        if (e == cudaSuccess) {
            e = cudaEventRecord(up, ss[0]);
            for (int k = 1; k < kSlots && e == cudaSuccess; ++k) e = cudaStreamWaitEvent(ss[k], up, 0);
            cudaEventDestroy(up);
        }
        if (e != cudaSuccess) {
            cudaStreamSynchronize(ss[0]);
            cudaFreeAsync(dA_shared, ss[0]);
            cudaStreamSynchronize(ss[0]);
            return fail(BLP_ERR_CUDA, std::string("shared polytope upload: ") + cudaGetErrorString(e));
        }
    }
    cudaEvent_t ev[kSlots];
    for (int k = 0; k < kSlots; ++k) BLP_CUDA_TRY(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
    long long s0[kSlots], sc[kSlots];
    for (int k = 0; k < kSlots; ++k) { s0[k] = -1; sc[k] = 0; }
    CopyPool &pool = copy_pool();
    // outputs of slot k's sub-batch back into the caller's buffers, once its D2H is done
    auto drain = [&](int k) -> cudaError_t {
        if (s0[k] < 0) return cudaSuccess;
        const cudaError_t e = cudaEventSynchronize(ev[k]);
        if (e != cudaSuccess) return e;
        const long long st0 = s0[k], cnt = sc[k];
        const char *o = st.out[k];
        pool.copy(objective + st0, o, (size_t)cnt * 8);             o += (size_t)cnt * 8;
        if (n) pool.copy(x + st0 * n, o, (size_t)cnt * n * 8);       o += (size_t)cnt * n * 8;
        std::memcpy(it1 + st0, o, (size_t)cnt * 4);                 o += (size_t)cnt * 4;
        std::memcpy(it2 + st0, o, (size_t)cnt * 4);                 o += (size_t)cnt * 4;
        std::memcpy(status + st0, o, (size_t)cnt);
        s0[k] = -1;
        return cudaSuccess;
    };
    int rc = BLP_OK;
    int i = 0;
    for (long long start = 0; start < count && rc == BLP_OK; start += chunk, ++i) {
        const int k = i % kSlots;
        cudaStream_t s = ss[k];
        const cudaError_t de = drain(k);
        if (de != cudaSuccess) { rc = fail(BLP_ERR_CUDA, cudaGetErrorString(de)); break; }
        const long long cnt = std::min(chunk, count - start);
        // stage this sub-batch's inputs: [A][b][c], packed
        char *p = st.in[k];
        if (src.gather()) {
            // one memcpy per LP array, LP ranges split over the copy threads (a shared
            // polytope: only the objectives)
            const size_t sa = shared_Ab ? 0 : szA, sb = shared_Ab ? 0 : szb;
            char *pA = p, *pb = p + (size_t)cnt * sa * 8, *pc = pb + (size_t)cnt * sb * 8;
            // split by bytes, not LP count: 128 LPs of 500 x 500 are 256 MB (C5 through the list
            // API: one copy thread at cnt / 256 = 0, 8.5 GB/s)
            const long long bytes = cnt * (long long)((sa + sb + n) * 8);
            const int parts = (int)std::min<long long>(pool.threads(), std::max<long long>(1, bytes >> 21));
            pool.parallel_for(parts, [&](int part) {
                const long long k0 = cnt * part / parts, k1 = cnt * (part + 1) / parts;
                for (long long q = k0; q < k1; ++q) {
                    const long long lpk = start + q;
                    if (sa) std::memcpy(pA + (size_t)q * sa * 8, src.Ap[lpk], sa * 8);
                    if (sb) std::memcpy(pb + (size_t)q * sb * 8, src.bp[lpk], sb * 8);
                    if (n) std::memcpy(pc + (size_t)q * n * 8, src.cp[lpk], (size_t)n * 8);
                }
            });
        } else {
            if (!shared_Ab) {
                if (szA) pool.copy(p, A + start * szA, (size_t)cnt * szA * 8);
                p += (size_t)cnt * szA * 8;
                if (szb) pool.copy(p, b + start * szb, (size_t)cnt * szb * 8);
                p += (size_t)cnt * szb * 8;
            }
            if (n) pool.copy(p, c + start * n, (size_t)cnt * n * 8);
        }
        const size_t bytes_in = (size_t)cnt * in_lp, bytes_out = (size_t)cnt * out_lp;
        char *buf = nullptr;
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&buf), bytes_in + bytes_out + 256, s);
        if (e != cudaSuccess) { rc = fail(BLP_ERR_CUDA, cudaGetErrorString(e)); break; }
        char *q = buf;
        const double *dA = dA_shared, *db = db_shared;
        if (!shared_Ab) {
            dA = reinterpret_cast<double *>(q); q += (size_t)cnt * szA * 8;
            db = reinterpret_cast<double *>(q); q += (size_t)cnt * szb * 8;
        }
        const double *dc = reinterpret_cast<double *>(q); q += (size_t)cnt * n * 8;
        char *dout = buf + bytes_in;                 // [objective][x][it1][it2][status], as the out slot
        double *dobj = reinterpret_cast<double *>(dout);
        double *dx = dobj + cnt;
        int32_t *dit1 = reinterpret_cast<int32_t *>(dx + (size_t)cnt * n);
        int32_t *dit2 = dit1 + cnt;
        int8_t *dst = reinterpret_cast<int8_t *>(dit2 + cnt);
        if (bytes_in) e = cudaMemcpyAsync(buf, st.in[k], bytes_in, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) { rc = fail(BLP_ERR_CUDA, cudaGetErrorString(e)); break; }
        rc = launch_solve(dA, db, dc, cnt, m, n, shared_Ab, lim, dst, dobj, dx, dit1, dit2, s);
        if (rc != BLP_OK) break;
        e = cudaMemcpyAsync(st.out[k], dout, bytes_out, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaEventRecord(ev[k], s);
        if (e == cudaSuccess) e = cudaFreeAsync(buf, s);
        if (e != cudaSuccess) { rc = fail(BLP_ERR_CUDA, cudaGetErrorString(e)); break; }
        s0[k] = start;
        sc[k] = cnt;
    }
    for (int k = 0; k < kSlots; ++k) {
        const cudaError_t de = drain(k);
        if (de != cudaSuccess && rc == BLP_OK) rc = fail(BLP_ERR_CUDA, cudaGetErrorString(de));
    }
    for (int k = 0; k < kSlots; ++k) {
        const cudaError_t e = cudaStreamSynchronize(ss[k]);
        if (e != cudaSuccess && rc == BLP_OK) rc = fail(BLP_ERR_CUDA, cudaGetErrorString(e));
        cudaEventDestroy(ev[k]);
    }
    if (dA_shared) {                         // every stream drained above
        cudaFreeAsync(dA_shared, ss[0]);
        cudaStreamSynchronize(ss[0]);
    }
    return rc;
}

// The per-device stream set of the host entry points (created once).
int device_streams(int device, int count) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto &ss = g_streams[device].s;
    if (ss.empty()) {
        ss.resize(count);
        for (auto &s : ss) BLP_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    }
    return BLP_OK;
}

}  // namespace

extern "C" {

int blp_abi_version(void) { return BLP_ABI_VERSION; }

double blp_probe_fp64_gflops(int32_t device) {
    DeviceGuard guard;
    g_last_error.clear();
    int sms = 0;
    if (cudaSetDevice(device) != cudaSuccess || device_sms(device, &sms) != BLP_OK) return -1.0;
    double *sink = nullptr;
    if (cudaMalloc(&sink, 8) != cudaSuccess) return -1.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = 8 * sms, threads = 256, iters = 8192;
    fp64_probe_kernel<<<grid, threads>>>(sink, 64, 0.999999, 1e-7);  // warm-up
    cudaEventRecord(e0);
    fp64_probe_kernel<<<grid, threads>>>(sink, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    g_launches.fetch_add(2, std::memory_order_relaxed);
    float ms = 0.f;
    const bool ok = cudaEventSynchronize(e1) == cudaSuccess && cudaEventElapsedTime(&ms, e0, e1) == cudaSuccess;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (!ok || ms <= 0.f) return -1.0;
    const double flops = 2.0 * 8.0 * (double)iters * grid * threads;  // one DMUL + one DADD per step
    return flops / (ms * 1e-3) / 1e9;
}

double blp_probe_smem_gbs(int32_t device) {
    DeviceGuard guard;
    g_last_error.clear();
    int sms = 0;
    if (cudaSetDevice(device) != cudaSuccess || device_sms(device, &sms) != BLP_OK) return -1.0;
    const int threads = 1024, iters = 4096;
    const size_t smem = (size_t)threads * 4 * 16;  // 64 KB: two CTAs (2048 threads) per SM
    if (cudaFuncSetAttribute(smem_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return -1.0;
    double *sink = nullptr;
    cudaEvent_t e0, e1;
    if (cudaMalloc(&sink, 8) != cudaSuccess) return -1.0;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = 2 * sms;
    smem_probe_kernel<<<grid, threads, smem>>>(sink, 64);  // warm-up
    cudaEventRecord(e0);
    smem_probe_kernel<<<grid, threads, smem>>>(sink, iters);
    cudaEventRecord(e1);
    g_launches.fetch_add(2, std::memory_order_relaxed);
    float ms = 0.f;
    const bool ok = cudaEventSynchronize(e1) == cudaSuccess && cudaEventElapsedTime(&ms, e0, e1) == cudaSuccess;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (!ok || ms <= 0.f) return -1.0;
    const double bytes = (double)grid * threads * 4.0 * 32.0 * iters;  // 16 B read + 16 B write per slot
    return bytes / (ms * 1e-3) / 1e9;
}

const char *blp_last_error(void) { return g_last_error.c_str(); }

int64_t blp_launch_count(void) { return g_launches.load(); }

int blp_shape_supported(int32_t m, int32_t n) {
    Plan P;
    if (m < 0 || n < 0) return 0;
    return plan_launch(m, n, &P) ? 1 : 0;
}

const char *blp_kernel_variant_mode(int32_t m, int32_t n, int32_t shared_Ab) {
    static thread_local std::string name;
    Plan P;
    if (!plan_launch(m, n, &P, shared_Ab != 0)) return "unsupported";
    name = P.name;
    return name.c_str();
}

const char *blp_kernel_variant(int32_t m, int32_t n) {
    Plan P;
    if (m < 0 || n < 0) return "invalid";
    plan_launch(m, n, &P);
    return P.name;
}

int blp_solve_batch_device(const double *A, const double *b, const double *c, int64_t count,
                           int32_t m, int32_t n, int32_t shared_Ab, const blp_limits *limits,
                           int8_t *status, double *objective, double *x, int32_t *iters1,
                           int32_t *iters2, void *cuda_stream) {
    g_last_error.clear();
    if (bad_args(A, b, c, count, m, n, status, objective, x, iters1, iters2))
        return fail(BLP_ERR_INVALID, "invalid arguments");
    return launch_solve(A, b, c, count, m, n, shared_Ab, limits, status, objective, x, iters1, iters2,
                        reinterpret_cast<cudaStream_t>(cuda_stream));
}

int blp_solve_batch_host(const double *A, const double *b, const double *c, int64_t count,
                         int32_t m, int32_t n, int32_t shared_Ab, const blp_limits *limits,
                         int8_t *status, double *objective, double *x, int32_t *iters1,
                         int32_t *iters2, int32_t device) {
    DeviceGuard guard;
    g_last_error.clear();
    if (bad_args(A, b, c, count, m, n, status, objective, x, iters1, iters2))
        return fail(BLP_ERR_INVALID, "invalid arguments");
    if (count == 0) return BLP_OK;
    if (device < 0 || device >= 64) return fail(BLP_ERR_INVALID, "device index out of range");
    BLP_CUDA_TRY(cudaSetDevice(device));
    constexpr int kStreams = 4;
    {
        const int rc = device_streams(device, kStreams);
        if (rc != BLP_OK) return rc;
    }
    const auto &ss = g_streams[device].s;
    // Pageable caller buffers: through the pinned staging ring (BLP_STAGE=0 disables).
    if (env_int("BLP_STAGE", 1) &&
        !(is_pinned(A) && is_pinned(b) && is_pinned(c) && is_pinned(status) && is_pinned(objective) &&
          is_pinned(x) && is_pinned(iters1) && is_pinned(iters2)))
    {
        InputSource src;
        src.A = A; src.b = b; src.c = c;
        return solve_host_staged(src, count, m, n, shared_Ab, limits, status, objective, x, iters1, iters2,
                                 device, ss);
    }
    // Sub-batches: BLP_HOST_CHUNKS of them (default 16), at least 2048 LPs each, the last ones
    // tapered (BLP_HOST_TAPER, default 2).  C2 1e5 (round-2 kernels, 13.8 ms pinned-H2D floor):
    // 16 chunks 14.66 ms uniform / 14.51 tapered; 20: 14.63 / 14.53; 24: 14.84 / 14.57;
    // 32: 15.0 / 15.0 (round 1, slower kernel: 16 -> 15.2, 32 -> 14.9, 64 -> 15.2).
    const int nchunks = std::max(1, env_int("BLP_HOST_CHUNKS", 16));
    const long long chunk = std::max<long long>(2048, (count + nchunks - 1) / nchunks);
    const size_t szA = (size_t)m * n, szb = (size_t)m;

    // Shared polytope (support-function mode): one H2D, every stream waits on it.
    // Errors inside the pipeline break out of it: the streams are always drained and the
    // shared buffers freed before returning, so no queued D2H can land in the caller's
    // buffers after this call has returned.
    double *dA_shared = nullptr, *db_shared = nullptr;
    cudaEvent_t shared_ready = nullptr;
    int rc = BLP_OK;
    auto check = [&](cudaError_t e, const char *what) {
        if (e != cudaSuccess && rc == BLP_OK) rc = fail(BLP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
        return rc == BLP_OK;
    };
    if (shared_Ab) {
        check(cudaMallocAsync(&dA_shared, std::max<size_t>(1, szA) * sizeof(double), ss[0]), "cudaMallocAsync");
        if (rc == BLP_OK) check(cudaMallocAsync(&db_shared, std::max<size_t>(1, szb) * sizeof(double), ss[0]), "cudaMallocAsync");
        if (rc == BLP_OK && szA) check(cudaMemcpyAsync(dA_shared, A, szA * sizeof(double), cudaMemcpyHostToDevice, ss[0]), "H2D");
        if (rc == BLP_OK && szb) check(cudaMemcpyAsync(db_shared, b, szb * sizeof(double), cudaMemcpyHostToDevice, ss[0]), "H2D");
        if (rc == BLP_OK) check(cudaEventCreateWithFlags(&shared_ready, cudaEventDisableTiming), "cudaEventCreate");
        if (rc == BLP_OK) check(cudaEventRecord(shared_ready, ss[0]), "cudaEventRecord");
        for (int k = 1; k < kStreams && rc == BLP_OK; ++k) check(cudaStreamWaitEvent(ss[k], shared_ready, 0), "cudaStreamWaitEvent");
    }
    // BLP_HOST_TAPER (default 2; 0 = uniform): the last sub-batches halve in size, so the
    // kernel + D2H after the final H2D is short (the pipeline's drain)
    const int taper = env_int("BLP_HOST_TAPER", 2);
    // BLP_HOST_RAMP (default 3): the first sub-batches grow chunk >> r, >> r-1, ... so the
    // first kernel starts after a short H2D (kernel-bound batches; C3 e2e 389.9 ms with a
    // uniform start, 371.9 with r = 2, 351.5 with r = 3 against a 349 ms kernel; C2, C4 unchanged)
    const int ramp = env_int("BLP_HOST_RAMP", 3);
    auto sub_size = [&](long long start) -> long long {
        const long long left = count - start;
        if (ramp > 0) {
            long long done = 0;
            for (int r = ramp; r >= 1; --r) {
                const long long sz = std::max<long long>(256, chunk >> r);
                if (start == done) return std::min(left, sz);
                done += sz;
            }
        }
        if (taper <= 0 || left > 2 * chunk) return std::min(chunk, left);
        const long long half = std::max<long long>(512, left / 2);
        return std::min(left, std::max<long long>(half, (chunk >> taper)));
    };
    int ci = 0;
    long long cnt = 0;
    for (long long start = 0; start < count && rc == BLP_OK; start += cnt, ++ci) {
        cnt = sub_size(start);
        cudaStream_t s = ss[ci % kStreams];
        const size_t bytes_in = shared_Ab ? (size_t)cnt * n * 8 : (size_t)cnt * (szA + szb + n) * 8;
        const size_t bytes_out = (size_t)cnt * (n * 8 + 8 + 1 + 8) + 64;
        char *buf = nullptr;
        if (!check(cudaMallocAsync(reinterpret_cast<void **>(&buf), bytes_in + bytes_out + 256, s), "cudaMallocAsync"))
            break;
        double *dA = dA_shared, *db = db_shared, *dc;
        char *p = buf;
        if (!shared_Ab) {
            dA = reinterpret_cast<double *>(p); p += (size_t)cnt * szA * 8;
            db = reinterpret_cast<double *>(p); p += (size_t)cnt * szb * 8;
        }
        dc = reinterpret_cast<double *>(p); p += (size_t)cnt * n * 8;
        double *dobj = reinterpret_cast<double *>(p); p += (size_t)cnt * 8;
        double *dx = reinterpret_cast<double *>(p); p += (size_t)cnt * n * 8;
        int32_t *dit1 = reinterpret_cast<int32_t *>(p); p += (size_t)cnt * 4;
        int32_t *dit2 = reinterpret_cast<int32_t *>(p); p += (size_t)cnt * 4;
        int8_t *dst = reinterpret_cast<int8_t *>(p);
        bool ok = true;
        if (!shared_Ab) {
            if (szA) ok = check(cudaMemcpyAsync(dA, A + start * szA, cnt * szA * 8, cudaMemcpyHostToDevice, s), "H2D");
            if (ok && szb) ok = check(cudaMemcpyAsync(db, b + start * szb, cnt * szb * 8, cudaMemcpyHostToDevice, s), "H2D");
        }
        if (ok && n) ok = check(cudaMemcpyAsync(dc, c + start * n, (size_t)cnt * n * 8, cudaMemcpyHostToDevice, s), "H2D");
        if (ok) {
            rc = launch_solve(dA, db, dc, cnt, m, n, shared_Ab, limits, dst, dobj, dx, dit1, dit2, s);
            ok = rc == BLP_OK;
        }
        if (ok) ok = check(cudaMemcpyAsync(status + start, dst, cnt, cudaMemcpyDeviceToHost, s), "D2H");
        if (ok) ok = check(cudaMemcpyAsync(objective + start, dobj, cnt * 8, cudaMemcpyDeviceToHost, s), "D2H");
        if (ok && n) ok = check(cudaMemcpyAsync(x + start * n, dx, (size_t)cnt * n * 8, cudaMemcpyDeviceToHost, s), "D2H");
        if (ok) ok = check(cudaMemcpyAsync(iters1 + start, dit1, cnt * 4, cudaMemcpyDeviceToHost, s), "D2H");
        if (ok) ok = check(cudaMemcpyAsync(iters2 + start, dit2, cnt * 4, cudaMemcpyDeviceToHost, s), "D2H");
        cudaFreeAsync(buf, s);
    }
    // drain every stream (also on error), then release the shared polytope
    for (int k = 0; k < kStreams; ++k) check(cudaStreamSynchronize(ss[k]), "cudaStreamSynchronize");
    if (dA_shared) cudaFree(dA_shared);
    if (db_shared) cudaFree(db_shared);
    if (shared_ready) cudaEventDestroy(shared_ready);
    return rc;
}

int blp_solve_batch_gather(const double *const *A, const double *const *b, const double *const *c,
                           int64_t count, int32_t m, int32_t n, const blp_limits *limits, int8_t *status,
                           double *objective, double *x, int32_t *iters1, int32_t *iters2, int32_t device) {
    DeviceGuard guard;
    g_last_error.clear();
    if (count < 0 || m < 0 || n < 0) return fail(BLP_ERR_INVALID, "invalid arguments");
    if (count == 0) return BLP_OK;
    if (!A || !b || !c || !status || !objective || !iters1 || !iters2 || (n > 0 && !x))
        return fail(BLP_ERR_INVALID, "invalid arguments");
    for (long long k = 0; k < count; ++k)
        if ((m && n && !A[k]) || (m && !b[k]) || (n && !c[k])) return fail(BLP_ERR_INVALID, "null LP array pointer");
    if (device < 0 || device >= 64) return fail(BLP_ERR_INVALID, "device index out of range");
    BLP_CUDA_TRY(cudaSetDevice(device));
    const int rc = device_streams(device, 4);
    if (rc != BLP_OK) return rc;
    InputSource src;
    src.Ap = A; src.bp = b; src.cp = c;
    // Every LP pointing at the same A and b (the support-function workload through the
    // reference's list API: one polytope object, many objectives): solved in support mode --
    // the polytope uploaded once, its phase 1 shared -- with outputs identical to solving
    // each LP on its own (tests/test_gpu_support_phase1.py).  BLP_GATHER_SHARED=0 disables.
    bool shared = env_int("BLP_GATHER_SHARED", 1) != 0;
    for (long long k = 1; k < count && shared; ++k) shared = A[k] == A[0] && b[k] == b[0];
    if (shared) { src.A = A[0]; src.b = b[0]; }
    return solve_host_staged(src, count, m, n, shared ? 1 : 0, limits, status, objective, x, iters1, iters2, device,
                             g_streams[device].s);
}

int blp_box_solve_device(const double *lower, const double *upper, const double *direction, int64_t count,
                         int32_t n, double *value, double *point, int32_t *status, void *cuda_stream) {
    g_last_error.clear();
    if (count < 0 || n < 0 || (count > 0 && (!value || !status || (n > 0 && (!lower || !upper || !direction || !point)))))
        return fail(BLP_ERR_INVALID, "invalid arguments");
    if (count == 0) return BLP_OK;
    int dev = 0, sms = 0;
    BLP_CUDA_TRY(cudaGetDevice(&dev));
    int rc = device_sms(dev, &sms);
    if (rc) return rc;
    blp::BoxBatch B{lower, upper, direction, count, n, value, point, status};
    const long long blocks = std::min<long long>((count + 255) / 256, (long long)sms * 8);
    blp::box_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(cuda_stream)>>>(B);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    BLP_CUDA_TRY(cudaGetLastError());
    return BLP_OK;
}

int blp_box_solve_host(const double *lower, const double *upper, const double *direction, int64_t count,
                       int32_t n, double *value, double *point, int32_t *status, int32_t device) {
    DeviceGuard guard;
    g_last_error.clear();
    if (count < 0 || n < 0) return fail(BLP_ERR_INVALID, "invalid arguments");
    if (count == 0) return BLP_OK;
    BLP_CUDA_TRY(cudaSetDevice(device));
    cudaStream_t s;
    BLP_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const size_t mat = (size_t)count * n * sizeof(double);
    char *buf = nullptr;
    int rc = BLP_OK;
    if (cudaMallocAsync(reinterpret_cast<void **>(&buf), 4 * mat + (size_t)count * 12 + 64, s) != cudaSuccess) {
        cudaStreamDestroy(s);
        return fail(BLP_ERR_CUDA, "cudaMallocAsync failed");
    }
    double *dl = reinterpret_cast<double *>(buf), *du = dl + (size_t)count * n, *dd = du + (size_t)count * n;
    double *dp = dd + (size_t)count * n, *dv = dp + (size_t)count * n;
    int32_t *dst = reinterpret_cast<int32_t *>(dv + count);
    if (mat) {
        cudaMemcpyAsync(dl, lower, mat, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(du, upper, mat, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dd, direction, mat, cudaMemcpyHostToDevice, s);
    }
    rc = blp_box_solve_device(dl, du, dd, count, n, dv, dp, dst, s);
    if (rc == BLP_OK) {
        cudaMemcpyAsync(value, dv, (size_t)count * 8, cudaMemcpyDeviceToHost, s);
        if (mat) cudaMemcpyAsync(point, dp, mat, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(status, dst, (size_t)count * 4, cudaMemcpyDeviceToHost, s);
    }
    cudaFreeAsync(buf, s);
    const cudaError_t e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (rc == BLP_OK && e != cudaSuccess) rc = fail(BLP_ERR_CUDA, cudaGetErrorString(e));
    return rc;
}

int blp_certify_batch_device(const double *A, const double *b, const double *c, const double *x, int64_t count,
                             int32_t m, int32_t n, int32_t shared_Ab, const int8_t *status, double tol,
                             double *max_reduced_cost, double *max_violation, double *max_negativity,
                             int8_t *needs_prices, void *cuda_stream) {
    g_last_error.clear();
    if (count < 0 || m < 0 || n < 0 || (count > 0 && (!c || !x || !status || !max_reduced_cost || !max_violation ||
                                                     !max_negativity || !needs_prices || (m > 0 && (!A || !b)))))
        return fail(BLP_ERR_INVALID, "invalid arguments");
    if (count == 0) return BLP_OK;
    int dev = 0, sms = 0;
    BLP_CUDA_TRY(cudaGetDevice(&dev));
    int rc = device_sms(dev, &sms);
    if (rc) return rc;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(cuda_stream);
    const size_t per_cta = (size_t)2 * m * m * sizeof(double);
    long long grid = std::min<long long>(count, (long long)sms * 8);
    if (per_cta) grid = std::max<long long>(1, std::min<long long>(grid, (1ll << 30) / (long long)per_cta));
    double *work = nullptr;
    if (per_cta && cudaMallocAsync(reinterpret_cast<void **>(&work), per_cta * grid, s) != cudaSuccess)
        return fail(BLP_ERR_CUDA, "cudaMallocAsync (certificate workspace) failed");
    const size_t smem = ((size_t)2 * n + 9 * (size_t)m + 32) * sizeof(double);
    if (smem > 48 * 1024) BLP_CUDA_TRY(cudaFuncSetAttribute(blp::cert_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    blp::CertBatch B{A, b, c, x, count, m, n, shared_Ab, status, tol, max_reduced_cost, max_violation, max_negativity,
                     needs_prices, work};
    blp::cert_kernel<<<(unsigned)grid, blp::kCertThreads, smem, s>>>(B);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const cudaError_t e = cudaGetLastError();
    if (work) cudaFreeAsync(work, s);
    if (e != cudaSuccess) return fail(BLP_ERR_CUDA, cudaGetErrorString(e));
    return BLP_OK;
}

int blp_certify_batch_host(const double *A, const double *b, const double *c, const double *x, int64_t count,
                           int32_t m, int32_t n, int32_t shared_Ab, const int8_t *status, double tol,
                           double *max_reduced_cost, double *max_violation, double *max_negativity,
                           int8_t *needs_prices, int32_t device) {
    DeviceGuard guard;
    g_last_error.clear();
    if (count < 0 || m < 0 || n < 0) return fail(BLP_ERR_INVALID, "invalid arguments");
    if (count == 0) return BLP_OK;
    BLP_CUDA_TRY(cudaSetDevice(device));
    cudaStream_t s;
    BLP_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const size_t na = (shared_Ab ? 1 : (size_t)count) * m * n, nb = (shared_Ab ? 1 : (size_t)count) * m;
    const size_t nc = (size_t)count * n;
    const size_t doubles = na + nb + 2 * nc + 3 * (size_t)count;
    char *buf = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void **>(&buf), doubles * 8 + 2 * (size_t)count + 64, s) != cudaSuccess) {
        cudaStreamDestroy(s);
        return fail(BLP_ERR_CUDA, "cudaMallocAsync failed");
    }
    double *dA = reinterpret_cast<double *>(buf), *db = dA + na, *dc = db + nb, *dx = dc + nc;
    double *drc = dx + nc, *dv = drc + count, *dn = dv + count;
    int8_t *dst = reinterpret_cast<int8_t *>(dn + count), *dneed = dst + count;
    if (na) cudaMemcpyAsync(dA, A, na * 8, cudaMemcpyHostToDevice, s);
    if (nb) cudaMemcpyAsync(db, b, nb * 8, cudaMemcpyHostToDevice, s);
    if (nc) {
        cudaMemcpyAsync(dc, c, nc * 8, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dx, x, nc * 8, cudaMemcpyHostToDevice, s);
    }
    cudaMemcpyAsync(dst, status, (size_t)count, cudaMemcpyHostToDevice, s);
    int rc = blp_certify_batch_device(dA, db, dc, dx, count, m, n, shared_Ab, dst, tol, drc, dv, dn, dneed, s);
    if (rc == BLP_OK) {
        cudaMemcpyAsync(max_reduced_cost, drc, (size_t)count * 8, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(max_violation, dv, (size_t)count * 8, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(max_negativity, dn, (size_t)count * 8, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(needs_prices, dneed, (size_t)count, cudaMemcpyDeviceToHost, s);
    }
    cudaFreeAsync(buf, s);
    const cudaError_t e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (rc == BLP_OK && e != cudaSuccess) rc = fail(BLP_ERR_CUDA, cudaGetErrorString(e));
    return rc;
}

int blp_certify_reprice_device(const double *A, const double *c, const double *y, int64_t count, int32_t m,
                               int32_t n, int32_t shared_Ab, const int8_t *mask, double *max_reduced_cost,
                               void *cuda_stream) {
    g_last_error.clear();
    if (count < 0 || m < 0 || n < 0 || (count > 0 && (!c || !mask || !max_reduced_cost || (m > 0 && (!A || !y)))))
        return fail(BLP_ERR_INVALID, "invalid arguments");
    if (count == 0) return BLP_OK;
    int dev = 0, sms = 0;
    BLP_CUDA_TRY(cudaGetDevice(&dev));
    int rc = device_sms(dev, &sms);
    if (rc) return rc;
    blp::CertPrices P{A, c, y, count, m, n, shared_Ab, mask, max_reduced_cost};
    const long long blocks = std::min<long long>((count + 7) / 8, (long long)sms * 8);
    blp::cert_prices_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(cuda_stream)>>>(P);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    BLP_CUDA_TRY(cudaGetLastError());
    return BLP_OK;
}

int blp_certify_reprice_host(const double *A, const double *c, const double *y, int64_t count, int32_t m,
                             int32_t n, int32_t shared_Ab, const int8_t *mask, double *max_reduced_cost,
                             int32_t device) {
    DeviceGuard guard;
    g_last_error.clear();
    if (count < 0 || m < 0 || n < 0) return fail(BLP_ERR_INVALID, "invalid arguments");
    if (count == 0) return BLP_OK;
    BLP_CUDA_TRY(cudaSetDevice(device));
    cudaStream_t s;
    BLP_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const size_t na = (shared_Ab ? 1 : (size_t)count) * m * n, nc = (size_t)count * n, ny = (size_t)count * m;
    char *buf = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void **>(&buf), (na + nc + ny + count) * 8 + count + 64, s) != cudaSuccess) {
        cudaStreamDestroy(s);
        return fail(BLP_ERR_CUDA, "cudaMallocAsync failed");
    }
    double *dA = reinterpret_cast<double *>(buf), *dc = dA + na, *dy = dc + nc, *drc = dy + ny;
    int8_t *dmask = reinterpret_cast<int8_t *>(drc + count);
    if (na) cudaMemcpyAsync(dA, A, na * 8, cudaMemcpyHostToDevice, s);
    if (nc) cudaMemcpyAsync(dc, c, nc * 8, cudaMemcpyHostToDevice, s);
    if (ny) cudaMemcpyAsync(dy, y, ny * 8, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(drc, max_reduced_cost, (size_t)count * 8, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(dmask, mask, (size_t)count, cudaMemcpyHostToDevice, s);
    int rc = blp_certify_reprice_device(dA, dc, dy, count, m, n, shared_Ab, dmask, drc, s);
    if (rc == BLP_OK) cudaMemcpyAsync(max_reduced_cost, drc, (size_t)count * 8, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(buf, s);
    const cudaError_t e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (rc == BLP_OK && e != cudaSuccess) rc = fail(BLP_ERR_CUDA, cudaGetErrorString(e));
    return rc;
}

}  // extern "C"

