// tmem_probe.cu -- microbenchmark: can tensor memory (TMEM) serve as a third
// on-chip tier for a row-per-lane tableau, next to registers and shared
// memory?  Each warp updates its rows' cells t <- t - f*r, NB batches of 8
// doubles (16 TMEM columns) per lane, through (a) tcgen05.ld/st and (b) LDS/STS.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/tmem_probe scripts/tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kWarps = 16;
constexpr int kCols = 128;          // TMEM columns per warp (4 warps share a lane quarter: 4 x 128 = 512)

__device__ __forceinline__ void tm_ld16(uint32_t a, uint32_t (&v)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(a));
}
__device__ __forceinline__ void tm_st16(uint32_t a, const uint32_t (&v)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                   "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
}

template <int MODE>  // 0: TMEM read+write, 1: TMEM read only, 2: smem read+write
__global__ void __launch_bounds__(kWarps * 32, 1) probe(double *sink, int iters, double f, double r) {
    __shared__ uint32_t taddr_s;
    extern __shared__ double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (MODE != 2) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                         ::"r"((unsigned)__cvta_generic_to_shared(&taddr_s)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    } else {
        __syncthreads();
    }
    const uint32_t base = (MODE != 2 ? taddr_s : 0u) + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(kCols * (warp >> 2));
    double acc = 0.0;
    constexpr int NB = kCols / 16;   // batches of 8 doubles
    // smem: per warp kCols/2 doubles per lane, column-major [c][lane] with stride 33
    double *col = sm + warp * (kCols / 2) * 33 + lane;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
        for (int b = 0; b < NB; ++b) {
            if (MODE == 2) {
                double t[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) t[k] = col[(b * 8 + k) * 33];
#pragma unroll
                for (int k = 0; k < 8; ++k) col[(b * 8 + k) * 33] = __dsub_rn(t[k], __dmul_rn(f, r));
            } else {
                uint32_t v[16];
                tm_ld16(base + 16 * b, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (MODE == 0) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        double t = __hiloint2double((int)v[2 * k + 1], (int)v[2 * k]);
                        t = __dsub_rn(t, __dmul_rn(f, r));
                        v[2 * k] = (uint32_t)__double2loint(t);
                        v[2 * k + 1] = (uint32_t)__double2hiint(t);
                    }
                    tm_st16(base + 16 * b, v);
                } else {
#pragma unroll
                    for (int k = 0; k < 8; ++k) acc += __hiloint2double((int)v[2 * k + 1], (int)v[2 * k]);
                }
            }
        }
        if (MODE == 0) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    if (acc == -1.0) sink[0] = acc;
    if (MODE != 2) {
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
    }
}

template <int MODE>
void run(const char *name, int sms, double *sink) {
    const int iters = 2000;
    const size_t smem = MODE == 2 ? (size_t)kWarps * (kCols / 2) * 33 * 8 : 0;
    cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<MODE><<<sms, kWarps * 32, smem>>>(sink, 10, 0.5, 0.25);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<MODE><<<sms, kWarps * 32, smem>>>(sink, iters, 0.5, 0.25);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const cudaError_t err = cudaGetLastError();
    const double bytes_per_sm = (double)iters * kWarps * 32 * (kCols / 2) * 8.0;   // bytes read per SM (writes equal for MODE 0/2)
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-22s %s  %.3f ms  read %.1f B/clk/SM  (%.2f TB/s chip read)\n", name, cudaGetErrorString(err), ms,
           bytes_per_sm / cyc, bytes_per_sm * sms / (ms * 1e-3) / 1e12);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *sink;
    cudaMalloc(&sink, 8);
    run<1>("tmem read", sms, sink);
    run<0>("tmem read+update+write", sms, sink);
    run<2>("smem read+update+write", sms, sink);
    return 0;
}
