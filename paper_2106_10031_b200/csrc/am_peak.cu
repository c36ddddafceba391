// am_peak.cu -- fp64 tensor-core (DMMA) peak microbenchmark.
// MEASURED_PEAKS.json carries HBM and bf16 peaks only; the composition kernel
// is fp64 DMMA-bound, so bench.py measures its roofline denominator with this
// register-resident loop of independent mma.sync m16n8k4 .f64 (8 accumulator
// chains per warp, 8 warps per CTA, 4 CTAs per SM).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/am_b200.h"

__global__ void k_dmma_peak(double* out, int iters) {
    double a0 = 1.0 + threadIdx.x * 1e-9, a1 = 0.5, b0 = 1e-3;
    double acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = 0.0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                         : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                         : "d"(a0), "d"(a1), "d"(b0));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
    if (s == 12345.678) out[0] = s;
}

// DFMA (CUDA-core fp64) peak for comparison
__global__ void k_dfma_peak(double* out, int iters) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = fma(x[i], 0.999999, 1e-7);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 12345.678) out[0] = s;
}

extern "C" int am_bench_fp64_peak(int device, double* h_out2) {
    if (cudaSetDevice(device) != cudaSuccess) return AM_ERR_NO_DEVICE;
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, device);
    double* d = nullptr;
    cudaMalloc(&d, 8);
    int blocks = p.multiProcessorCount * 4, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        k_dmma_peak<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
    }
    // flops: per mma m16n8k4 = 2*16*8*4 = 1024 per warp
    double warps = (double)blocks * threads / 32;
    h_out2[0] = warps * iters * 8 * 1024.0 / (best * 1e-3) / 1e12;
    best = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        k_dfma_peak<<<blocks, threads>>>(d, iters * 8);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
    }
    h_out2[1] = (double)blocks * threads * iters * 8 * 8 * 2.0 / (best * 1e-3) / 1e12;
    cudaFree(d);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return cudaGetLastError() == cudaSuccess ? AM_OK : AM_ERR_CUDA;
}
