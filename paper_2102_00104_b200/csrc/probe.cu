// Bench-only FP64 peak probe (not part of the product ABI): the roofline's
// FP64 denominator is not in MEASURED_PEAKS.json, so bench.py measures it on
// the box — a DFMA loop and a DMMA (mma.sync m8n8k4 f64) loop, best of both.
#include <cuda_runtime.h>
#include <cstdint>

__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

__global__ void __launch_bounds__(256) dmma_loop(double* out, int iters, double a, double b) {
    double acc[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-3;
    double fa = a + threadIdx.x, fb = b - threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(fa), "d"(fb));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) out[0] = s;
}

extern "C" int ttsvd_probe_fp64(int device, double* dfma_tflops, double* dmma_tflops) {
    cudaSetDevice(device);
    cudaDeviceProp p{};
    cudaGetDeviceProperties(&p, device);
    double* out = nullptr;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 20000;
    float best_f = 1e30f, best_m = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        float t = 0;
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&t, e0, e1);
        if (rep && t < best_f) best_f = t;
        cudaEventRecord(e0);
        dmma_loop<<<blocks, threads>>>(out, iters / 4, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&t, e0, e1);
        if (rep && t < best_m) best_m = t;
    }
    const double fl_f = 2.0 * 8.0 * iters * (double)blocks * threads;
    const double fl_m = 2.0 * 256.0 * 4.0 * (iters / 4) * (double)blocks * (threads / 32);
    *dfma_tflops = fl_f / (best_f * 1e-3) / 1e12;
    *dmma_tflops = fl_m / (best_m * 1e-3) / 1e12;
    cudaFree(out);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
