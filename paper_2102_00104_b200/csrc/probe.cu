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

// the sm_90+ f64 shapes: ptxas lowers them to several DMMA.8x8x4 (SASS),
// so they cannot beat m8n8k4; measured to confirm
template <int K>
__global__ void __launch_bounds__(256) dmma16_loop(double* out, int iters, double a, double b) {
    double acc[2][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[i][e] = threadIdx.x * 1e-3 + e;
    const double fa = a + threadIdx.x, fb = b - threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            if constexpr (K == 4)
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                             : "d"(fa), "d"(fa * 0.5), "d"(fb));
            else if constexpr (K == 8)
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                             : "d"(fa), "d"(fa * 0.5), "d"(fa * 0.25), "d"(fa * 0.125), "d"(fb), "d"(fb * 0.5));
            else
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                             : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                             : "d"(fa), "d"(fa * 0.5), "d"(fa * 0.25), "d"(fa * 0.125), "d"(fa * 2), "d"(fa * 3),
                               "d"(fa * 4), "d"(fa * 5), "d"(fb), "d"(fb * 0.5), "d"(fb * 0.25), "d"(fb * 2));
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) s += acc[i][e];
    if (s == 12345.678) out[0] = s;
}

// TF/s of mma.sync m16n8k4 / m16n8k8 / m16n8k16 f64 (bench.py records them
// beside the m8n8k4 figure)
extern "C" int ttsvd_probe_fp64_shapes(int device, double* k4, double* k8, double* k16) {
    cudaSetDevice(device);
    cudaDeviceProp p{};
    cudaGetDeviceProperties(&p, device);
    double* out = nullptr;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = p.multiProcessorCount * 8, threads = 256;
    double* res[3] = {k4, k8, k16};
    for (int v = 0; v < 3; ++v) {
        const int K = 4 << v, iters = 20000 / K;
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            float t = 0;
            cudaEventRecord(e0);
            if (v == 0) dmma16_loop<4><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            else if (v == 1) dmma16_loop<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            else dmma16_loop<16><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&t, e0, e1);
            if (rep && t < best) best = t;
        }
        const double fl = 2.0 * 16 * 8 * K * 2.0 * iters * (double)blocks * (threads / 32);
        *res[v] = fl / (best * 1e-3) / 1e12;
    }
    cudaFree(out);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
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
