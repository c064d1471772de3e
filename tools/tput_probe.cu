// Diagnostics: per-SM throughput of the bidiagonalisation's instruction mix
// with 512 threads (16 warps) on one SM: independent DFMA, 64-bit shuffles,
// 64-bit selects, broadcast LDS.64.  Prints cycles per warp-instruction per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_var/tput_probe tools/tput_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) k(double* out, long long* cyc, double y, int n) {
    __shared__ double sm[64];
    if (threadIdx.x < 64) sm[threadIdx.x] = threadIdx.x * 0.5;
    __syncthreads();
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
    const bool up = threadIdx.x & 1;
    long long t0, t1;
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fma(a[j], y, 1e-9);
    __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = __shfl_xor_sync(0xffffffffu, a[j], 1 + j % 4);
    __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
            const double s = up ? a[j] : a[j + 1];
            const double kk = up ? a[j + 1] : a[j];
            a[j] = s;
            a[j + 1] = kk;
        }
    __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) cyc[2] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] += sm[(i + j) & 63];
    __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) cyc[3] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = a[j] * y;
    __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) cyc[4] = t1 - t0;
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
    out[threadIdx.x] = s;
}

int main() {
    double* o;
    long long* c;
    cudaMalloc(&o, 1024 * 8);
    cudaMallocManaged(&c, 16 * 8);
    const int n = 2000;
    for (int rep = 0; rep < 2; ++rep) {
        k<<<1, 512>>>(o, c, 1.0000001, n);
        cudaDeviceSynchronize();
    }
    const double wi = 16.0 * 8 * n;  // warp-instructions per SM per test
    printf("DFMA      %.2f cyc per warp-instr per SM\n", c[0] / wi);
    printf("SHFL64    %.2f cyc per 64-bit warp-shuffle per SM\n", c[1] / wi);
    printf("SEL64 x2  %.2f cyc per swap pair-element per SM\n", c[2] / wi);
    printf("LDS64+ADD %.2f cyc per (broadcast LDS.64 + DADD) per SM\n", c[3] / wi);
    printf("DMUL      %.2f cyc per warp-instr per SM\n", c[4] / wi);
    return 0;
}
