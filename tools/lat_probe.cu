// Latency probe (diagnostics): dependent chains of FP64 / shuffle ops in one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a0, int n) {
    double x = a0 + threadIdx.x * 1e-3, y = 1.0000001;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
    t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + 1e-9;
    t1 = clock64(); if (threadIdx.x == 0) cyc[1] = t1 - t0;
    // 64-bit shuffle xor chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-12;
    t1 = clock64(); if (threadIdx.x == 0) cyc[2] = t1 - t0;
    // rsqrt chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = rsqrt(x + 1.0);
    t1 = clock64(); if (threadIdx.x == 0) cyc[3] = t1 - t0;
    // __drcp_rn chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __drcp_rn(x + 1.0);
    t1 = clock64(); if (threadIdx.x == 0) cyc[4] = t1 - t0;
    // sqrt chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
    t1 = clock64(); if (threadIdx.x == 0) cyc[5] = t1 - t0;
    // select chain (64-bit FSEL pair)
    const bool b = threadIdx.x & 1;
    double z = x * 0.5;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { double t = b ? x : z; z = x; x = t + 0.0; }
    t1 = clock64(); if (threadIdx.x == 0) cyc[6] = t1 - t0;
    // independent DFMA throughput for one warp (8 chains)
    double a[8];
    for (int j = 0; j < 8; ++j) a[j] = x + j;
    t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fma(a[j], y, 1e-9);
    t1 = clock64(); if (threadIdx.x == 0) cyc[7] = t1 - t0;
    double s = 0; for (int j = 0; j < 8; ++j) s += a[j];
    // independent shuffle throughput (8 chains)
    t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = __shfl_xor_sync(0xffffffffu, a[j], 1 + j % 4);
    t1 = clock64(); if (threadIdx.x == 0) cyc[8] = t1 - t0;
    for (int j = 0; j < 8; ++j) s += a[j];
    out[threadIdx.x] = x + s + z;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 16 * 8);
    const int n = 1000;
    for (int rep = 0; rep < 2; ++rep) { k<<<1, 32>>>(o, c, 1.5, n); cudaDeviceSynchronize(); }
    const char* nm[] = {"dfma", "dadd", "shfl64+dadd", "rsqrt64", "drcp_rn", "dsqrt", "fsel64 swap+dadd", "8x dfma (per iter)", "8x shfl64 (per iter)"};
    for (int i = 0; i < 9; ++i) printf("%-22s %.1f cyc/iter\n", nm[i], (double)c[i] / n);
    return 0;
}
