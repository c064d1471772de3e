// Diagnostics: per-phase cycles of tsqr_t128_kernel<256> (CTA 0, thread 0;
// built with -DTTSVD_T2_PROF) on an n x M matrix.  Phases per panel
// iteration: [5] next panel's columns scratch -> smem (+ barrier), [6] R diag
// fetch wait, [1] wait for phase A, [2] panel chain, [3] T build, [4] wait for
// the trailing update; [0] tile load + panel 0 + its T.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DTTSVD_T2_PROF -o tools/_var/t2_prof tools/t2_prof.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_2102_00104_b200/csrc/ttsvd_kernels.cuh"
#include "../paper_2102_00104_b200/csrc/tsqr_blk.cuh"
#include "../paper_2102_00104_b200/csrc/tsqr_la.cuh"
#include "../paper_2102_00104_b200/csrc/tsqr_t128.cuh"
using namespace ttsvd_b200;
__global__ void fill(double* x, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull;
        z ^= z >> 29; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 32;
        x[i] = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    }
}
int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : (1 << 20);
    const int M = argc > 2 ? atoi(argv[2]) : 256;
    const int G = 148;
    double *X, *R, *S; long long* prof;
    cudaMalloc(&X, (size_t)n * M * 8);
    cudaMalloc(&R, (size_t)G * blk_rsize(M) * 8);
    cudaMalloc(&S, (size_t)G * 256 * M * 8);
    cudaMalloc(&prof, G * 64);
    fill<<<1184, 256>>>(X, (size_t)n * M);
    cudaFuncSetAttribute(tsqr_t128_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t2_smem_bytes(256));
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(prof, 0, G * 64);
        T2Args ta{X, n, n, R, S, M, M, prof, ColSplit{0, 0}};
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        tsqr_t128_kernel<256><<<G, kT2Threads, t2_smem_bytes(256)>>>(ta);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long p[8]; cudaMemcpy(p, prof, 64, cudaMemcpyDeviceToHost);
        const double tiles = (double)n / G / 256, pans = tiles * (M / 32 - 1);
        printf("n=%lld M=%d: %.3f ms (%s); per tile: load+panel0+T %.0f; per later panel: stage %.0f rdiag %.0f waitA %.0f chain %.0f T %.0f wait-update %.0f\n",
               (long long)n, M, ms, cudaGetErrorString(cudaGetLastError()), p[0] / tiles, p[5] / pans, p[6] / pans, p[1] / pans, p[2] / pans, p[3] / pans, p[4] / pans);
    }
    return 0;
}
