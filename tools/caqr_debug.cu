// Experiment (not in the product library; DESIGN.md §3 'measured and dropped'):
// the CAQR kernel of tools/caqr_experiment.cuh.  Diagnostics for caqr_kernel: per-stage wall time of the panel's slot-0 CTA
// (globaltimer marks, CAQR_PROF build) on a seeded Gaussian n x m matrix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/caqr_debug.cu -o tools/caqr_debug
//   ./tools/caqr_debug n m G
#define CAQR_PROF 1
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include "../paper_2102_00104_b200/csrc/ttsvd_kernels.cuh"
#include "caqr_experiment.cuh"
using namespace ttsvd_b200;

int main(int argc, char** argv) {
    const int64_t n = atoll(argv[1]);
    const int m = atoi(argv[2]), G = atoi(argv[3]);
    const int M = (m + 31) / 32 * 32, npan = M / 32;
    std::mt19937_64 eng(7);
    std::normal_distribution<double> nd;
    std::vector<double> hx((size_t)n * m);
    for (auto& v : hx) v = nd(eng);
    double *X, *A, *S, *R;
    long long* prof;
    cudaMalloc(&X, n * m * 8);
    cudaMalloc(&A, n * M * 8);
    cudaMalloc(&S, (size_t)(G + 16) * 1024 * 8);
    cudaMalloc(&R, (size_t)m * m * 8);
    cudaMalloc(&prof, npan * 24 * 8);
    cudaMemset(prof, 0, npan * 24 * 8);
    cudaMemcpyToSymbol(g_caqr_prof, &prof, sizeof(prof));
    cudaMemcpy(X, hx.data(), n * m * 8, cudaMemcpyHostToDevice);
    const size_t smem = caqr_smem_bytes();
    cudaFuncSetAttribute(caqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    CaqrArgs a{X, n, A, n, n, m, M, S, S + (size_t)G * 1024, R, m};
    void* args[] = {&a};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaLaunchCooperativeKernel((const void*)caqr_kernel, dim3(G), dim3(kCaqrThreads), args, smem, 0);
    cudaEventRecord(e0);
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)caqr_kernel, dim3(G), dim3(kCaqrThreads), args, smem, 0);
    cudaEventRecord(e1);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> t(npan * 24);
    cudaMemcpy(t.data(), prof, t.size() * 8, cudaMemcpyDeviceToHost);
    printf("%lld x %d, G %d: %s, %.3f ms\n", (long long)n, m, G, cudaGetErrorString(e), ms);
    const char* nm[5] = {"load", "qr", "formT", "apply", "R+sync"};
    for (int st = 0; st < 3; ++st) {
        double acc[5] = {0};
        for (int p = 0; p < npan; ++p)
            for (int k = 0; k < 5; ++k) {
                const long long a0 = t[p * 24 + st * 6 + k], a1 = t[p * 24 + st * 6 + k + 1];
                if (a0 && a1) acc[k] += (a1 - a0) * 1e-3;
            }
        printf("  stage %d:", st);
        for (int k = 0; k < 5; ++k) printf(" %s %.1f", nm[k], acc[k]);
        printf(" (us, summed over panels)\n");
    }
    return e == cudaSuccess ? 0 : 1;
}
