// Diagnostics: phase cycles of bd_reg_kernel (BD_MARK slots 0..6, CTA C-1
// thread 0) on an n x m work matrix like config 2's (rank 32 + 1e-8 noise).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/_var/bd_prof tools/bd_prof.cu
// Run:   tools/_var/bd_prof [m]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstring>
#include <cmath>
#include <random>
#include <cuda_runtime.h>
#ifndef BD_NOPROF
#define TTSVD_BD_PROF 1
#endif
#ifndef TTSVD_BD_PROF_TID
#define TTSVD_BD_PROF_TID 0
#endif
#include "../paper_2102_00104_b200/csrc/ttsvd_kernels.cuh"
#include "../paper_2102_00104_b200/csrc/jacobi_blk.cuh"
#include "../paper_2102_00104_b200/csrc/bidiag.cuh"
using namespace ttsvd_b200;

template <int CPC, int C>
float run(double* A, int n, int m, double* ws, long long* prof) {
    BdArgs ba{A, n, m, CPC, ws, ws + m, ws + 2 * m, ws + 3 * m, prof};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kBdThreads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaFuncSetAttribute(bd_reg_kernel<CPC, C>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, bd_reg_kernel<CPC, C>, ba);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        printf("launch failed: %s\n", cudaGetErrorString(err));
        exit(1);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 512, n = m;
    std::mt19937_64 g(3);
    std::normal_distribution<double> nd;
    std::vector<double> L((size_t)n * 32), Rm((size_t)32 * m), A((size_t)n * m);
    for (auto& v : L) v = nd(g);
    for (auto& v : Rm) v = nd(g);
    for (int j = 0; j < m; ++j)
        for (int i = 0; i < n; ++i) {
            double s = 0;
            for (int t = 0; t < 32; ++t) s += L[(size_t)t * n + i] * Rm[(size_t)j * 32 + t];
            A[(size_t)j * n + i] = s + 1e-8 * nd(g);
        }
    double *dA, *dA0, *ws;
    long long* prof;
    cudaMalloc(&dA, A.size() * 8);
    cudaMalloc(&dA0, A.size() * 8);
    cudaMalloc(&ws, ((size_t)3 * m + 2 * (n + 1) + 16 * (size_t)n + 32 * 17) * 8);
    cudaMalloc(&prof, 16 * 12 * 8);
    cudaMemcpy(dA0, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
    const int need = (m + 15) / 16;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(dA, dA0, A.size() * 8, cudaMemcpyDeviceToDevice);
        cudaMemset(prof, 0, 16 * 12 * 8);
        float ms = need <= 16 ? run<16, 16>(dA, n, m, ws, prof) : run<32, 16>(dA, n, m, ws, prof);
        cudaMemcpy(dA, dA0, A.size() * 8, cudaMemcpyDeviceToDevice);
        float ms0 = need <= 16 ? run<16, 16>(dA, n, m, ws, nullptr) : run<32, 16>(dA, n, m, ws, nullptr);
        {
            std::vector<double> de(2 * m);
            cudaMemcpy(de.data(), ws, 2 * m * 8, cudaMemcpyDeviceToHost);
            double cs = 0;
            unsigned long long hx = 0;
            for (int q = 0; q < 2 * m - 1; ++q) {
                cs += fabs(de[q]);
                unsigned long long b;
                memcpy(&b, &de[q], 8);
                hx = hx * 1000003ull ^ b;
            }
            printf("  d/e checksum %.17g hash %016llx\n", cs, hx);
        }
        long long p[16 * 12];
        cudaMemcpy(p, prof, sizeof(p), cudaMemcpyDeviceToHost);
        printf("m=%d: %.3f ms (unprofiled %.3f ms)\n", m, ms, ms0);
        if (rep < 2) continue;
        for (int r = 0; r < 16; ++r) {
            long long tot = 0;
            for (int q = 0; q < 12; ++q) tot += p[r * 12 + q];
            if (!tot) continue;
            printf("  cta %2d cycles/step:", r);
            for (int q = 0; q < 12; ++q) printf(" [%d] %4.0f", q, (double)p[r * 12 + q] / m);
            printf("  total %.0f\n", (double)tot / m);
        }
    }
    return 0;
}
