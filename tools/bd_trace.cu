// Diagnostics: cross-CTA timeline of bd_reg_kernel steps (globaltimer, ns).
// Events per step: 0 reflect products done, 1 past the second CTA barrier,
// 2 E1 sent, 3 EN arrived, 4 (reducer) E1 arrived, 5 E2 sent, 6 E2 arrived.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTTSVD_BD_TRACE=480 -DTTSVD_BD_K0=200 -o tools/_var/bd_trace tools/bd_trace.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#include "../paper_2102_00104_b200/csrc/ttsvd_kernels.cuh"
#include "../paper_2102_00104_b200/csrc/jacobi_blk.cuh"
#include "../paper_2102_00104_b200/csrc/bidiag.cuh"
using namespace ttsvd_b200;

int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 512, n = m;
    std::mt19937_64 g(3);
    std::normal_distribution<double> nd;
    std::vector<double> A((size_t)n * m);
    for (auto& v : A) v = nd(g);
    double *dA, *ws;
    long long* prof;
    cudaMalloc(&dA, A.size() * 8);
    cudaMalloc(&ws, ((size_t)3 * m + 2 * (n + 1) + 16 * (size_t)n + 32 * 17) * 8);
    cudaMalloc(&prof, 16 * 8 * 8 * 8);
    cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(prof, 0, 16 * 8 * 8 * 8);
    BdArgs ba{dA, n, m, 32, ws, ws + m, ws + 2 * m, ws + 3 * m, prof};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(kBdThreads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaFuncSetAttribute(bd_reg_kernel<32, 16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (cudaLaunchKernelEx(&cfg, bd_reg_kernel<32, 16>, ba) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
        printf("failed\n");
        return 1;
    }
    std::vector<long long> p(16 * 64);
    cudaMemcpy(p.data(), prof, p.size() * 8, cudaMemcpyDeviceToHost);
    long long t0 = p[0];
    for (auto v : p)
        if (v && v < t0) t0 = v;
    for (int s = 0; s < 8; ++s) {
        printf("step +%d\n", s);
        for (int r = 0; r < 16; ++r) {
            printf("  cta %2d:", r);
            for (int e = 0; e < 7; ++e) {
                const long long v = p[(r * 8 + e) * 8 + s];
                if (v) printf(" e%d %6lld", e, v - t0);
                else printf(" e%d      -", e);
            }
            printf("\n");
        }
    }
    return 0;
}
