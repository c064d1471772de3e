// Diagnostics: phase cycles of gqr_kernel (CTA 0 thread 0, GqrArgs::prof)
// on config-2-like shapes.  Phases: [0] stage, [1] reflectors, [2]
// writeback+S+T, [3] W partial, [4] W reduce, [5] update, [6] per-reflector
// partials, [7] per-reflector barrier + sums + scalars.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/_var/gqr_prof tools/gqr_prof.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#include "../paper_2102_00104_b200/csrc/ttsvd_kernels.cuh"
#include "../paper_2102_00104_b200/csrc/tsqr_blk.cuh"
#include "../paper_2102_00104_b200/csrc/gqr.cuh"
using namespace ttsvd_b200;

template <int NT>
void run(int64_t n, int m, int G) {
    const int M = (m + 31) / 32 * 32;
    std::mt19937_64 g(5);
    std::normal_distribution<double> nd;
    std::vector<double> A((size_t)n * M);
    for (auto& v : A) v = nd(g);
    double *dA, *dA0, *pp;
    long long* prof;
    cudaMalloc(&dA, A.size() * 8);
    cudaMalloc(&dA0, A.size() * 8);
    cudaMemcpy(dA0, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
    const size_t np = (size_t)2 * G * 33 + (size_t)G * 1024 + (size_t)G * 32 * M;
    cudaMalloc(&pp, (np + 64 + (size_t)32 * M + 1024) * 8);
    cudaMalloc(&prof, 8 * 8);
    const int rows_max = (int)((n + G - 1) / G);
    const size_t smem = gqr_smem_bytes(rows_max, NT);
    cudaFuncSetAttribute(gqr_kernel<false, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(dA, dA0, A.size() * 8, cudaMemcpyDeviceToDevice);
        cudaMemset(prof, 0, 64);
        GqrArgs ga{dA, n, n, m, M, pp, pp + np, pp + np + 64, pp + np + 64 + (size_t)32 * M, rep == 2 ? prof : nullptr};
        void* args[] = {&ga};
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaError_t err = cudaLaunchCooperativeKernel((const void*)gqr_kernel<false, NT>, dim3(G), dim3(NT), args, smem, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (err != cudaSuccess) {
            printf("launch failed: %s\n", cudaGetErrorString(err));
            return;
        }
        long long p[8];
        cudaMemcpy(p, prof, 64, cudaMemcpyDeviceToHost);
        printf("n=%lld m=%d G=%d NT=%d: %.3f ms%s", (long long)n, m, G, NT, ms, rep == 2 ? "  per reflector:" : "\n");
        if (rep == 2) {
            const char* nm[8] = {"stage", "refl", "wb+S+T", "Wpart", "Wred", "update", "partials", "sync+sums+scal"};
            for (int q = 0; q < 8; ++q) printf(" %s %.0f", nm[q], (double)p[q] / m);
            printf("\n");
        }
    }
    cudaFree(dA);
    cudaFree(dA0);
    cudaFree(pp);
    cudaFree(prof);
}

int main() {
    run<256>(4096, 512, 64);
    run<512>(65536, 512, 148);
    run<256>(37888, 256, 148);
    run<256>(65536, 512, 256);
    return 0;
}
