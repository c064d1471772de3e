// Diagnostics: time tsqr_gt_kernel variants (lanes per stream P, rows per
// fold U, CTAs per SM MB, stages ST) on a 2^24 x 16 and a 2^23 x 32 matrix.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/gt_probe tools/gt_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2102_00104_b200/csrc/ttsvd_kernels.cuh"
namespace ttsvd_b200 { constexpr unsigned kFull = 0xffffffffu; }
#include "../paper_2102_00104_b200/csrc/tsqr_gt.cuh"
using namespace ttsvd_b200;
__global__ void fill(double* x, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull;
        z ^= z >> 29; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 32;
        x[i] = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    }
}
template <int M, int P, int U, int MB, int ST>
void run(const double* X, int64_t n, int m, double* out) {
    constexpr int G = 32 / P, SR = G * U;
    auto fn = tsqr_gt_kernel<M, P, U, MB, ST>;
    const size_t smem = gt_smem_bytes<M, P, U, ST>();
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPtThreads, smem);
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, fn);
    const int64_t ctas = 148 * (per_sm > 0 ? per_sm : 1);
    const int64_t T = ctas * (kPtThreads / 32) * G;
    GsArgs ga{X, n, n, m, T, out, T * m};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    fn<<<(unsigned)ctas, kPtThreads, smem>>>(ga);
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) fn<<<(unsigned)ctas, kPtThreads, smem>>>(ga);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("M=%d P=%d U=%d MB=%d ST=%d: regs %d local %zu smem %zu KB, %d CTA/SM, %.3f ms (%s) SR=%d\n", M, P, U, MB, ST,
           fa.numRegs, fa.localSizeBytes, smem >> 10, per_sm, ms / 3, cudaGetErrorString(cudaGetLastError()), SR);
}
int main() {
    const int64_t n16 = 1 << 24, n32 = 1 << 23;
    double *X, *out;
    cudaMalloc(&X, (size_t)n16 * 16 * 8);
    cudaMalloc(&out, (size_t)148 * 2 * 8 * 32 * 32 * 32 * 8);
    fill<<<1184, 256>>>(X, (size_t)n16 * 16);
    run<16, 4, 8, 1, 2>(X, n16, 16, out);
    run<32, 8, 8, 1, 2>(X, n32, 32, out);
    return 0;
}
