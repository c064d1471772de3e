// Diagnostics: latency of bj_solve (one warp) on a random 8x8 Gram.
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
#include "../paper_2102_00104_b200/csrc/tsqr_blk.cuh"
#include "../paper_2102_00104_b200/csrc/jacobi_blk.cuh"
using namespace ttsvd_b200;
__global__ void probe(long long* cyc, double* out, int reps) {
    __shared__ double gpart[kBjWorkers][64];
    __shared__ double G[72], Q[72];
    const int lane = threadIdx.x;
    for (int w = 0; w < kBjWorkers; ++w)
        for (int e = lane; e < 64; e += 32) {
            const int i = e >> 3, j = e & 7;
            gpart[w][e] = (i == j ? 1.0 + 0.1 * i : 0.01 * ((i * 7 + j * 3) % 5)) + (i == j ? 0 : 0.001 * w);
        }
    __syncwarp();
    long long t0 = clock64();
    int any = 0;
    for (int r = 0; r < reps; ++r) any += bj_solve(gpart, G, Q, 0, 1, false, lane);
    long long t1 = clock64();
    if (lane == 0) cyc[0] = (t1 - t0) / reps;
    out[lane] = G[lane] + Q[lane] + any;
}
int main() {
    long long* c; double* o;
    cudaMallocManaged(&c, 64); cudaMalloc(&o, 4096);
    for (int i = 0; i < 2; ++i) { probe<<<1, 32>>>(c, o, 50); cudaDeviceSynchronize(); }
    printf("bj_solve (4 sub-rounds): %lld cycles  (%s)\n", c[0], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
