// Diagnostics: cycles per reflector of t2_panel (four panel warps, 128-row
// tile), alone and next to 8 warps issuing DMMA with shared-memory operands
// (the update warps' load on the SM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/t2panel_probe tools/t2panel_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2102_00104_b200/csrc/ttsvd_kernels.cuh"
#include "../paper_2102_00104_b200/csrc/tsqr_blk.cuh"
#include "../paper_2102_00104_b200/csrc/tsqr_la.cuh"
#include "../paper_2102_00104_b200/csrc/tsqr_t128.cuh"
using namespace ttsvd_b200;
template <int PW>
__global__ void __launch_bounds__(384, 1) probe(double* out, long long* cyc, int reps, int busy) {
    constexpr int Pld = 32 * PW + 4;
    extern __shared__ __align__(16) double sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* Pb = sm;
    double* Rp = Pb + 2 * 32 * Pld;
    double* Sm = Rp + 32 * kLaRld;
    double* Tm0 = Sm + 32 * kTld;
    double* tau = Tm0 + 2 * 32 * kLaTld;
    double* pvall = tau + 32;
    double* dpart = pvall + PW * 32;
    for (int e = threadIdx.x; e < 2 * 32 * Pld; e += blockDim.x) Pb[e] = 0.001 * ((e * 7919) % 1000) - 0.5;
    for (int e = threadIdx.x; e < 32 * kLaRld; e += blockDim.x) Rp[e] = (e % (kLaRld + 1) == 0) ? 3.0 : 0.01 * (e % 13);
    __syncthreads();
    volatile __shared__ int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    if (warp < PW) {
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) t2_panel<PW>(Pb, Rp, tau, pvall, dpart, Sm, warp, lane);
        long long t1 = clock64();
        if (lane == 0 && warp == 0) cyc[0] = t1 - t0;
        if (threadIdx.x == 0) stop = 1;
    } else if (busy) {
        double acc[4][2] = {};
        const double* V = Pb + 32 * Pld;
        int it = 0;
        while (!stop) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
#pragma unroll
                for (int u = 0; u < 4; ++u) dmma884(acc[u], V[(4 * kk + (lane & 3)) * Pld + 8 * u + (lane >> 2) + (it & 7)], 1.0001);
            ++it;
        }
        if (acc[0][0] == 12345.0) out[0] = acc[1][1];
    }
}
template <int PW>
void run(double* o, long long* c) {
    size_t smem = t2_smem_bytes(32 * PW);
    cudaFuncSetAttribute(probe<PW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int reps = 20;
    for (int busy : {0, 1}) {
        for (int i = 0; i < 2; ++i) { probe<PW><<<1, 384, smem>>>(o, c, reps, busy); cudaDeviceSynchronize(); }
        printf("PW=%d (%d rows) update warps busy=%d: %.0f cyc/panel = %.0f cyc/reflector\n", PW, 32 * PW, busy,
               (double)c[0] / reps, (double)c[0] / reps / 32);
    }
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 4096); cudaMallocManaged(&c, 64);
    run<4>(o, c);
    run<6>(o, c);
    run<8>(o, c);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
