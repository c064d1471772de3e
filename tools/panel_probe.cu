// Diagnostics: cycles per reflector of la_panel / la_build_t, one warp alone
// and with a competing warp on the same SM sub-partition.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2102_00104_b200/csrc/ttsvd_kernels.cuh"
#include "../paper_2102_00104_b200/csrc/tsqr_blk.cuh"
#include "../paper_2102_00104_b200/csrc/tsqr_la.cuh"
using namespace ttsvd_b200;
__global__ void probe(double* out, long long* cyc, int reps, int w2) {
    extern __shared__ __align__(16) double sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int me = (warp == 0) ? 0 : (warp == w2 ? 1 : -1);
    double* Bt = sm + (me > 0 ? 8192 : 0);
    double* Rp = Bt + 32 * kBlkLdb;
    double* Sm = Rp + 32 * kLaRld;
    double* Tm = Sm + 32 * kTld;
    double* tau = Tm + 32 * kLaTld;
    double* pv = tau + 32;
    if (me >= 0) {
        for (int e = lane; e < 32 * kBlkLdb; e += 32) Bt[e] = 0.001 * ((e * 7919) % 1000) - 0.5;
        for (int e = lane; e < 32 * kLaRld; e += 32) Rp[e] = (e % (kLaRld + 1) == 0) ? 3.0 : 0.01 * (e % 13);
    }
    __syncthreads();
    if (me < 0) return;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) la_panel(Bt, 0, Rp, tau, pv, Sm, lane);
    long long t1 = clock64();
    for (int r = 0; r < reps; ++r) la_build_t(Sm, tau, Tm, lane);
    long long t2 = clock64();
    if (lane == 0 && me == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
    out[lane] = Bt[lane] + Tm[lane];
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 4096); cudaMallocManaged(&c, 64);
    size_t smem = (8192 + 32 * kBlkLdb + 32 * kLaRld + 32 * kTld + 32 * kLaTld + 64) * 8;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int reps = 20;
    for (int w2 : {-1, 4, 1}) {
        for (int i = 0; i < 2; ++i) { probe<<<1, 256, smem>>>(o, c, reps, w2); cudaDeviceSynchronize(); }
        printf("second panel warp %2d: %.0f cyc/panel = %.0f cyc/reflector; build_t: %.0f cyc\n", w2, (double)c[0] / reps, (double)c[0] / reps / 32, (double)c[1] / reps);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
