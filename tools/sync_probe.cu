// Diagnostics: cost of grid.sync (cooperative launch, 1 CTA per SM) and of a
// flag-based all-CTA barrier.
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void gsync(int iters, long long* out) {
    cg::grid_group g = cg::this_grid();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) g.sync();
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}
__global__ void flagsync(int iters, unsigned* ctr, long long* out) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(ctr, 1u);
            const unsigned target = (unsigned)(i + 1) * gridDim.x;
            while (*(volatile unsigned*)ctr < target) {}
            __threadfence();
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}
int main() {
    long long* o; unsigned* c;
    cudaMallocManaged(&o, 64); cudaMalloc(&c, 64);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int iters = 2000;
    for (int threads : {256, 512}) {
        void* args[] = {&iters, &o};
        cudaLaunchCooperativeKernel((void*)gsync, sms, threads, args, 0, 0);
        cudaDeviceSynchronize();
        cudaLaunchCooperativeKernel((void*)gsync, sms, threads, args, 0, 0);
        cudaDeviceSynchronize();
        printf("grid.sync %d CTAs x %d: %.0f cycles = %.2f us\n", sms, threads, (double)o[0] / iters, (double)o[0] / iters / 1965.0);
        cudaMemset(c, 0, 4);
        void* a2[] = {&iters, &c, &o};
        cudaLaunchCooperativeKernel((void*)flagsync, sms, threads, a2, 0, 0);
        cudaDeviceSynchronize();
        printf("flag barrier %d CTAs x %d: %.0f cycles = %.2f us (%s)\n", sms, threads, (double)o[0] / iters, (double)o[0] / iters / 1965.0, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
