// Diagnostics: cluster.sync and DSMEM round-trip latency (16-CTA cluster).
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void __cluster_dims__(16, 1, 1) k16(int iters, long long* out) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double buf[64];
    buf[threadIdx.x & 63] = threadIdx.x;
    cl.sync();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) cl.sync();
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < iters; ++i) {
        const double* rb = cl.map_shared_rank(buf, (cl.block_rank() + 1 + i) % 16);
        s += *(volatile const double*)(rb + (threadIdx.x & 63));
    }
    long long t2 = clock64();
    cl.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = (t1 - t0) / iters; out[1] = (t2 - t1) / iters; out[2] = (long long)s; }
}
int main() {
    long long* o; cudaMallocManaged(&o, 64);
    cudaFuncSetAttribute(k16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int r = 0; r < 2; ++r) { k16<<<16, 256>>>(1000, o); cudaDeviceSynchronize(); }
    printf("cluster.sync (16 CTAs x 256): %lld cycles; dependent DSMEM load: %lld cycles (%s)\n", o[0], o[1], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
