#include <cstdio>
#include <cuda_runtime.h>
template <int KIND, int N>
__global__ void k(const uint4* p, long long* out, unsigned* sink) {
    const int lane = threadIdx.x;
    unsigned acc = 0;
    long long best = 1LL << 60;
    for (int rep = 0; rep < 20; ++rep) {
        uint4 w[N];
        long long t0 = clock64();
#pragma unroll
        for (int u = 0; u < N; ++u) {
            const uint4* a = p + (size_t)(u * 4 + rep * 64 * 4) * 32 + lane;
            if (KIND == 0) asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[u].x), "=r"(w[u].y), "=r"(w[u].z), "=r"(w[u].w) : "l"(a) : "memory");
            else if (KIND == 1) asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[u].x), "=r"(w[u].y), "=r"(w[u].z), "=r"(w[u].w) : "l"(a) : "memory");
            else if (KIND == 2) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[u].x), "=r"(w[u].y), "=r"(w[u].z), "=r"(w[u].w) : "l"(a) : "memory");
            else asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[u].x), "=r"(w[u].y), "=r"(w[u].z), "=r"(w[u].w) : "l"(a));
        }
        unsigned s = 0;
#pragma unroll
        for (int u = 0; u < N; ++u) s += w[u].x ^ w[u].y;
        acc += s;
        long long t1 = clock64();
        if (t1 - t0 < best) best = t1 - t0;
    }
    if (lane == 0) out[0] = best;
    sink[lane] = acc;
}
template <int KIND, int N> void run(const char* nm, uint4* p, long long* o, unsigned* s) {
    k<KIND, N><<<1, 32>>>(p, o, s); cudaDeviceSynchronize();
    printf("%s N=%d: %lld cycles\n", nm, N, o[0]);
}
int main() {
    uint4* p; long long* o; unsigned* s;
    cudaMalloc(&p, 64 << 20); cudaMemset(p, 1, 64 << 20); cudaMallocManaged(&o, 64); cudaMalloc(&s, 4096);
    run<0, 1>("volatile", p, o, s); run<0, 4>("volatile", p, o, s); run<0, 16>("volatile", p, o, s);
    run<1, 1>("relaxed.gpu", p, o, s); run<1, 16>("relaxed.gpu", p, o, s);
    run<2, 1>("cg+memclobber", p, o, s); run<2, 16>("cg+memclobber", p, o, s);
    run<3, 16>("cg", p, o, s);
}
