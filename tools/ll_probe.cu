// Diagnostics: latency of an all-CTA reduction of 32 doubles per CTA through
// LL records (lo, flag, hi, flag) in global memory, one CTA per SM.
//   mode 0: flat      — every CTA polls all G records
//   mode 1: two-level — groups of 16 publish to a leader, every CTA polls the
//                       group totals
//   mode 2: grid.sync + plain stores/loads (reference point)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ll_probe tools/ll_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

template <int VOL>
__device__ __forceinline__ void st4(uint4* p, double v, unsigned f) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    if (VOL)
        asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"((unsigned)b), "r"(f),
                     "r"((unsigned)(b >> 32)), "r"(f)
                     : "memory");
    else
        asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"((unsigned)b), "r"(f),
                     "r"((unsigned)(b >> 32)), "r"(f)
                     : "memory");
}
template <int VOL>
__device__ __forceinline__ uint4 ld4(const uint4* p) {
    uint4 r;
    if (VOL == 2)
        asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                     : "l"(p)
                     : "memory");
    else if (VOL == 1)
        asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                     : "l"(p)
                     : "memory");
    else
        asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                     : "l"(p)
                     : "memory");
    return r;
}
__device__ __forceinline__ double val(uint4 r) {
    return __longlong_as_double((long long)(((unsigned long long)r.z << 32) | r.x));
}

template <int MODE, int VOL>
__global__ void probe(int iters, uint4* ll, double* plain, long long* out, double* sink) {
    cg::grid_group grid = cg::this_grid();
    const int G = gridDim.x, c = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int NG = (G + 15) / 16;
    __shared__ double sh[32];
    double acc = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const unsigned flag = 1000u + it;
        const int buf = it & 1;
        const double mine = (double)(c + 1) * (lane + 1) + acc * 1e-30;
        double tot = 0.0;
        if (MODE == 2) {
            if (warp == 0) plain[(buf * G + c) * 32 + lane] = mine;
            grid.sync();
            if (warp == 0) {
                double s = 0.0;
                for (int q = 0; q < G; q += 4) {
                    double v0 = __ldcg(&plain[(buf * G + q) * 32 + lane]);
                    double v1 = q + 1 < G ? __ldcg(&plain[(buf * G + q + 1) * 32 + lane]) : 0.0;
                    double v2 = q + 2 < G ? __ldcg(&plain[(buf * G + q + 2) * 32 + lane]) : 0.0;
                    double v3 = q + 3 < G ? __ldcg(&plain[(buf * G + q + 3) * 32 + lane]) : 0.0;
                    s += (v0 + v1) + (v2 + v3);
                }
                tot = s;
            }
        } else if (MODE == 0) {
            uint4* rec = ll + (size_t)buf * G * 32;
            if (warp == 0) st4<VOL>(rec + c * 32 + lane, mine, flag);
            if (warp == 0) {
                double s = 0.0;
                for (int q0 = 0; q0 < G; q0 += 16) {
                    uint4 w[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        if (q0 + u < G) w[u] = ld4<VOL>(rec + (q0 + u) * 32 + lane);
                    for (;;) {
                        bool ok = true;
#pragma unroll
                        for (int u = 0; u < 16; ++u)
                            if (q0 + u < G && (w[u].y != flag || w[u].w != flag)) {
                                ok = false;
                                w[u] = ld4<VOL>(rec + (q0 + u) * 32 + lane);
                            }
                        if (__all_sync(0xffffffffu, ok)) break;
                    }
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        if (q0 + u < G) s += val(w[u]);
                }
                tot = s;
            }
        } else if (MODE == 6 || MODE == 7) {
            // flat, records of 8 lanes (one 128-byte line) — MODE 7: records
            // packed densely (8 records per 1 KB) instead of 512-byte strides
            const int RS = (MODE == 6) ? 32 : 8;
            uint4* rec = ll + (size_t)buf * G * RS;
            if (warp == 0 && lane < 8) st4<VOL>(rec + c * RS + lane, mine, flag);
            if (warp == 0) {
                double s = 0.0;
                if (lane < 8) {
                    for (int q0 = 0; q0 < G; q0 += 16) {
                        uint4 w[16];
#pragma unroll
                        for (int u = 0; u < 16; ++u)
                            if (q0 + u < G) w[u] = ld4<VOL>(rec + (q0 + u) * RS + lane);
                        for (;;) {
                            bool ok = true;
#pragma unroll
                            for (int u = 0; u < 16; ++u)
                                if (q0 + u < G && (w[u].y != flag || w[u].w != flag)) {
                                    ok = false;
                                    w[u] = ld4<VOL>(rec + (q0 + u) * RS + lane);
                                }
                            if (ok) break;
                        }
#pragma unroll
                        for (int u = 0; u < 16; ++u)
                            if (q0 + u < G) s += val(w[u]);
                    }
                }
                tot = s;
            }
        } else if (MODE == 8) {
            // push-based three hops, every line read by exactly one CTA:
            // member -> leader inbox; leader -> every leader's inbox; leader ->
            // every member's inbox
            uint4* in1 = ll + (size_t)buf * G * 16 * 32;                    // [c][16][32]
            uint4* in2 = ll + (size_t)2 * G * 16 * 32 + (size_t)buf * G * 10 * 32;  // [c][10][32]
            uint4* in3 = ll + (size_t)2 * G * 26 * 32 + (size_t)buf * G * 32;       // [c][32]
            if (warp == 0) {
                const int grp = c / 16, first = grp * 16, cnt = min(16, G - first);
                if (c != first) {
                    st4<VOL>(in1 + ((size_t)first * 16 + (c - first)) * 32 + lane, mine, flag);
                    uint4 w = ld4<VOL>(in3 + (size_t)c * 32 + lane);
                    while (!__all_sync(0xffffffffu, w.y == flag && w.w == flag)) w = ld4<VOL>(in3 + (size_t)c * 32 + lane);
                    tot = val(w);
                } else {
                    double gs = mine;
                    uint4 w[16];
#pragma unroll
                    for (int u = 1; u < 16; ++u)
                        if (u < cnt) w[u] = ld4<VOL>(in1 + ((size_t)c * 16 + u) * 32 + lane);
                    for (;;) {
                        bool ok = true;
#pragma unroll
                        for (int u = 1; u < 16; ++u)
                            if (u < cnt && (w[u].y != flag || w[u].w != flag)) {
                                ok = false;
                                w[u] = ld4<VOL>(in1 + ((size_t)c * 16 + u) * 32 + lane);
                            }
                        if (__all_sync(0xffffffffu, ok)) break;
                    }
#pragma unroll
                    for (int u = 1; u < 16; ++u)
                        if (u < cnt) gs += val(w[u]);
                    for (int l = 0; l < NG; ++l) st4<VOL>(in2 + ((size_t)(l * 16) * 10 + grp) * 32 + lane, gs, flag);
                    uint4 x[10];
#pragma unroll
                    for (int u = 0; u < 10; ++u)
                        if (u < NG) x[u] = ld4<VOL>(in2 + ((size_t)c * 10 + u) * 32 + lane);
                    for (;;) {
                        bool ok = true;
#pragma unroll
                        for (int u = 0; u < 10; ++u)
                            if (u < NG && (x[u].y != flag || x[u].w != flag)) {
                                ok = false;
                                x[u] = ld4<VOL>(in2 + ((size_t)c * 10 + u) * 32 + lane);
                            }
                        if (__all_sync(0xffffffffu, ok)) break;
                    }
                    double t = 0.0;
#pragma unroll
                    for (int u = 0; u < 10; ++u)
                        if (u < NG) t += val(x[u]);
                    for (int u = 1; u < cnt; ++u) st4<VOL>(in3 + (size_t)(first + u) * 32 + lane, t, flag);
                    tot = t;
                }
            }
        } else if (MODE == 4) {
            // flag words + plain data: writer st data, st.release flag; reader
            // lane polls ld.acquire flag, then the warp loads the data
            double* d1 = plain + (size_t)buf * G * 32;
            double* d2 = plain + (size_t)2 * G * 32 + (size_t)buf * NG * 32;
            unsigned* f1 = reinterpret_cast<unsigned*>(ll) + (size_t)buf * 256;
            unsigned* f2 = reinterpret_cast<unsigned*>(ll) + 512 + (size_t)buf * 64;
            if (warp == 0) {
                const int grp = c / 16, first = grp * 16;
                double s = mine;
                if (c != first) {
                    d1[c * 32 + lane] = mine;
                    __syncwarp();
                    if (lane == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f1 + c), "r"(flag) : "memory");
                } else {
                    const int cnt = min(16, G - first);
                    if (lane > 0 && lane < cnt) {
                        unsigned f;
                        do {
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(f1 + first + lane) : "memory");
                        } while (f != flag);
                    }
                    __syncwarp();
                    double w[16];
#pragma unroll
                    for (int u = 1; u < 16; ++u)
                        if (u < cnt) w[u] = __ldcg(&d1[(first + u) * 32 + lane]);
#pragma unroll
                    for (int u = 1; u < 16; ++u)
                        if (u < cnt) s += w[u];
                    d2[grp * 32 + lane] = s;
                    __syncwarp();
                    if (lane == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f2 + grp), "r"(flag) : "memory");
                }
                if (lane < NG) {
                    unsigned f;
                    do {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(f2 + lane) : "memory");
                    } while (f != flag);
                }
                __syncwarp();
                double w[10];
#pragma unroll
                for (int u = 0; u < 10; ++u)
                    if (u < NG) w[u] = __ldcg(&d2[u * 32 + lane]);
                double t = 0.0;
#pragma unroll
                for (int u = 0; u < 10; ++u)
                    if (u < NG) t += w[u];
                tot = t;
            }
        } else if (MODE == 5) {
            // ping-pong between CTA 0 and CTA 1 (one LL word), others idle
            if (warp == 0 && lane == 0 && c < 2) {
                uint4* slot = ll + (size_t)c * 32;        // written by c
                uint4* peer = ll + (size_t)(1 - c) * 32;  // read by c
                if (c == 0) {
                    st4<VOL>(slot, mine, flag);
                    uint4 w;
                    do { w = ld4<VOL>(peer); } while (w.y != flag || w.w != flag);
                    tot = val(w);
                } else {
                    uint4 w;
                    do { w = ld4<VOL>(peer); } while (w.y != flag || w.w != flag);
                    st4<VOL>(slot, val(w), flag);
                    tot = val(w);
                }
            }
        } else {
            uint4* l1 = ll + (size_t)buf * G * 32;
            uint4* l2 = ll + (size_t)2 * G * 32 + (size_t)buf * NG * 32;
            if (warp == 0) {
                const int grp = c / 16, first = grp * 16;
                double s = mine;
                if (c != first) {
                    st4<VOL>(l1 + c * 32 + lane, mine, flag);
                } else {
                    const int cnt = min(16, G - first);
                    uint4 w[16];
#pragma unroll
                    for (int u = 1; u < 16; ++u)
                        if (u < cnt) w[u] = ld4<VOL>(l1 + (first + u) * 32 + lane);
                    for (;;) {
                        bool ok = true;
#pragma unroll
                        for (int u = 1; u < 16; ++u)
                            if (u < cnt && (w[u].y != flag || w[u].w != flag)) {
                                ok = false;
                                w[u] = ld4<VOL>(l1 + (first + u) * 32 + lane);
                            }
                        if (__all_sync(0xffffffffu, ok)) break;
                        if (MODE == 3) __nanosleep(40);
                    }
#pragma unroll
                    for (int u = 1; u < 16; ++u)
                        if (u < cnt) s += val(w[u]);
                    st4<VOL>(l2 + grp * 32 + lane, s, flag);
                }
                uint4 w[10];
#pragma unroll
                for (int u = 0; u < 10; ++u)
                    if (u < NG) w[u] = ld4<VOL>(l2 + u * 32 + lane);
                for (;;) {
                    bool ok = true;
#pragma unroll
                    for (int u = 0; u < 10; ++u)
                        if (u < NG && (w[u].y != flag || w[u].w != flag)) {
                            ok = false;
                            w[u] = ld4<VOL>(l2 + u * 32 + lane);
                        }
                    if (__all_sync(0xffffffffu, ok)) break;
                    if (MODE == 3) __nanosleep(40);
                }
                double t = 0.0;
#pragma unroll
                for (int u = 0; u < 10; ++u)
                    if (u < NG) t += val(w[u]);
                tot = t;
            }
        }
        if (warp == 0) sh[lane] = tot;
        __syncthreads();
        acc += sh[(lane + it) & 31];
        __syncthreads();
    }
    long long t1 = clock64();
    if (c == 0 && threadIdx.x == 0) out[0] = t1 - t0;
    if (acc == 12345.0) sink[0] = acc;
}

template <int MODE, int VOL>
void run(const char* name, int sms, int threads, uint4* ll, double* plain, long long* o, double* sink) {
    int iters = 2000;
    cudaMemset(ll, 0, (size_t)60 * 160 * 32 * 16);
    void* args[] = {&iters, &ll, &plain, &o, &sink};
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(ll, 0, (size_t)60 * 160 * 32 * 16);
        cudaLaunchCooperativeKernel((void*)probe<MODE, VOL>, sms, threads, args, 0, 0);
        cudaDeviceSynchronize();
    }
    cudaError_t e = cudaGetLastError();
    printf("%-28s G=%d threads=%d: %.0f cycles per exchange (%s)\n", name, sms, threads, (double)o[0] / iters,
           cudaGetErrorString(e));
}

int main() {
    long long* o;
    double *plain, *sink;
    uint4* ll;
    cudaMallocManaged(&o, 64);
    cudaMalloc(&ll, (size_t)60 * 160 * 32 * 16);
    cudaMalloc(&plain, (size_t)4 * 160 * 32 * 8);
    cudaMalloc(&sink, 64);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int G : {2, 16, 32, 148}) {
        run<1, 1>("LL two-level pull", G, 32, ll, plain, o, sink);
        run<8, 1>("LL three-hop push", G, 32, ll, plain, o, sink);
    }
    return 0;
}
