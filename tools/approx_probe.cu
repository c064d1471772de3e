// diagnostics: relative error of the f64 SFU seeds (rsqrt/rcp .approx.ftz)
#include <cstdio>
#include <cmath>
__global__ void k(const double* x, double* er, double* ec, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double y, z;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x[i]));
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(z) : "d"(x[i]));
    er[i] = fabs(y * sqrt(x[i]) - 1.0);
    ec[i] = fabs(z * x[i] - 1.0);
}
int main() {
    const int n = 1 << 20;
    double *x, *er, *ec;
    cudaMallocManaged(&x, n * 8); cudaMallocManaged(&er, n * 8); cudaMallocManaged(&ec, n * 8);
    unsigned long long s = 88172645463325252ull;
    for (int i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x[i] = std::ldexp(1.0 + (s % 1000003) / 1000003.0, (int)(s % 200) - 100); }
    k<<<n / 256, 256>>>(x, er, ec, n);
    cudaDeviceSynchronize();
    double mr = 0, mc = 0;
    for (int i = 0; i < n; ++i) { mr = fmax(mr, er[i]); mc = fmax(mc, ec[i]); }
    printf("rsqrt.approx.f64 max rel err %.3e (2^%.1f), rcp.approx.f64 %.3e (2^%.1f)\n", mr, log2(mr), mc, log2(mc));
}
