// Experiment (not in the product library; DESIGN.md §3 "measured and
// dropped"): the config-2 step-1 TSMM with its rows staged by TMA bulk copies
// (cp.async.bulk + mbarrier) instead of per-thread 8-byte cp.async.
// 2^24 x 16 . 16 x 16 (tools/tsmm_ab.py, B200): per-CTA 256-row chunks with a
// CTA barrier per chunk 0.98 ms (2-4 stages, L2 hints: no change); per-warp
// 32-row slices with a per-warp mbarrier 0.80 ms (3 stages; 2: 0.98, 5: 1.18);
// per-thread cp.async (the library's tsmm_async_kernel) 0.745 ms.
#pragma once
namespace ttsvd_b200 {
// K_TSMM for narrow X (m <= 32, n a multiple of 256): the streamed rows are
// staged in shared memory by the bulk-copy engine (TMA: cp.async.bulk, one
// column segment per instruction, completion counted in bytes on an
// mbarrier), kBulkStages slices in flight per warp.  The streamed bytes need
// no load instructions from the threads, which only do the FMAs and the
// coalesced stores.  Same arithmetic and output placement as tsmm_kernel.
constexpr int kBulkStages = 3;
__device__ __forceinline__ void bulk_mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_mbar_expect(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n BULK_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra BULK_WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}

template <int KC>
__global__ void __launch_bounds__(256) tsmm_bulk_kernel(const double* __restrict__ X, int64_t n, int m, int64_t ldx,
                                                        const double* __restrict__ V, int64_t ldv, int k,
                                                        double* __restrict__ Y, int64_t out_rows, int64_t ldy) {
    // per-warp pipelines: warp w streams 32-row slices (rows 32 w .. 32 w + 31
    // of every 256-row chunk); lane j < m copies column j of the slice (256
    // bytes) with one bulk copy; the warp's own mbarrier counts the bytes, so
    // no CTA-wide barrier is ever needed (as with per-thread cp.async, whose
    // threads only ever wait for their own copies)
    extern __shared__ __align__(128) double tsm[];
    __shared__ __align__(8) unsigned long long mbar[8][kBulkStages];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* xb = tsm + (size_t)warp * kBulkStages * m * 32;        // per warp: kBulkStages x m x 32
    double* Vs = tsm + (size_t)8 * kBulkStages * m * 32;            // m x KC
    const int c0 = blockIdx.y * KC;
    const int kc = min(KC, k - c0);
    const int64_t chunks = n / 256;
    auto bar = [&](int s) { return (unsigned)__cvta_generic_to_shared(&mbar[warp][s]); };
    auto issue = [&](int64_t ch, int s) {
        if (lane == 0) bulk_mbar_expect(bar(s), (unsigned)m * 256u);
        __syncwarp();
        if (lane < m)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(
                    (unsigned)__cvta_generic_to_shared(xb + ((size_t)s * m + lane) * 32)),
                "l"(X + (int64_t)lane * ldx + ch * 256 + 32 * warp), "r"(bar(s))
                : "memory");
    };
    if (lane == 0)
        for (int s = 0; s < kBulkStages; ++s) bulk_mbar_init(bar(s), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int e = tid; e < m * KC; e += blockDim.x) {
        const int j = e / KC, c = e % KC;
        Vs[e] = (c < kc) ? V[(int64_t)(c0 + c) * ldv + j] : 0.0;
    }
    __syncthreads();
    const bool divisible = (n % out_rows) == 0;
    const int64_t n_next = divisible ? n / out_rows : 0;
    int64_t ch = blockIdx.x;
    for (int s = 0; s < kBulkStages; ++s)
        if (ch + (int64_t)s * gridDim.x < chunks) issue(ch + (int64_t)s * gridDim.x, s);
    unsigned phase = 0;
    for (int s = 0; ch < chunks; ch += gridDim.x) {
        bulk_mbar_wait(bar(s), phase);
        const int64_t i = ch * 256 + 32 * warp + lane;
        const double* xr = xb + (size_t)s * m * 32 + lane;
        double acc[KC];
#pragma unroll
        for (int c = 0; c < KC; ++c) acc[c] = 0.0;
#pragma unroll 4
        for (int j = 0; j < m; ++j) {
            const double x = xr[j * 32];
            const double* vj = Vs + j * KC;
#pragma unroll
            for (int c = 0; c < KC; ++c) acc[c] = fma(vj[c], x, acc[c]);
        }
        __syncwarp();  // the warp's slice of stage s has been read: refill it
        const int64_t nx = ch + (int64_t)kBulkStages * gridDim.x;
        if (nx < chunks) issue(nx, s);
        if (divisible) {
            const int64_t b = i / out_rows, ii = i - b * out_rows;
#pragma unroll
            for (int c = 0; c < KC; ++c)
                if (c < kc) Y[(b + n_next * (c0 + c)) * ldy + ii] = acc[c];
        } else {
#pragma unroll
            for (int c = 0; c < KC; ++c)
                if (c < kc) {
                    const int64_t p = i + n * (c0 + c);
                    const int64_t col = p / out_rows;
                    Y[col * ldy + (p - col * out_rows)] = acc[c];
                }
        }
        if (++s == kBulkStages) {
            s = 0;
            phase ^= 1;
        }
    }
}


}  // namespace ttsvd_b200
