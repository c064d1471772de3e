// C-ABI and C++ host drivers of the B200 TT-SVD hot path (include/ttsvd_cu.h).
//
// Host side mirrors the reference drivers:
//   run_chain / tt_svd_tsqr        tt_svd.hpp:159-199, 281-290   (Alg. 2)
//   tt_svd_distributed             tt_svd.hpp:520-631            (Alg. 5)
// and launches the sm_100a kernels of ttsvd_kernels.cuh.  There is no CPU
// fallback anywhere in this library: every numeric step runs on the device.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is dlopen'ed on first use

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/ttsvd_cu.h"
#include "ttsvd_kernels.cuh"
#include "tsqr_blk.cuh"
#include "gqr.cuh"
#include "jacobi_blk.cuh"
#include "bidiag.cuh"
#include "tsqr_la.cuh"
#include "tsqr_t128.cuh"
#include "tsqr_ws.cuh"
#include "tsqr_pt.cuh"
#include "tsqr_gt.cuh"
#include "tsmm_dt.cuh"

using namespace ttsvd_b200;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define TT_CUDA(call)                                                                                     \
    do {                                                                                                  \
        cudaError_t e_ = (call);                                                                          \
        if (e_ != cudaSuccess) {                                                                          \
            return fail(e_ == cudaErrorMemoryAllocation ? TTSVD_ERR_ALLOCATION : TTSVD_ERR_DEVICE,        \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                              \
        }                                                                                                 \
    } while (0)

#define TT_TRY(call)                 \
    do {                             \
        int rc_ = (call);            \
        if (rc_ != TTSVD_OK) return rc_; \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

}  // namespace

struct ttsvd_cu_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    int coop_max_blocks = 0;  // co-resident CTAs of jacobi_coop_kernel
    int64_t launches = 0;
    bool timing = false;
    // grow-only device workspaces
    DevBuf ws_R, ws_R2, ws_P, ws_Scr, ws_G, ws_Gp, ws_A, ws_V, ws_Vacc, ws_U, ws_sigma, ws_flags, ws_work[2], ws_X, ws_send, ws_recv, ws_thick[2], ws_gs, ws_bd;
    std::vector<DevBuf> ws_slab;  // tt_svd_distributed: two ping-pong work buffers per local slab
    DevBuf host_stage;  // pinned
    DevBuf host_cores;  // pinned arena of the steps' V blocks (core_from_vt after the chain)
    DevBuf ws_gt_state;  // tsqr_gt_kernel in row chunks: the streams' running R factors between launches
    cudaStream_t copy_stream = nullptr;  // host entry: H2D of X in row chunks under the first TSQR
    cudaEvent_t copy_ev = nullptr;
    DevBuf ws_rank;     // K6: per step (rank, sum sigma^2) written by rank_epilogue_kernel
    DevBuf host_sig;    // pinned: per step the sigmas and the K6 record of a speculative chain
    cudaEvent_t ev[9] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    // svd_work's bidiagonal path leaves the vectors for svd_vectors (the
    // driver knows the rank only after the sigmas): A holds the reflectors
    bool bd_pending = false;
    const double* bd_A = nullptr;
    int bd_n = 0, bd_m = 0;
    int last_kernel = 0;  // TTSVD_K_* of the last tsqr_device main sweep (ev[5], ev[6] bracket it when timing)
    // kernel attributes and occupancies are properties of the device, so they
    // are cached per context (one device each), never process-wide
    std::map<const void*, int> smem_attr;
    std::map<std::tuple<const void*, int, size_t>, int> occ;
    // NCCL communicator of a distributed run (ttsvd_cu_ctx_comm_init*):
    // tt_svd_distributed all-gathers the R factors over it on `stream`
    ncclComm_t comm = nullptr;
    int comm_rank = 0, comm_size = 1;
};

struct ttsvd_cu_tt {
    std::vector<int64_t> dims, ranks;
    std::vector<std::vector<double>> cores;
    std::vector<ttsvd_cu_step> steps;
    std::vector<std::vector<double>> sigmas;
};

namespace {

int ensure(DevBuf& b, size_t bytes) {
    if (b.bytes >= bytes) return TTSVD_OK;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    const size_t alloc = std::max<size_t>(bytes, 256);
    TT_CUDA(cudaMalloc(&b.p, alloc));
    b.bytes = alloc;
    return TTSVD_OK;
}

int ensure_host(DevBuf& b, size_t bytes) {
    if (b.bytes >= bytes) return TTSVD_OK;
    if (b.p) cudaFreeHost(b.p);
    b.p = nullptr;
    b.bytes = 0;
    TT_CUDA(cudaMallocHost(&b.p, std::max<size_t>(bytes, 4096)));
    b.bytes = std::max<size_t>(bytes, 4096);
    return TTSVD_OK;
}

template <class T>
T* as(DevBuf& b) {
    return static_cast<T*>(b.p);
}

// ---- NCCL, loaded at run time (the single-GPU path never needs it) -------
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // the libnccl.so.2 already in the process (e.g. torch's) is reused by soname
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
        api.comm_init_all = reinterpret_cast<decltype(api.comm_init_all)>(sym("ncclCommInitAll"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_init_all && api.all_gather && api.comm_destroy &&
                 api.error_string;
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

#define TT_NCCL(call)                                                                                     \
    do {                                                                                                  \
        const ncclResult_t r_ = (call);                                                                   \
        if (r_ != ncclSuccess) return fail(TTSVD_ERR_DEVICE, std::string(#call) + ": " + nccl().error_string(r_)); \
    } while (0)

int64_t padded_stride_h(int64_t n) {
    if (n < 1) return -1;
    if (n <= 64) return 64;
    int64_t q = (n + 63) / 64;
    if (q % 2 == 0) ++q;
    return 64 * q;
}

int check_launch(ttsvd_cu_ctx* ctx, const char* what) {
    ctx->launches += 1;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(TTSVD_ERR_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
    return TTSVD_OK;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize [, NonPortableClusterSize])
// for `fn` on the context's device, once per (context, kernel) and size.
int kattr(ttsvd_cu_ctx* ctx, const void* fn, int smem_bytes, bool nonportable_cluster = false) {
    auto it = ctx->smem_attr.find(fn);
    if (it != ctx->smem_attr.end() && it->second >= smem_bytes) return TTSVD_OK;
    TT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
    if (nonportable_cluster) TT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    ctx->smem_attr[fn] = smem_bytes;
    return TTSVD_OK;
}

// co-resident CTAs per SM of `fn` at (threads, dynamic smem) on the context's device
int koccupancy(ttsvd_cu_ctx* ctx, const void* fn, int threads, size_t smem, int* per_sm) {
    const auto key = std::make_tuple(fn, threads, smem);
    auto it = ctx->occ.find(key);
    if (it != ctx->occ.end()) {
        *per_sm = it->second;
        return TTSVD_OK;
    }
    int v = 0;
    TT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, fn, threads, smem));
    ctx->occ[key] = v;
    *per_sm = v;
    return TTSVD_OK;
}

// static shared memory of `fn`
int kstatic_smem(const void* fn, int* bytes) {
    cudaFuncAttributes fa;
    TT_CUDA(cudaFuncGetAttributes(&fa, fn));
    *bytes = (int)fa.sharedSizeBytes;
    return TTSVD_OK;
}

int set_device(ttsvd_cu_ctx* ctx) {
    if (!ctx) return fail(TTSVD_ERR_INVALID, "null context");
    TT_CUDA(cudaSetDevice(ctx->device));
    return TTSVD_OK;
}

// internal: the kernel a shape dispatches to cannot read a split-column view
// (ColSplit) in place; the caller materialises the view and calls again
constexpr int kNoView = -2;
constexpr int64_t kSqMaxRows = 1 << 16;  // 32 < m <= 64 up to here: levels of single tiles (tsqr_t2_levels)
constexpr int kTsqrThreads = 256;
constexpr int kSmemLimit = 227 * 1024;
constexpr int kTsmmSmem = 200 * 1024;  // V block of tsmm_kernel (m x KC doubles)

// ---------------------------------------------------------------- K_TSQR ----
struct TsqrPlan {
    int bt, ldb, r_in_smem;
    size_t smem;
};

TsqrPlan tsqr_plan(int m) {
    TsqrPlan p;
    p.r_in_smem = (m <= 64);
    const size_t r_bytes = p.r_in_smem ? (size_t)m * m * 8 : 0;
    const size_t tile_budget = m <= 64 ? 64 * 1024 : 160 * 1024;
    int bt = (int)std::max<size_t>(1, tile_budget / ((size_t)m * 8));
    bt = std::min(bt, 2048);
    if (bt >= 32) bt = bt / 32 * 32;
    p.bt = bt;
    p.ldb = bt;
    p.smem = r_bytes + (size_t)p.ldb * m * 8 + (kTsqrThreads / 32 + 4) * 8;
    return p;
}

int launch_tsqr_kernel(ttsvd_cu_ctx* ctx, const TsqrArgs& a, int grid, size_t smem) {
    TT_TRY(kattr(ctx, (const void*)tsqr_tile_kernel<kTsqrThreads>, kSmemLimit));
    tsqr_tile_kernel<kTsqrThreads><<<grid, kTsqrThreads, smem, ctx->stream>>>(a);
    return check_launch(ctx, "tsqr_tile_kernel");
}

// ---- blocked DMMA path (m > 32) ----
constexpr int kSmallM = 32;

int set_la_attr(ttsvd_cu_ctx* ctx) {
    int ss = 0;
    TT_TRY(kstatic_smem((const void*)tsqr_la_kernel, &ss));
    return kattr(ctx, (const void*)tsqr_la_kernel, kSmemLimit - ss);
}

int launch_blk(ttsvd_cu_ctx* ctx, const BlkArgs& a, int grid) {
    TT_TRY(set_la_attr(ctx));
    tsqr_la_kernel<<<grid, kLaThreads, la_smem_bytes(a.M), ctx->stream>>>(a);
    return check_launch(ctx, "tsqr_la_kernel");
}

int copy_leading(ttsvd_cu_ctx* ctx, const double* Rws, int M, int m, double* R) {
    copy_leading_kernel<<<std::max(1, std::min(1024, (m * m + 255) / 256)), 256, 0, ctx->stream>>>(Rws, M, m, R);
    return check_launch(ctx, "copy_leading_kernel");
}

// merge tree over `count` packed workspace parts in `parts` (overwritten);
// the final packed factor lands in `out`.
int merge_tree_blk(ttsvd_cu_ctx* ctx, double* parts, int64_t count, int m, int M, double* out) {
    const int64_t RS = blk_rsize(M);
    if (count == 1) {
        TT_CUDA(cudaMemcpyAsync(out, parts, (size_t)RS * 8, cudaMemcpyDeviceToDevice, ctx->stream));
        return TTSVD_OK;
    }
    TT_TRY(ensure(ctx->ws_R2, (size_t)((count + 1) / 2) * RS * 8));
    double* src = parts;
    double* bufs[2] = {as<double>(ctx->ws_R2), parts};
    int flip = 0;
    while (count > 1) {
        const int64_t next = (count + 1) / 2;
        double* dst = (next == 1) ? out : bufs[flip];
        BlkArgs a{src, count, (int64_t)M, dst, nullptr, m, M, 1, nullptr};
        TT_TRY(launch_blk(ctx, a, (int)next));
        src = dst;
        count = next;
        flip ^= 1;
    }
    return TTSVD_OK;
}

int pack_parts(ttsvd_cu_ctx* ctx, const double* parts, int64_t P, int m, int M, double* out) {
    const int64_t total = P * blk_rsize(M);
    pack_parts_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, ctx->stream>>>(parts, P, m, M,
                                                                                                   out);
    return check_launch(ctx, "pack_parts_kernel");
}

int gqr_device(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ld, double* R);

// Fixed index-ordered merge tree over `count` parts (each m x m, ld m); the
// result lands in R_final.  Level l pairs (2i, 2i+1); an odd tail is carried.
int merge_tree(ttsvd_cu_ctx* ctx, double* parts, int64_t count, int m, double* R_final) {
    if (count == 1) {
        TT_CUDA(cudaMemcpyAsync(R_final, parts, (size_t)m * m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
        return TTSVD_OK;
    }
    if (m > kSmallM) {
        const int M = (m + 31) / 32 * 32;
        const int64_t RS = blk_rsize(M);
        if (count >= 4 && count * m >= M && count * m <= (int64_t)kGqrMaxRows * ctx->num_sms) {
            // one cooperative QR of the stacked factors (rows q*m .. q*m+m-1 = part q)
            const int64_t ns = count * m;
            TT_TRY(ensure(ctx->ws_G, (size_t)ns * M * 8));
            double* Aw = as<double>(ctx->ws_G);
            if (M > m) TT_CUDA(cudaMemsetAsync(Aw + (size_t)ns * m, 0, (size_t)ns * (M - m) * 8, ctx->stream));
            for (int64_t q = 0; q < count; ++q)
                TT_CUDA(cudaMemcpy2DAsync(Aw + q * m, (size_t)ns * 8, parts + q * m * m, (size_t)m * 8, (size_t)m * 8, m,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
            const int rc = gqr_device(ctx, Aw, ns, m, ns, R_final);
            if (rc != -1) return rc;
        }
        TT_TRY(ensure(ctx->ws_P, (size_t)(count + 1) * RS * 8));
        double* P = as<double>(ctx->ws_P);
        TT_TRY(pack_parts(ctx, parts, count, m, M, P));
        double* out = P + count * RS;
        TT_TRY(merge_tree_blk(ctx, P, count, m, M, out));
        return copy_leading(ctx, out, M, m, R_final);
    }
    TT_TRY(ensure(ctx->ws_R2, (size_t)((count + 1) / 2) * m * m * 8));
    TsqrPlan p = tsqr_plan(m);
    double* src = parts;
    double* bufs[2] = {as<double>(ctx->ws_R2), parts};
    int flip = 0;
    while (count > 1) {
        const int64_t next = (count + 1) / 2;
        double* dst = (next == 1) ? R_final : bufs[flip];
        TsqrArgs a{src, count, (int64_t)m, dst, m, p.bt, p.ldb, 1, p.r_in_smem, nullptr};
        TT_TRY(launch_tsqr_kernel(ctx, a, (int)next, p.smem));
        src = dst;
        count = next;
        flip ^= 1;
    }
    return TTSVD_OK;
}

// Cooperative whole-grid blocked QR (gqr.cuh) of X (n x m, ld): R (m x m).
// Returns -1 when the shape does not fit one co-resident grid.
int gqr_device(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ld, double* R) {
    const int M = (m + 31) / 32 * 32;
    if (n < M || n > (int64_t)kGqrMaxRows * ctx->num_sms) return -1;
    // a cooperative grid of up to one CTA per SM, 64 target rows per CTA (more
    // CTAs: the blocked updates spread wider; config 2 step 4, 4096 x 512:
    // 3.30 ms at 128 rows, 3.07 at 64)
    int64_t Gq = std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms, n / 64));
    while ((n + Gq - 1) / Gq > kGqrMaxRows) ++Gq;
    const int rows_max = (int)((n + Gq - 1) / Gq);
    // more than 256 rows per CTA: 512 threads (one row each; the blocked
    // updates gain more than the reflector chain loses — config 2 step 3
    // 6.31 -> 5.74 ms); otherwise 256 (steps with <= 256 rows per CTA are
    // slower with 512)
    const int gnt = rows_max > 256 ? 512 : 256;
    const size_t smem = gqr_smem_bytes(rows_max, gnt);
    const void* gfn = gnt == 512 ? (const void*)gqr_kernel<false, 512> : (const void*)gqr_kernel<false, 256>;
    TT_TRY(kattr(ctx, gfn, kSmemLimit));
    int per_sm = 0;
    TT_TRY(koccupancy(ctx, gfn, gnt, smem, &per_sm));
    if (per_sm < 1 || Gq > (int64_t)per_sm * ctx->num_sms) return -1;
    TT_TRY(ensure(ctx->ws_G, (size_t)n * M * 8));
    const size_t np = (size_t)2 * Gq * 33 + (size_t)Gq * 1024 + (size_t)Gq * 32 * M;
    TT_TRY(ensure(ctx->ws_Gp, (np + 64 + (size_t)32 * M + 1024) * 8));
    double* Aw = as<double>(ctx->ws_G);
    if (X != Aw) {
        TT_CUDA(cudaMemcpy2DAsync(Aw, (size_t)n * 8, X, (size_t)ld * 8, (size_t)n * 8, m, cudaMemcpyDeviceToDevice,
                                  ctx->stream));
        if (M > m) TT_CUDA(cudaMemsetAsync(Aw + (size_t)n * m, 0, (size_t)n * (M - m) * 8, ctx->stream));
    }
    double* pp = as<double>(ctx->ws_Gp);
    GqrArgs ga{Aw, n, n, m, M, pp, pp + np, pp + np + 64, pp + np + 64 + (size_t)32 * M, nullptr};
    {
        void* args[] = {&ga};
        TT_CUDA(cudaLaunchCooperativeKernel(gfn, dim3((unsigned)Gq), dim3(gnt), args, smem, ctx->stream));
    }
    TT_TRY(check_launch(ctx, "gqr_kernel"));
    gqr_extract_kernel<<<std::max(1, std::min(1024, (m * m + 255) / 256)), 256, 0, ctx->stream>>>(Aw, n, m, R);
    return check_launch(ctx, "gqr_extract_kernel");
}

// Merge of `count` packed factors by one cooperative QR of their stack
// (replaces log2(count) levels of single-CTA merges).  -1 if it does not fit.
int merge_stack_gqr(ttsvd_cu_ctx* ctx, const double* parts, int64_t count, int m, int M, double* R) {
    const int64_t n = count * M;
    if (count < 4 || n > (int64_t)kGqrMaxRows * ctx->num_sms) return -1;
    TT_TRY(ensure(ctx->ws_G, (size_t)n * M * 8));
    double* Aw = as<double>(ctx->ws_G);
    const int64_t tot = n * M;
    stack_packed_kernel<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 8192), 256, 0, ctx->stream>>>(parts, count, M,
                                                                                                    Aw);
    TT_TRY(check_launch(ctx, "stack_packed_kernel"));
    return gqr_device(ctx, Aw, n, m, n, R);
}

// R (m x m) of X (n x m, ld) — n may be smaller than m (the structured kernel
// does not need n >= m; gram_triangular's square padding is implicit).
// R_init (m x m) optionally seeds a single job (reduce_block).
// events bracketing the main sweep kernel of tsqr_device (timing mode)
inline void kmark(ttsvd_cu_ctx* ctx, int i, int kernel) {
    if (ctx->timing) cudaEventRecord(ctx->ev[5 + i], ctx->stream);
    ctx->last_kernel = kernel;
}

// m <= 32: warp streams (tsqr_ws.cuh), levels of stacked factors until one
// stream is left.
template <int SW>
int tsqr_ws_levels(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ld, double* R, bool mark) {
    int per_sm = 0;
    const size_t smem = ws_smem_bytes<SW>();
    TT_TRY(kattr(ctx, (const void*)tsqr_ws_kernel<SW>, (int)smem));
    TT_TRY(koccupancy(ctx, (const void*)tsqr_ws_kernel<SW>, kWsThreads, smem, &per_sm));
    per_sm = std::max(1, per_sm);
    constexpr int per_cta = (kWsThreads / 32) * (32 / SW);
    const int64_t max_streams = (int64_t)per_sm * ctx->num_sms * per_cta;
    const double* src = X;
    int64_t rows = n, sld = ld;
    int flip = 0;
    for (;;) {
        // >= 2 tiles per stream (the levels are latency chains: config 2
        // step 1's levels 0.23 ms at 4 tiles, 0.20 at 2, 0.25 at 1), and
        // >= 4 m rows per stream so that every level cuts the rows by >= 4x
        int64_t S = std::min<int64_t>(rows / std::max<int64_t>(64, 4 * (int64_t)m), max_streams);
        if (S < 1) S = 1;
        if (S > 1) {
            TT_TRY(ensure(ctx->ws_R, (size_t)S * m * m * 8));
            TT_TRY(ensure(ctx->ws_R2, (size_t)S * m * m * 8));
        }
        double* out = (S == 1) ? R : as<double>(flip ? ctx->ws_R2 : ctx->ws_R);
        const int64_t ldo = (S == 1) ? m : S * m;
        WsArgs wa{src, rows, sld, m, S, out, ldo};
        const int64_t grid = (S + per_cta - 1) / per_cta;
        if (mark && src == X) kmark(ctx, 0, TTSVD_K_WS);
        tsqr_ws_kernel<SW><<<(unsigned)grid, kWsThreads, smem, ctx->stream>>>(wa);
        TT_TRY(check_launch(ctx, "tsqr_ws_kernel"));
        if (mark && src == X) kmark(ctx, 1, TTSVD_K_WS);
        if (S == 1) return TTSVD_OK;
        src = out;
        rows = S * m;
        sld = S * m;
        flip ^= 1;
    }
}

// mark: bracket the first level with the timing events (false for the tail
// of another kernel's levels)
int tsqr_ws_device(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ld, double* R, bool mark = true) {
    return m <= 16 ? tsqr_ws_levels<16>(ctx, X, n, m, ld, R, mark) : tsqr_ws_levels<32>(ctx, X, n, m, ld, R, mark);
}

// m <= 8: thread streams (tsqr_pt.cuh), levels of stacked factors (~64 rows
// per thread stream once the grid is full) until one thread is left.
template <int M>
int tsqr_pt_levels(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int64_t ld, double* R) {
    // rows per fold (x (U x M) and R stay in registers); measured on B200:
    // U = 4 keeps two CTAs per SM for m = 5, 6, U = 8 wins at m = 7, 8
    constexpr int U = (M == 5 || M == 6) ? 4 : 8;
    int per_sm = 0;
    TT_TRY(koccupancy(ctx, (const void*)tsqr_pt_kernel<M, U>, kPtThreads, 0, &per_sm));
    per_sm = std::max(1, per_sm);
    const int64_t max_t = (int64_t)per_sm * ctx->num_sms * kPtThreads;
    const double* src = X;
    int64_t rows = n, sld = ld;
    int flip = 0;
    for (;;) {
        int64_t T = std::min<int64_t>(rows / 64, max_t);
        if (T < 1) T = 1;
        if (T > 1) {
            TT_TRY(ensure(ctx->ws_R, (size_t)T * M * M * 8));
            TT_TRY(ensure(ctx->ws_R2, (size_t)T * M * M * 8));
        }
        double* out = (T == 1) ? R : as<double>(flip ? ctx->ws_R2 : ctx->ws_R);
        const int64_t ldo = (T == 1) ? M : T * M;
        PtArgs pa{src, rows, sld, T, out, ldo};
        if (src == X) kmark(ctx, 0, TTSVD_K_PT);
        tsqr_pt_kernel<M, U><<<(unsigned)((T + kPtThreads - 1) / kPtThreads), kPtThreads, 0, ctx->stream>>>(pa);
        TT_TRY(check_launch(ctx, "tsqr_pt_kernel"));
        if (src == X) kmark(ctx, 1, TTSVD_K_PT);
        if (T == 1) return TTSVD_OK;
        src = out;
        rows = T * M;
        sld = T * M;
        flip ^= 1;
    }
}

int tsqr_pt_device(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ld, double* R) {
    switch (m) {
        case 1: return tsqr_pt_levels<1>(ctx, X, n, ld, R);
        case 2: return tsqr_pt_levels<2>(ctx, X, n, ld, R);
        case 3: return tsqr_pt_levels<3>(ctx, X, n, ld, R);
        case 4: return tsqr_pt_levels<4>(ctx, X, n, ld, R);
        case 5: return tsqr_pt_levels<5>(ctx, X, n, ld, R);
        case 6: return tsqr_pt_levels<6>(ctx, X, n, ld, R);
        case 7: return tsqr_pt_levels<7>(ctx, X, n, ld, R);
        case 8: return tsqr_pt_levels<8>(ctx, X, n, ld, R);
        default: return TTSVD_ERR_INVALID;
    }
}

// 8 < m <= 32: group streams (tsqr_gs_kernel, P lanes per stream, M the
// padded width), levels of stacked factors as tsqr_pt_levels.
template <int M, int P, int U>
int tsqr_gs_levels(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ld, double* R) {
    int per_sm = 0;
    TT_TRY(koccupancy(ctx, (const void*)tsqr_gs_kernel<M, P, U>, kPtThreads, 0, &per_sm));
    per_sm = std::max(1, per_sm);
    const int64_t max_t = (int64_t)per_sm * ctx->num_sms * (kPtThreads / P);
    int64_t T = std::max<int64_t>(1, std::min<int64_t>(n / 64, max_t));
    // the stacked factors get their own buffer (the warp-stream tail uses
    // ws_R / ws_R2)
    DevBuf& ob = ctx->ws_gs;
    if (T > 1) TT_TRY(ensure(ob, (size_t)T * m * m * 8));
    double* out = (T == 1) ? R : as<double>(ob);
    const int64_t ldo = (T == 1) ? m : T * m;
    GsArgs ga{X, n, ld, m, T, out, ldo};
    kmark(ctx, 0, TTSVD_K_GS);
    const int64_t threads = (T * P + 31) / 32 * 32;
    tsqr_gs_kernel<M, P, U><<<(unsigned)((threads + kPtThreads - 1) / kPtThreads), kPtThreads, 0, ctx->stream>>>(ga);
    TT_TRY(check_launch(ctx, "tsqr_gs_kernel"));
    kmark(ctx, 1, TTSVD_K_GS);
    if (T == 1) return TTSVD_OK;
    // the stacked factors are short: warp streams finish them with far
    // shorter per-stream chains than another group-stream level
    return tsqr_ws_device(ctx, out, T * m, m, T * m, R, false);
}

// Tall and 16-byte aligned: the same streams fed by the bulk-copy engine
// (tsqr_gt.cuh), one 8-warp CTA per SM, every warp at least one full slice.
constexpr int gt_threads(int M) { return M <= 16 ? 384 : kPtThreads; }
constexpr int kGtMaxWarps = 12;

template <int M, int P, int U>
int tsqr_gt_levels(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ld, double* R, ColSplit cs) {
    constexpr int G = 32 / P, SR = G * U, NTH = gt_threads(M), NWp = NTH / 32;
    const void* fn = (const void*)tsqr_gt_kernel<M, P, U, 1, kGtStages, NTH>;
    TT_TRY(kattr(ctx, fn, (int)gt_smem_bytes<M, P, U, kGtStages, NTH>()));
    const int64_t slices = (n + SR - 1) / SR;
    const int64_t ctas = std::min<int64_t>(ctx->num_sms, slices / NWp);
    const int64_t T = ctas * NWp * G;
    DevBuf& ob = ctx->ws_gs;
    TT_TRY(ensure(ob, (size_t)T * m * m * 8));
    double* out = as<double>(ob);
    GsArgs ga{X, n, ld, m, T, out, T * m, cs};
    kmark(ctx, 0, TTSVD_K_GT);
    tsqr_gt_kernel<M, P, U, 1, kGtStages, NTH>
        <<<(unsigned)ctas, NTH, gt_smem_bytes<M, P, U, kGtStages, NTH>(), ctx->stream>>>(ga);
    TT_TRY(check_launch(ctx, "tsqr_gt_kernel"));
    kmark(ctx, 1, TTSVD_K_GT);
    return tsqr_ws_device(ctx, out, T * m, m, T * m, R, false);
}

// The same sweep in `chunks` launches over consecutive row ranges (whole
// rounds of the grid's warps, so every stream folds the same slices in the
// same order as in one launch: identical bits); before(row_lo, row_hi) runs
// ahead of each launch — the host entry enqueues that range's H2D there.
template <int M, int P, int U, class Before>
int tsqr_gt_chunked(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ld, double* R, int chunks,
                    Before before) {
    constexpr int G = 32 / P, SR = G * U, MC = M / P, NTH = gt_threads(M), NWp = NTH / 32;
    const void* fn = (const void*)tsqr_gt_kernel<M, P, U, 1, kGtStages, NTH>;
    TT_TRY(kattr(ctx, fn, (int)gt_smem_bytes<M, P, U, kGtStages, NTH>()));
    const int64_t slices = (n + SR - 1) / SR;
    const int64_t ctas = std::min<int64_t>(ctx->num_sms, slices / NWp);
    const int64_t Wt = ctas * NWp, T = Wt * G;
    TT_TRY(ensure(ctx->ws_gs, (size_t)T * m * m * 8));
    TT_TRY(ensure(ctx->ws_gt_state, (size_t)Wt * 32 * M * MC * 8));
    double* out = as<double>(ctx->ws_gs);
    const int64_t rounds = (slices + Wt - 1) / Wt, rpc = (rounds + chunks - 1) / chunks;
    kmark(ctx, 0, TTSVD_K_GT);
    for (int64_t c = 0; c * rpc * Wt < slices; ++c) {
        const int64_t lo = c * rpc * Wt, hi = std::min(slices, (c + 1) * rpc * Wt);
        TT_TRY(before(lo * SR, std::min(n, hi * SR)));
        GsArgs ga{X, n, ld, m, T, out, T * m, ColSplit{0, 0}, lo, hi, as<double>(ctx->ws_gt_state),
                  (c > 0 ? 1 : 0) | (hi < slices ? 2 : 0)};
        tsqr_gt_kernel<M, P, U, 1, kGtStages, NTH>
            <<<(unsigned)ctas, NTH, gt_smem_bytes<M, P, U, kGtStages, NTH>(), ctx->stream>>>(ga);
        TT_TRY(check_launch(ctx, "tsqr_gt_kernel"));
    }
    kmark(ctx, 1, TTSVD_K_GT);
    return tsqr_ws_device(ctx, out, T * m, m, T * m, R, false);
}

// tsqr_gs_device dispatches a shape to the TMA-staged kernel under these conditions
bool gt_eligible(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ld) {
    return m > 8 && m <= kSmallM && n >= (int64_t)ctx->num_sms * kGtMaxWarps * 64 * 4 && (ld & 1) == 0 &&
           ((uintptr_t)X & 15) == 0;
}

int tsqr_gs_device(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ld, double* R,
                   ColSplit cs = ColSplit{0, 0}) {
    if (gt_eligible(ctx, X, n, m, ld) && (cs.q == 0 || (cs.ld_lo & 1) == 0))
        return m <= 16 ? tsqr_gt_levels<16, 4, 8>(ctx, X, n, m, ld, R, cs)
                       : tsqr_gt_levels<32, 8, 8>(ctx, X, n, m, ld, R, cs);
    if (cs.q) return kNoView;
    // measured on B200 (tools/gs_var.sh): 4 lanes per stream at m <= 16, 8 at m <= 32
    // (a whole warp per stream at 32 < m <= 64 measured slower than t128)
    return m <= 16 ? tsqr_gs_levels<16, 4, 8>(ctx, X, n, m, ld, R) : tsqr_gs_levels<32, 8, 8>(ctx, X, n, m, ld, R);
}

// Tall tiles (tsqr_t128_kernel, one CTA per SM) + one cooperative QR of the
// 148 stacked factors.  chunk_rows > 0: the sweep runs in launches over
// consecutive row ranges, the per-CTA factors carried from launch to launch;
// before(row_lo, row_hi) runs ahead of each launch (the thick-bounds host
// entry enqueues that range's H2D there).
template <class Before>
int tsqr_t128_run(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ld, double* R, ColSplit cs,
                  int64_t chunk_rows, Before before) {
    const int M = (m + 31) / 32 * 32;
    const int64_t RS = blk_rsize(M);
    // 256-row tiles (8 panel + 8 update warps of a 512-thread CTA): the
    // reflector chain per row is half the 128-row tile's (config 2 step 2
    // sweep: 13.7 ms at 128 rows / 384 threads, 12.35 at 192 / 384, 11.8
    // at 256 / 512; 12.8 at 320 / 512).
    const int t2rows = n >= (int64_t)ctx->num_sms * 4 * 256 ? 256 : 128;
    const int64_t Gt = ctx->num_sms;
    TT_TRY(ensure(ctx->ws_R, (size_t)Gt * RS * 8));
    TT_TRY(ensure(ctx->ws_Scr, (size_t)Gt * t2rows * M * 8));
    double* parts = as<double>(ctx->ws_R);
    const void* tfn = t2rows == 256 ? (const void*)tsqr_t128_kernel<256> : (const void*)tsqr_t128_kernel<128>;
    TT_TRY(kattr(ctx, tfn, (int)t2_smem_bytes(t2rows)));
    kmark(ctx, 0, TTSVD_K_T128);
    const int64_t step = chunk_rows > 0 ? chunk_rows : n;
    for (int64_t lo = 0; lo < n; lo += step) {
        const int64_t hi = std::min(n, lo + step);
        TT_TRY(before(lo, hi));
        T2Args ta{X, n, ld, parts, as<double>(ctx->ws_Scr), m, M, nullptr, cs, lo, hi, lo > 0 ? 1 : 0};
        if (t2rows == 256)
            tsqr_t128_kernel<256><<<(unsigned)Gt, kT2Threads, t2_smem_bytes(256), ctx->stream>>>(ta);
        else
            tsqr_t128_kernel<128><<<(unsigned)Gt, kT2Threads, t2_smem_bytes(128), ctx->stream>>>(ta);
        TT_TRY(check_launch(ctx, "tsqr_t128_kernel"));
    }
    kmark(ctx, 1, TTSVD_K_T128);
    const int rc = merge_stack_gqr(ctx, parts, Gt, m, M, R);
    if (rc != -1) return rc;
    TT_TRY(ensure(ctx->ws_P, (size_t)RS * 8));
    TT_TRY(merge_tree_blk(ctx, parts, Gt, m, M, as<double>(ctx->ws_P)));
    return copy_leading(ctx, as<double>(ctx->ws_P), M, m, R);
}

// 32 < m <= 64, small n (config 1's m = 64 steps): levels of 256-row tiles on
// the tall-tile kernel, one tile per CTA (register-tile panels, phase A on
// DMMA), the packed factors re-stacked densely for the next level until one
// tile is left (a 4-ary combine tree in index order, tsqr.hpp:204-240).
// ~60 us per level against ~90 us for the former column-per-lane tile kernel
// (two CTA barriers and 64 shared-memory loads per thread and reflector) and
// ~5 us per reflector for the cooperative grid on these shapes.
int tsqr_t2_levels(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ld, double* R) {
    const int M = (m + 31) / 32 * 32;
    const int64_t RS = blk_rsize(M);
    TT_TRY(kattr(ctx, (const void*)tsqr_t128_kernel<256>, (int)t2_smem_bytes(256)));
    const double* src = X;
    int64_t rows = n, sld = ld;
    int mm = m;
    for (;;) {
        const int64_t T = (rows + 255) / 256;
        TT_TRY(ensure(ctx->ws_R, (size_t)T * RS * 8));
        TT_TRY(ensure(ctx->ws_Scr, (size_t)T * 256 * M * 8));
        double* parts = as<double>(ctx->ws_R);
        T2Args ta{src, rows, sld, parts, as<double>(ctx->ws_Scr), mm, M, nullptr, ColSplit{0, 0}, 0, 0, 0};
        tsqr_t128_kernel<256><<<(unsigned)T, kT2Threads, t2_smem_bytes(256), ctx->stream>>>(ta);
        TT_TRY(check_launch(ctx, "tsqr_t128_kernel"));
        if (T == 1) return copy_leading(ctx, parts, M, m, R);
        TT_TRY(ensure(ctx->ws_G, (size_t)T * M * M * 8));
        double* Aw = as<double>(ctx->ws_G);
        const int64_t tot = T * M * M;
        stack_packed_kernel<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 8192), 256, 0, ctx->stream>>>(parts, T, M, Aw);
        TT_TRY(check_launch(ctx, "stack_packed_kernel"));
        src = Aw;
        rows = T * M;
        sld = T * M;
        mm = M;  // the stacked factors are M wide (columns m .. M-1 zero)
    }
}

// the shapes tsqr_device sends to tsqr_t128_run
bool t128_eligible(ttsvd_cu_ctx* ctx, int64_t n, int m) {
    const int M = (m + 31) / 32 * 32;
    return m > kSmallM && !(m <= 64 && n <= kSqMaxRows) && !(n >= M && n <= (int64_t)256 * M) &&
           n >= (int64_t)ctx->num_sms * 4 * kT2Rows;
}

int tsqr_device(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ld, double* R,
                const double* R_init = nullptr, ColSplit cs = ColSplit{0, 0}) {
    ctx->last_kernel = TTSVD_K_NONE;
    if (m > kSmallM) {
        const int M = (m + 31) / 32 * 32;
        const int64_t RS = blk_rsize(M);
        // a split-column view is read in place by the tall-tile kernel only
        if (cs.q && (R_init || (m <= 64 && n <= kSqMaxRows) || (n >= M && n <= (int64_t)256 * M) ||
                     n < (int64_t)ctx->num_sms * 4 * kT2Rows))
            return kNoView;
        if (!R_init && m <= 64 && n <= kSqMaxRows) {
            kmark(ctx, 0, TTSVD_K_SQ);
            const int rc = tsqr_t2_levels(ctx, X, n, m, ld, R);
            kmark(ctx, 1, TTSVD_K_SQ);
            return rc;
        }
        // Short-fat (n <= 256 M, n <= 512 rows per SM): one cooperative grid
        // factorises the whole matrix (gqr.cuh), no merge tree.
        if (!R_init && n >= M && n <= (int64_t)256 * M) {
            kmark(ctx, 0, TTSVD_K_GQR);
            const int rc = gqr_device(ctx, X, n, m, ld, R);
            kmark(ctx, 1, TTSVD_K_GQR);
            if (rc != -1) return rc;
            ctx->last_kernel = 0;
        }
        // Tall: ROWS-row tiles, one CTA per SM, when every CTA gets >= 4 tiles
        // (the 148 factors are merged by one cooperative QR of their stack).
        // 256-row tiles (8 panel + 8 update warps of a 512-thread CTA): the
        // reflector chain per row is half the 128-row tile's (config 2 step 2
        // sweep: 13.7 ms at 128 rows / 384 threads, 12.35 at 192 / 384, 11.8
        // at 256 / 512; 12.8 at 320 / 512).
        if (!R_init && n >= (int64_t)ctx->num_sms * 4 * kT2Rows)
            return tsqr_t128_run(ctx, X, n, m, ld, R, cs, 0, [](int64_t, int64_t) { return TTSVD_OK; });
        int per_sm = 1;
        TT_TRY(set_la_attr(ctx));
        TT_TRY(koccupancy(ctx, (const void*)tsqr_la_kernel, kLaThreads, la_smem_bytes(M), &per_sm));
        per_sm = std::max(1, per_sm);
        int64_t G = std::max<int64_t>(1, n / (4 * (int64_t)M));
        G = std::min<int64_t>(G, (int64_t)per_sm * ctx->num_sms);
        if (R_init) G = 1;
        TT_TRY(ensure(ctx->ws_R, (size_t)(G + 1) * RS * 8));
        double* parts = as<double>(ctx->ws_R);
        double* Rinit_ws = nullptr;
        if (R_init) {
            Rinit_ws = parts + RS;
            TT_TRY(pack_parts(ctx, R_init, 1, m, M, Rinit_ws));
        }
        BlkArgs a{X, n, ld, parts, Rinit_ws, m, M, 0, nullptr};
        kmark(ctx, 0, TTSVD_K_LA);
        TT_TRY(launch_blk(ctx, a, (int)G));
        kmark(ctx, 1, TTSVD_K_LA);
        if (G > 1) {
            const int rc = merge_stack_gqr(ctx, parts, G, m, M, R);
            if (rc != -1) return rc;
            TT_TRY(ensure(ctx->ws_P, (size_t)RS * 8));
            TT_TRY(merge_tree_blk(ctx, parts, G, m, M, as<double>(ctx->ws_P)));
            return copy_leading(ctx, as<double>(ctx->ws_P), M, m, R);
        }
        return copy_leading(ctx, parts, M, m, R);
    }
    if (cs.q && (R_init || m <= 8 || n < 4096)) return kNoView;
    if (!R_init && m <= 8 && n >= 4096) return tsqr_pt_device(ctx, X, n, m, ld, R);
    if (!R_init && n >= 4096) return tsqr_gs_device(ctx, X, n, m, ld, R, cs);
    TsqrPlan p = tsqr_plan(m);
    const int64_t min_rows = std::max<int64_t>(p.bt, 8 * (int64_t)m);
    int64_t G = std::max<int64_t>(1, n / min_rows);
    G = std::min<int64_t>(G, 2 * (int64_t)ctx->num_sms);
    if (R_init) G = 1;
    TT_TRY(ensure(ctx->ws_R, (size_t)G * m * m * 8));
    double* parts = as<double>(ctx->ws_R);
    TsqrArgs a{X, n, ld, G == 1 ? R : parts, m, p.bt, p.ldb, 0, p.r_in_smem, R_init};
    kmark(ctx, 0, TTSVD_K_V1);
    TT_TRY(launch_tsqr_kernel(ctx, a, (int)G, p.smem));
    kmark(ctx, 1, TTSVD_K_V1);
    if (G == 1) return TTSVD_OK;
    return merge_tree(ctx, parts, G, m, R);
}

// ----------------------------------------------------------------- K_SVD ----
int transpose_device(ttsvd_cu_ctx* ctx, const double* src, int64_t rows, int64_t cols, int64_t ld, double* dst) {
    dim3 block(32, 8);
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    transpose_kernel<<<grid, block, 0, ctx->stream>>>(src, rows, cols, ld, dst);
    return check_launch(ctx, "transpose_kernel");
}

constexpr int kJacobiThreads = 256;
constexpr int kJacobiSmemThreads = 512;

// One-sided Jacobi on A (n x m, ld n, device, overwritten).  With Vacc the
// rotations are accumulated.  Returns sweeps used via *sweeps.
// Cluster-resident block Jacobi (no accumulation, jacobi_blk.cuh).
int jacobi_bj(ttsvd_cu_ctx* ctx, double* A, int n, int m, int* status, bool* launched) {
    *launched = false;
    const int n8 = (n + 7) / 8 * 8;
    const int ldc = bj_ldc(n8);
    const int nblk = (m + 3) / 4;
    const int C = (nblk + 2 * kBjSlots - 1) / (2 * kBjSlots);
    const size_t smem = bj_smem_bytes(ldc);
    int static_smem = 0;
    TT_TRY(kstatic_smem((const void*)jacobi_bj_kernel, &static_smem));
    TT_TRY(kattr(ctx, (const void*)jacobi_bj_kernel, kSmemLimit - static_smem, true));
    if (C > 16 || smem > (size_t)(kSmemLimit - static_smem)) return TTSVD_OK;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kBjThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, jacobi_bj_kernel, &cfg) != cudaSuccess || ncl < 1) {
        (void)cudaGetLastError();
        return TTSVD_OK;
    }
    BjArgs ba{A, n, m, n8, ldc, C, status, 30, nullptr};
    TT_CUDA(cudaLaunchKernelEx(&cfg, jacobi_bj_kernel, ba));
    TT_TRY(check_launch(ctx, "jacobi_bj_kernel"));
    *launched = true;
    return TTSVD_OK;
}

int jacobi_device(ttsvd_cu_ctx* ctx, double* A, int n, int m, double* Vacc) {
    TT_TRY(ensure(ctx->ws_flags, 64 * sizeof(int)));
    int* flags = as<int>(ctx->ws_flags);
    TT_CUDA(cudaMemsetAsync(flags, 0, 64 * sizeof(int), ctx->stream));
    JacobiArgs a{A, Vacc, n, m, flags, flags + 40, 30};
    const size_t smem = ((size_t)n * m + (Vacc ? (size_t)m * m : 0)) * 8;
    if (!Vacc && m >= 96) {
        bool launched = false;
        TT_TRY(jacobi_bj(ctx, A, n, m, flags + 40, &launched));
        if (launched) return TTSVD_OK;
    }
    if (smem <= 220 * 1024) {
        TT_TRY(kattr(ctx, (const void*)jacobi_smem_kernel<kJacobiSmemThreads>, kSmemLimit));
        jacobi_smem_kernel<kJacobiSmemThreads><<<1, kJacobiSmemThreads, smem, ctx->stream>>>(a);
        TT_TRY(check_launch(ctx, "jacobi_smem_kernel"));
        return TTSVD_OK;
    }
    {
        const int warps_per = kJacobiThreads / 32;
        int grid = (m / 2 + warps_per - 1) / warps_per;
        grid = std::max(1, std::min(grid, ctx->coop_max_blocks));
        void* args[] = {&a};
        TT_CUDA(cudaLaunchCooperativeKernel((const void*)jacobi_coop_kernel<kJacobiThreads>, dim3(grid),
                                            dim3(kJacobiThreads), args, 0, ctx->stream));
        TT_TRY(check_launch(ctx, "jacobi_coop_kernel"));
    }
    return TTSVD_OK;
}

int jacobi_status(ttsvd_cu_ctx* ctx, int* sweeps) {
    int h = 0;
    TT_CUDA(cudaMemcpyAsync(&h, as<int>(ctx->ws_flags) + 40, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    TT_CUDA(cudaStreamSynchronize(ctx->stream));
    *sweeps = h;
    if (h < 0) return fail(TTSVD_ERR_CONVERGENCE, "jacobi_svd: no convergence in 30 sweeps");
    return TTSVD_OK;
}

int finalize_device(ttsvd_cu_ctx* ctx, const double* A, int n, int m, const double* Vacc, double* sigma, double* Uout,
                    double* Vout) {
    const size_t smem = (size_t)m * 8 + (size_t)2 * m * sizeof(int) + 64 * 8;
    jacobi_finalize_kernel<512><<<1, 512, smem, ctx->stream>>>(A, n, m, Vacc, sigma, Uout, Vout);
    return check_launch(ctx, "jacobi_finalize_kernel");
}

// Bidiagonal path (bidiag.cuh) of svd_work: sigma now, the vectors later by
// svd_vectors.  Returns -1 (nothing launched) when A does not fit the cluster.
// the bidiagonal path from m = 16 (config 2 steps 1 and 6: 0.17 -> 0.10 ms, 0.21 -> 0.12 ms)
constexpr int kBdMinM = 16;
// cluster size C and columns per CTA of the register-resident
// bidiagonalisation (C * cpc >= m).  Measured (config 1, m = 64 steps;
// config 2 m = 256 steps): 8 CTAs for m <= 128 (config 1 4.20 -> 4.09 ms),
// 16 above (m = 256 on 8 CTAs: 1.49 -> 1.96 ms; on 4: the same).
void bd_shape(int m, int* C, int* cpc) {
    const int c = m <= 128 ? 8 : kBdCluster;
    const int need = (m + c - 1) / c;
    *C = c;
    *cpc = need <= 8 ? 8 : (need <= 16 ? 16 : 32);
}

template <int CPC>
void (*bd_reg_for(int C))(BdArgs) {
    if constexpr (CPC <= 16)
        if (C == 8) return bd_reg_kernel<CPC, 8>;
    return bd_reg_kernel<CPC, kBdCluster>;
}

int bd_sigma(ttsvd_cu_ctx* ctx, double* A, int n, int m, double* sigma) {
    int C = kBdCluster, cpc = 8;
    const bool reg = n <= kBdThreads;
    if (reg) {
        bd_shape(m, &C, &cpc);
    } else {
        const int need = (m + kBdCluster - 1) / kBdCluster;
        cpc = need <= 8 ? 8 : (need <= 16 ? 16 : 32);
    }
    if ((m + C - 1) / C > 32 || n < m) return -1;
    void (*kern)(BdArgs) = reg ? (cpc == 8 ? bd_reg_for<8>(C) : (cpc == 16 ? bd_reg_for<16>(C) : bd_reg_for<32>(C)))
                               : (cpc == 8 ? bd_kernel<8> : (cpc == 16 ? bd_kernel<16> : bd_kernel<32>));
    const size_t smem = reg ? 0 : bd_smem_bytes(n, cpc);
    int ss = 0;
    TT_TRY(kstatic_smem((const void*)kern, &ss));
    TT_TRY(kattr(ctx, (const void*)kern, kSmemLimit - ss, true));
    if (smem > (size_t)(kSmemLimit - ss)) return -1;
    TT_TRY(ensure(ctx->ws_bd, ((size_t)3 * m + 2 * (size_t)(n + 1) + (size_t)kBdCluster * n + 32 * (kBdCluster + 1)) * 8));
    double* d = as<double>(ctx->ws_bd);
    double* e = d + m;
    double* tauL = e + m;
    double* xg = tauL + m;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kBdThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    BdArgs ba{A, n, m, cpc, d, e, tauL, xg, nullptr};
    TT_CUDA(cudaLaunchKernelEx(&cfg, kern, ba));
    TT_TRY(check_launch(ctx, "bd_kernel"));
    const int wpb = kBisThreads / 32;
    bd_bisect_kernel<<<(m + wpb - 1) / wpb, kBisThreads, (size_t)(2 * m) * 8, ctx->stream>>>(d, e, m, sigma);
    TT_TRY(check_launch(ctx, "bd_bisect_kernel"));
    ctx->bd_pending = true;
    ctx->bd_A = A;
    ctx->bd_n = n;
    ctx->bd_m = m;
    return TTSVD_OK;
}

// The leading r left singular vectors of svd_work's A (n x r, ld n) when the
// bidiagonal path ran; no-op after the Jacobi path (its Vout is complete).
int svd_vectors(ttsvd_cu_ctx* ctx, int64_t r, const double* sigma, double* Vout) {
    if (!ctx->bd_pending) return TTSVD_OK;
    ctx->bd_pending = false;
    const int n = ctx->bd_n, m = ctx->bd_m;
    if (r < 1) return TTSVD_OK;
    r = std::min<int64_t>(r, m);
    double* d = as<double>(ctx->ws_bd);
    double* e = d + m;
    double* tauL = e + m;
    TT_TRY(ensure(ctx->ws_Scr, (size_t)r * (7 * 2 * (size_t)m + m) * 8));
    double* scratch = as<double>(ctx->ws_Scr);
    double* X = scratch + (size_t)r * 7 * 2 * m;
    BdVecArgs va{d, e, sigma, m, (int)r, scratch, X};
    const size_t tsm = (size_t)kTwWarps * 4 * m * 8;
    TT_TRY(kattr(ctx, (const void*)bd_twisted_kernel, kSmemLimit));
    bd_twisted_kernel<<<(unsigned)((r + kTwWarps - 1) / kTwWarps), kTwWarps * 32, tsm, ctx->stream>>>(va);
    TT_TRY(check_launch(ctx, "bd_twisted_kernel"));
    // clusters (rare): inverse iteration with modified Gram-Schmidt
    bd_vectors_kernel<<<1, (unsigned)std::min<int64_t>(1024, (r + 31) / 32 * 32), 0, ctx->stream>>>(va);
    TT_TRY(check_launch(ctx, "bd_vectors_kernel"));
    if (n <= 512) {
        TT_TRY(kattr(ctx, (const void*)bd_back4s_kernel<8>, (int)bd_back4s_smem(8)));
        TT_TRY(kattr(ctx, (const void*)bd_back4s_kernel<16>, (int)bd_back4s_smem(16)));
        const unsigned gs = (unsigned)((r + kB4sVpw * kB4sWarps - 1) / (kB4sVpw * kB4sWarps));
        if (n <= 256)
            bd_back4s_kernel<8><<<gs, kB4sWarps * 32, bd_back4s_smem(8), ctx->stream>>>(ctx->bd_A, tauL, n, m, X,
                                                                                        (int)r, Vout);
        else
            bd_back4s_kernel<16><<<gs, kB4sWarps * 32, bd_back4s_smem(16), ctx->stream>>>(ctx->bd_A, tauL, n, m, X,
                                                                                          (int)r, Vout);
        return check_launch(ctx, "bd_back4s_kernel");
    }
    const size_t smem = (size_t)kBackWarps * n * 8;
    TT_TRY(kattr(ctx, (const void*)bd_back_kernel, kSmemLimit));
    bd_back_kernel<<<(unsigned)((r + kBackWarps - 1) / kBackWarps), kBackWarps * 32, smem, ctx->stream>>>(
        ctx->bd_A, tauL, n, m, X, (int)r, Vout);
    return check_launch(ctx, "bd_back_kernel");
}

// sigma and right singular vectors of a work matrix.
//   accumulate == true (the small_svd / jacobi_svd API, small_svd.hpp:72-114):
//     one-sided Jacobi on the columns of R with the rotations accumulated
//     into V — the reference's algorithm, V orthonormal to working precision
//     even for sigma ~ 0;
//   accumulate == false (the TT-SVD driver): one-sided Jacobi on the columns
//     of R^T (tall step) or W^T (wide step, tt_svd.hpp:91-103); the
//     orthogonalised columns are sigma_j v_j, so V := their normalisation
//     (with the reference's deterministic completion for sigma <= n eps
//     sigma_1).  No rotation accumulation, and Jacobi on the transposed
//     triangular factor converges in ~40% fewer sweeps (Drmac's observation;
//     15 -> 9 sweeps on config-2-like factors, tools/ measurements).  The
//     driver only consumes the leading r columns, with sigma_r above the
//     numerical-zero level (choose_rank), where this V is accurate.
// src is (src_rows x src_cols, ld); sigma gets nsig values, Vout is
// (cols x nsig, ld cols).
int svd_work(ttsvd_cu_ctx* ctx, const double* src, int64_t src_rows, int64_t src_cols, int64_t src_ld, bool transpose,
             bool accumulate, double* sigma, double* Vout, int* sweeps) {
    const int64_t n = transpose ? src_cols : src_rows;   // column length of A
    const int64_t m = transpose ? src_rows : src_cols;   // columns of A
    TT_TRY(ensure(ctx->ws_A, (size_t)n * m * 8));
    double* A = as<double>(ctx->ws_A);
    if (transpose) {
        TT_TRY(transpose_device(ctx, src, src_rows, src_cols, src_ld, A));
    } else {
        TT_CUDA(cudaMemcpy2DAsync(A, n * 8, src, src_ld * 8, n * 8, m, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    ctx->bd_pending = false;
    if (!accumulate) {
        if (m >= kBdMinM) {
            const int rc = bd_sigma(ctx, A, (int)n, (int)m, sigma);
            if (rc != -1) {
                *sweeps = 0;
                return rc;
            }
        }
        TT_TRY(jacobi_device(ctx, A, (int)n, (int)m, nullptr));
        TT_TRY(jacobi_status(ctx, sweeps));
        return finalize_device(ctx, A, (int)n, (int)m, nullptr, sigma, Vout, nullptr);
    }
    TT_TRY(ensure(ctx->ws_Vacc, (size_t)m * m * 8));
    TT_TRY(ensure(ctx->ws_U, (size_t)n * m * 8));
    double* Vacc = as<double>(ctx->ws_Vacc);
    TT_TRY(jacobi_device(ctx, A, (int)n, (int)m, Vacc));
    TT_TRY(jacobi_status(ctx, sweeps));
    return finalize_device(ctx, A, (int)n, (int)m, Vacc, sigma, as<double>(ctx->ws_U), Vout);
}

// ---------------------------------------------------------------- K_TSMM ----
template <int KC>
int launch_tsmm(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ldx, const double* V, int64_t ldv, int k,
                double* Y, int64_t out_rows, int64_t ldy) {
    const size_t smem = (size_t)m * KC * 8;
    if (smem > (size_t)kSmemLimit) return fail(TTSVD_ERR_SHAPE, "tsmm_kernel: V block exceeds shared memory");
    TT_TRY(kattr(ctx, (const void*)tsmm_kernel<KC>, kSmemLimit));
    const int chunks = (k + KC - 1) / KC;
    int64_t blocks = (n + 255) / 256;
    blocks = std::min<int64_t>(blocks, (int64_t)ctx->num_sms * 8);
    dim3 grid((unsigned)std::max<int64_t>(blocks, 1), (unsigned)chunks);
    tsmm_kernel<KC><<<grid, 256, smem, ctx->stream>>>(X, n, m, ldx, V, ldv, k, Y, out_rows, ldy);
    return check_launch(ctx, "tsmm_kernel");
}

template <int KC>
int launch_tsmm_async(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ldx, const double* V, int64_t ldv,
                      int k, double* Y, int64_t out_rows, int64_t ldy) {
    const size_t smem = ((size_t)((m * KC + 1) & ~1) + (size_t)2 * m * 256) * 8;
    int per_sm = 1;
    TT_TRY(kattr(ctx, (const void*)tsmm_async_kernel<KC>, kSmemLimit));
    TT_TRY(koccupancy(ctx, (const void*)tsmm_async_kernel<KC>, 256, smem, &per_sm));
    const int64_t chunks = (n + 255) / 256;
    const int64_t blocks = std::min<int64_t>(chunks, (int64_t)std::max(1, per_sm) * ctx->num_sms);
    const int ychunks = (k + KC - 1) / KC;
    tsmm_async_kernel<KC><<<dim3((unsigned)blocks, (unsigned)ychunks), 256, smem, ctx->stream>>>(X, n, m, ldx, V, ldv,
                                                                                              k, Y, out_rows, ldy);
    return check_launch(ctx, "tsmm_async_kernel");
}

template <int KC>
int launch_tsmm_async_wide(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ldx, const double* V,
                           int64_t ldv, int k, double* Y, int64_t out_rows, int64_t ldy) {
    const size_t smem = ((size_t)((m * KC + 1) & ~1) + (size_t)2 * 32 * 256) * 8;
    if (smem > (size_t)kSmemLimit) return -1;
    TT_TRY(kattr(ctx, (const void*)tsmm_async_wide_kernel<KC>, kSmemLimit));
    int per_sm = 1;
    TT_TRY(koccupancy(ctx, (const void*)tsmm_async_wide_kernel<KC>, 256, smem, &per_sm));
    const int64_t chunks = (n + 255) / 256;
    const int64_t blocks = std::min<int64_t>(chunks, (int64_t)std::max(1, per_sm) * ctx->num_sms);
    const int ychunks = (k + KC - 1) / KC;
    tsmm_async_wide_kernel<KC><<<dim3((unsigned)blocks, (unsigned)ychunks), 256, smem, ctx->stream>>>(
        X, n, m, ldx, V, ldv, k, Y, out_rows, ldy);
    return check_launch(ctx, "tsmm_async_wide_kernel");
}

template <int NT>
int launch_tsmm_dmma(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ldx, const double* V, int64_t ldv,
                     int k, double* Y, int64_t out_rows, int64_t ldy) {
    const size_t smem = (size_t)((m + 3) & ~3) * tsmm_vld(NT) * 8;
    TT_TRY(kattr(ctx, (const void*)tsmm_dmma_kernel<NT>, kSmemLimit));
    const int chunks = (k + 8 * NT - 1) / (8 * NT);
    int64_t blocks = (n + 255) / 256;
    blocks = std::min<int64_t>(blocks, (int64_t)ctx->num_sms * 4);
    dim3 grid((unsigned)std::max<int64_t>(blocks, 1), (unsigned)chunks);
    tsmm_dmma_kernel<NT><<<grid, 256, smem, ctx->stream>>>(X, n, m, ldx, V, ldv, k, Y, out_rows, ldy);
    return check_launch(ctx, "tsmm_dmma_kernel");
}

int tsmm_device(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int m, int64_t ldx, const double* V, int64_t ldv, int k,
                double* Y, int64_t out_rows, int64_t out_cols, int64_t ldy, ColSplit cs = ColSplit{0, 0}) {
    int rc;
    // FP64 tensor cores once the FMA kernels turn compute-bound (k > 8 output
    // columns, m >= 32): rows staged by TMA bulk copies (tsmm_dt.cuh), one
    // persistent CTA per SM; fragments straight from X (tsmm_dmma_kernel) when
    // the staged kernel's alignment / divisibility conditions do not hold
    const int dt_nt = k > 16 ? 4 : 2;
    const int dt_stages = dt_smem_bytes(m, 4, dt_nt) <= (size_t)kSmemLimit - 2048 ? 4 : 2;
    const bool dt = k > 8 && m >= 32 && n >= (int64_t)1 << 16 && n % kDtRows == 0 && m % kDtCols == 0 &&
                    (ldx & 1) == 0 && ((uintptr_t)X & 15) == 0 && (cs.q == 0 || (cs.ld_lo & 1) == 0) &&
                    dt_smem_bytes(m, dt_stages, dt_nt) <= (size_t)kSmemLimit - 2048;
    if (cs.q && !dt) return kNoView;  // only the TMA-staged kernel reads a split-column view
    const bool dmma = !dt && k > 16 && m >= 32 && n >= (int64_t)1 << 18 &&
                      (size_t)((m + 3) & ~3) * tsmm_vld(4) * 8 <= 200 * 1024;
    if (dt || dmma) {
        if (dt) {
            void (*fn)(const double*, int64_t, int, int64_t, const double*, int64_t, int, double*, int64_t, int64_t,
                       ColSplit) =
                dt_nt == 4 ? (dt_stages == 4 ? tsmm_dt_kernel<4, 4> : tsmm_dt_kernel<2, 4>)
                           : (dt_stages == 4 ? tsmm_dt_kernel<4, 2> : tsmm_dt_kernel<2, 2>);
            TT_TRY(kattr(ctx, (const void*)fn, kSmemLimit - 2048));
            dim3 grid((unsigned)std::min<int64_t>(ctx->num_sms, (n / kDtRows + 7) / 8),
                      (unsigned)((k + 8 * dt_nt - 1) / (8 * dt_nt)));
            fn<<<grid, 256, dt_smem_bytes(m, dt_stages, dt_nt), ctx->stream>>>(X, n, m, ldx, V, ldv, k, Y, out_rows, ldy, cs);
            rc = check_launch(ctx, "tsmm_dt_kernel");
        } else {
            rc = launch_tsmm_dmma<4>(ctx, X, n, m, ldx, V, ldv, k, Y, out_rows, ldy);
        }
        if (rc != TTSVD_OK) return rc;
        if (ldy > out_rows) {
            const int64_t pad = (ldy - out_rows) * out_cols;
            const int blocks = (int)std::min<int64_t>((pad + 255) / 256, 1024);
            zero_padding_kernel<<<std::max(blocks, 1), 256, 0, ctx->stream>>>(Y, out_rows, ldy, out_cols);
            return check_launch(ctx, "zero_padding_kernel");
        }
        return TTSVD_OK;
    }
    if (n <= (int64_t)1 << 14 && m >= 32 && (size_t)(m + 256) * 8 * 8 <= (size_t)kSmemLimit) {
        // short X (the last steps of a chain): 32 rows x 8 output columns per
        // CTA, the contraction split over its warps
        const size_t smem = (size_t)(m + 256) * 8 * 8;
        TT_TRY(kattr(ctx, (const void*)tsmm_small_kernel<8>, kSmemLimit));
        dim3 grid((unsigned)((n + 31) / 32), (unsigned)((k + 7) / 8));
        tsmm_small_kernel<8><<<grid, 256, smem, ctx->stream>>>(X, n, m, ldx, V, ldv, k, Y, out_rows, ldy);
        rc = check_launch(ctx, "tsmm_small_kernel");
    } else if (k > 1 && k <= 16 && m <= 32 && n >= (int64_t)1 << 18) {
        // narrow X: rows staged by cp.async (tsmm_async_kernel; measured
        // against TMA bulk staging, tools/tsmm_bulk_experiment.cuh)
        rc = k <= 4 ? launch_tsmm_async<4>(ctx, X, n, m, ldx, V, ldv, k, Y, out_rows, ldy)
                    : (k <= 8 ? launch_tsmm_async<8>(ctx, X, n, m, ldx, V, ldv, k, Y, out_rows, ldy)
                              : launch_tsmm_async<16>(ctx, X, n, m, ldx, V, ldv, k, Y, out_rows, ldy));
    } else if (k > 1 && k <= 32 && m > 32 && n >= (int64_t)1 << 16 && !dmma &&
               (rc = k <= 4 ? launch_tsmm_async_wide<4>(ctx, X, n, m, ldx, V, ldv, k, Y, out_rows, ldy)
                            : (k <= 8 ? launch_tsmm_async_wide<8>(ctx, X, n, m, ldx, V, ldv, k, Y, out_rows, ldy)
                                      : (k <= 16 || (size_t)m * 32 * 8 + 2 * 32 * 256 * 8 > (size_t)kSmemLimit
                                             ? launch_tsmm_async_wide<16>(ctx, X, n, m, ldx, V, ldv, k, Y, out_rows, ldy)
                                             : launch_tsmm_async_wide<32>(ctx, X, n, m, ldx, V, ldv, k, Y, out_rows,
                                                                          ldy)))) != -1) {
        // wider X: column blocks of the row chunk staged by cp.async
    } else {
        // KC output columns per CTA pass, capped so V's m x KC block fits
        // shared memory (more column chunks on grid.y otherwise)
        int kc = k <= 1 ? 1 : (k <= 2 ? 2 : (k <= 4 ? 4 : (k <= 8 ? 8 : (k <= 16 ? 16 : 32))));
        while (kc > 1 && (size_t)m * kc * 8 > (size_t)kTsmmSmem) kc /= 2;
        switch (kc) {
            case 1: rc = launch_tsmm<1>(ctx, X, n, m, ldx, V, ldv, k, Y, out_rows, ldy); break;
            case 2: rc = launch_tsmm<2>(ctx, X, n, m, ldx, V, ldv, k, Y, out_rows, ldy); break;
            case 4: rc = launch_tsmm<4>(ctx, X, n, m, ldx, V, ldv, k, Y, out_rows, ldy); break;
            case 8: rc = launch_tsmm<8>(ctx, X, n, m, ldx, V, ldv, k, Y, out_rows, ldy); break;
            case 16: rc = launch_tsmm<16>(ctx, X, n, m, ldx, V, ldv, k, Y, out_rows, ldy); break;
            default: rc = launch_tsmm<32>(ctx, X, n, m, ldx, V, ldv, k, Y, out_rows, ldy); break;
        }
    }
    if (rc != TTSVD_OK) return rc;
    if (ldy > out_rows) {
        const int64_t pad = (ldy - out_rows) * out_cols;
        const int blocks = (int)std::min<int64_t>((pad + 255) / 256, 1024);
        zero_padding_kernel<<<blocks, 256, 0, ctx->stream>>>(Y, out_rows, ldy, out_cols);
        TT_TRY(check_launch(ctx, "zero_padding_kernel"));
    }
    return TTSVD_OK;
}

// --------------------------------------------------------------- drivers ----
// tt_svd.hpp:111-118 choose_rank + small_svd.hpp:49-63 select_rank (host
// scalar arithmetic on the singular values copied back once per step).
int64_t select_rank_h(const double* sigma, int64_t m, double delta, int64_t r_max) {
    double tail = 0.0;
    int64_t r_delta = m;
    for (int64_t j = m; j-- > 0;) {
        tail += sigma[j] * sigma[j];
        if (tail <= delta * delta) r_delta = j;
        else break;
    }
    int64_t r = std::min(r_max, r_delta);
    if (r < 1) r = 1;
    return std::min(r, std::max<int64_t>(m, 1));
}

int64_t choose_rank_h(const double* sigma, int64_t len, int64_t cols, int64_t nsig, double delta, int64_t r_max,
                      int64_t rows) {
    const double sigma1 = len > 0 ? sigma[0] : 0.0;
    const double zero_level = 32.0 * DBL_EPSILON * sigma1 * std::sqrt((double)std::max(rows, cols));
    const double delta_eff = std::max(delta, zero_level);
    return std::min(select_rank_h(sigma, len, delta_eff, r_max), nsig);
}

double sigma_norm_h(const double* s, int64_t m) {
    double t = 0.0;
    for (int64_t j = 0; j < m; ++j) t += s[j] * s[j];
    return std::sqrt(t);
}

// K6, the rank rule on the device (derive_delta / select_rank / choose_rank,
// small_svd.hpp:41-63, tt_svd.hpp:111-118): one thread repeats
// choose_rank_h's arithmetic operation by operation (explicit round-to-nearest
// multiplies and adds, no contraction) on the step's sigmas and leaves
// (rank, sum sigma^2) in device memory, so a chain can run without a host
// round trip per step.
__global__ void rank_epilogue_kernel(const double* __restrict__ sigma, int64_t len, int64_t cols, int64_t nsig,
                                     double delta, int64_t r_max, int64_t rows, double* __restrict__ rec) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double sigma1 = len > 0 ? sigma[0] : 0.0;
    const double zero_level =
        __dmul_rn(__dmul_rn(__dmul_rn(32.0, DBL_EPSILON), sigma1), sqrt((double)(rows > cols ? rows : cols)));
    const double delta_eff = delta > zero_level ? delta : zero_level;
    const double d2 = __dmul_rn(delta_eff, delta_eff);
    double tail = 0.0;
    int64_t r_delta = len;
    for (int64_t j = len; j-- > 0;) {
        tail = __dadd_rn(tail, __dmul_rn(sigma[j], sigma[j]));
        if (tail <= d2) r_delta = j;
        else break;
    }
    int64_t r = r_max < r_delta ? r_max : r_delta;
    if (r < 1) r = 1;
    const int64_t cap = len > 1 ? len : 1;
    if (r > cap) r = cap;
    if (r > nsig) r = nsig;
    double t = 0.0;
    for (int64_t j = 0; j < len; ++j) t = __dadd_rn(t, __dmul_rn(sigma[j], sigma[j]));
    rec[0] = (double)r;
    rec[1] = t;  // ||Sigma||_F^2 (sigma_norm_h squares and sums in the same order)
}

// the rank choose_rank_h returns when no sigma tail falls below delta_eff
int64_t predicted_rank_h(int64_t len, int64_t nsig, int64_t r_max) {
    int64_t r = std::min(r_max, len);
    if (r < 1) r = 1;
    r = std::min(r, std::max<int64_t>(len, 1));
    return std::min(r, nsig);
}

constexpr int kMispredict = -1000;  // internal: a speculative chain met a rank below its prediction

struct Timer {
    ttsvd_cu_ctx* ctx;
    bool on;
    explicit Timer(ttsvd_cu_ctx* c) : ctx(c), on(c->timing) {}
    void mark(int i) {
        if (on) cudaEventRecord(ctx->ev[i], ctx->stream);
    }
    double ms(int a, int b) {
        if (!on) return 0.0;
        float t = 0.f;
        cudaEventSynchronize(ctx->ev[b]);
        cudaEventElapsedTime(&t, ctx->ev[a], ctx->ev[b]);
        return (double)t;
    }
};

struct WorkView {
    const double* data;
    int64_t rows, cols, ld;
};

// D2H of `count` doubles through the pinned stage (synchronises the stream).
int d2h(ttsvd_cu_ctx* ctx, double* dst, const double* src, size_t count) {
    TT_TRY(ensure_host(ctx->host_stage, count * 8));
    TT_CUDA(cudaMemcpyAsync(ctx->host_stage.p, src, count * 8, cudaMemcpyDeviceToHost, ctx->stream));
    TT_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(dst, ctx->host_stage.p, count * 8);
    return TTSVD_OK;
}

// Alg. 2 loop (tt_svd.hpp:159-199).
// delta_io: in, a truncation parameter (< 0: derive it from the first step,
// small_svd.hpp:41 — run_chain takes the spec by reference, tt_svd.hpp:160);
// out, the one used.  first_sigma_norm_out: ||Sigma||_F of the first step
// (ChainResult::first_sigma_norm, tt_svd.hpp:153-156).
//
// spec: the chain runs without a host round trip per step.  Every step's
// rank is PREDICTED on the host (min(r_max, #sigma): what the rule gives
// unless a sigma tail falls below delta_eff), the true rank is computed on
// the device by rank_epilogue_kernel (K6) and lands, with the sigmas, in
// pinned memory; after the one synchronisation that ends the chain the
// records are compared and a chain that met a smaller rank anywhere returns
// kMispredict (the caller runs it again step by step).  Only used when delta
// is known up front (eps = 0, or a given delta of 0).
// cs0: the column layout of the FIRST work matrix (thick-bounds' merged view
// of X, read in place by K_TSQR / K_TSMM; kNoView when the first step's TSQR
// kernel cannot, before anything has run).
int run_chain_impl(ttsvd_cu_ctx* ctx, WorkView cur, const std::vector<int64_t>& dims, int64_t r_max, double eps,
                   int64_t d_for_delta, ttsvd_cu_tt* out, double* delta_io, double* first_sigma_norm_out,
                   bool spec, ColSplit cs0, const double* R_first) {
    const int64_t d = (int64_t)dims.size();
    out->dims = dims;
    out->cores.assign(d, {});
    out->ranks.assign(d + 1, 1);
    out->steps.clear();
    out->sigmas.clear();
    double delta = delta_io ? *delta_io : -1.0;
    struct SpecStep {
        size_t off;  // of the step's record in host_sig (doubles): nsig sigmas, then (rank, sum sigma^2)
        int64_t nsig, pred;
        size_t step;  // index into out->steps / out->sigmas
    };
    // Which steps run ahead of their rank: only those whose prediction is the
    // cap r_max, and only once a step checked on the host has reached the cap
    // (a train that saturates r_max at one unfolding does so at the next);
    // while the ranks still grow with the matrix, and after any checked step
    // came out below its prediction (a rank-deficient tensor), the step waits
    // for its sigmas as before.  A speculated step that misses still costs a
    // rerun of the chain.
    bool trust = false;
    std::vector<SpecStep> spec_steps;
    size_t spec_off = 0;
    if (spec) {
        if (delta < 0.0) {
            if (d_for_delta < 2) return fail(TTSVD_ERR_DEGENERATE, "derive_delta: requires d >= 2");
            delta = 0.0;  // eps = 0: delta = 0 whatever the first step's norm is
        }
        // the predicted shapes give the size of the pinned record arena
        size_t need = 0;
        int64_t rows_s = cur.rows, r_s = 1;
        for (int64_t i = d - 1; i >= 1; --i) {
            const int64_t m_s = dims[i] * r_s;
            const int64_t nsig_s = std::min(m_s, rows_s);
            need += (size_t)nsig_s + 2;
            r_s = predicted_rank_h(nsig_s, nsig_s, r_max);
            rows_s /= dims[i - 1];
        }
        TT_TRY(ensure_host(ctx->host_sig, need * 8));
        TT_TRY(ensure(ctx->ws_rank, (size_t)d * 2 * 8));
    }
    int64_t r = 1;
    int which = 0;
    Timer tm(ctx);
    std::vector<double> sig;
    struct PendingCore {
        int64_t i;
        size_t off;
        int64_t m, rnew, n_i, r;
    };
    std::vector<PendingCore> pending;
    size_t core_off = 0;
    // build the cores whose V blocks have landed in the arena (stream synchronised)
    auto flush_cores = [&]() {
        const double* base = as<double>(ctx->host_cores);
        for (const PendingCore& pc : pending) {
            const double* Vh = base + pc.off;
            std::vector<double> core((size_t)(pc.rnew * pc.n_i * pc.r));
            for (int64_t b = 0; b < pc.r; ++b)
                for (int64_t x = 0; x < pc.n_i; ++x)
                    for (int64_t a = 0; a < pc.rnew; ++a)
                        core[a + pc.rnew * (x + pc.n_i * b)] = Vh[a * pc.m + (x + pc.n_i * b)];
            out->cores[pc.i] = std::move(core);
        }
        pending.clear();
        core_off = 0;
    };
    for (int64_t i = d - 1; i >= 1; --i) {
        const int64_t n_i = dims[i];
        const int64_t m = n_i * r;
        if (m != cur.cols) return fail(TTSVD_ERR_SHAPE, "run_chain: work matrix width mismatch");
        ttsvd_cu_step st{};
        st.rows = cur.rows;
        st.cols = m;
        const bool tall = cur.rows >= cur.cols;
        const ColSplit cs = (i == d - 1) ? cs0 : ColSplit{0, 0};
        if (cs.q && !tall) return kNoView;
        const int64_t nsig = tall ? m : cur.rows;
        TT_TRY(ensure(ctx->ws_sigma, (size_t)std::max<int64_t>(m, nsig) * 8));
        TT_TRY(ensure(ctx->ws_V, (size_t)m * std::max<int64_t>(nsig, 1) * 8));
        double* d_sigma = as<double>(ctx->ws_sigma);
        double* d_V = as<double>(ctx->ws_V);
        int sweeps = 0;
        tm.mark(0);
        if (tall) {
            TT_TRY(ensure(ctx->ws_X, (size_t)m * m * 8));
            double* R = as<double>(ctx->ws_X);
            if (i == d - 1 && R_first) {
                // the host entry factored the first work matrix while X was arriving
                if (R_first != R) TT_CUDA(cudaMemcpyAsync(R, R_first, (size_t)m * m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
                ctx->last_kernel = TTSVD_K_GT;
            } else {
                TT_TRY(tsqr_device(ctx, cur.data, cur.rows, (int)m, cur.ld, R, nullptr, cs));
            }
            tm.mark(1);
            TT_TRY(svd_work(ctx, R, m, m, m, true, false, d_sigma, d_V, &sweeps));
        } else {
            tm.mark(1);
            // wide step (tt_svd.hpp:91-103): Jacobi on W^T, V := its U
            TT_TRY(svd_work(ctx, cur.data, cur.rows, cur.cols, cur.ld, true, false, d_sigma, d_V, &sweeps));
        }
        tm.mark(2);
        sig.resize(nsig);
        int64_t rnew;
        const int64_t pred = predicted_rank_h(nsig, nsig, r_max);
        if (spec && trust && pred == r_max) {
            double* rec = as<double>(ctx->ws_rank) + 2 * (size_t)spec_steps.size();
            rank_epilogue_kernel<<<1, 32, 0, ctx->stream>>>(d_sigma, nsig, cur.cols, nsig, delta, r_max, cur.rows, rec);
            TT_TRY(check_launch(ctx, "rank_epilogue_kernel"));
            double* hs = as<double>(ctx->host_sig) + spec_off;
            TT_CUDA(cudaMemcpyAsync(hs, d_sigma, (size_t)nsig * 8, cudaMemcpyDeviceToHost, ctx->stream));
            TT_CUDA(cudaMemcpyAsync(hs + nsig, rec, 16, cudaMemcpyDeviceToHost, ctx->stream));
            rnew = pred;
            spec_steps.push_back(SpecStep{spec_off, nsig, rnew, out->steps.size()});
            spec_off += (size_t)nsig + 2;
        } else {
            TT_TRY(d2h(ctx, sig.data(), d_sigma, nsig));
            if (i == d - 1 && first_sigma_norm_out) *first_sigma_norm_out = sigma_norm_h(sig.data(), nsig);
            if (delta < 0.0) {
                if (d_for_delta < 2) return fail(TTSVD_ERR_DEGENERATE, "derive_delta: requires d >= 2");
                delta = eps / std::sqrt((double)(d_for_delta - 1)) * sigma_norm_h(sig.data(), nsig);
                if (delta_io) *delta_io = delta;
            }
            rnew = choose_rank_h(sig.data(), nsig, cur.cols, nsig, delta, r_max, cur.rows);
            if (rnew < pred) spec = false;             // rank-deficient: no more running ahead
            else if (pred == r_max) trust = true;      // the cap is reached
        }
        st.nsig = nsig;
        st.rank = rnew;
        tm.mark(7);
        TT_TRY(svd_vectors(ctx, rnew, d_sigma, d_V));
        tm.mark(8);
        // core_from_vt (tt_svd.hpp:121-128) from the first rnew columns of V:
        // an asynchronous D2H into the pinned core arena, the core is built
        // after the chain (one host round trip per step instead of two)
        {
            const size_t need = (size_t)m * rnew;
            if (core_off + need > ctx->host_cores.bytes / 8) {
                TT_CUDA(cudaStreamSynchronize(ctx->stream));
                flush_cores();
                TT_TRY(ensure_host(ctx->host_cores, std::max<size_t>(need, (size_t)1 << 20) * 8 * 2));
            }
            TT_CUDA(cudaMemcpyAsync(as<double>(ctx->host_cores) + core_off, d_V, need * 8, cudaMemcpyDeviceToHost,
                                    ctx->stream));
            pending.push_back(PendingCore{i, core_off, m, rnew, n_i, r});
            core_off += need;
        }
        out->ranks[i] = rnew;
        // fused TSMM + reshape into the next step's padded layout
        const int64_t n_next = dims[i - 1];
        const int64_t out_rows = cur.rows / n_next;
        const int64_t out_cols = n_next * rnew;
        const int64_t ldy = padded_stride_h(out_rows);
        TT_TRY(ensure(ctx->ws_work[which], (size_t)ldy * out_cols * 8));
        double* Y = as<double>(ctx->ws_work[which]);
        tm.mark(3);
        {
            int rc = tsmm_device(ctx, cur.data, cur.rows, (int)m, cur.ld, d_V, m, (int)rnew, Y, out_rows, out_cols, ldy, cs);
            if (rc == kNoView) {
                // the rank left the kernel that reads the view: materialise it
                // (copy_logical, storage.hpp:158-172) for this one product
                const int64_t ldm = padded_stride_h(cur.rows);
                TT_TRY(ensure(ctx->ws_thick[0], (size_t)ldm * m * 8));
                double* Wm = as<double>(ctx->ws_thick[0]);
                for (int64_t id = 0; id < m / cs.q; ++id)
                    TT_CUDA(cudaMemcpy2DAsync(Wm + id * cs.q * ldm, (size_t)ldm * 8, cur.data + id * cur.ld,
                                              (size_t)cs.ld_lo * 8, (size_t)cur.rows * 8, (size_t)cs.q,
                                              cudaMemcpyDeviceToDevice, ctx->stream));
                rc = tsmm_device(ctx, Wm, cur.rows, (int)m, ldm, d_V, m, (int)rnew, Y, out_rows, out_cols, ldy);
            }
            if (rc != TTSVD_OK) return rc;
        }
        tm.mark(4);
        if (tm.on) {
            st.t_tsqr_ms = tm.ms(0, 1);
            st.t_svd_ms = tm.ms(1, 2) + tm.ms(7, 8);  // sigmas + the leading vectors
            st.t_tsmm_ms = tm.ms(3, 4);
            if (tall && ctx->last_kernel) st.t_tsqr_sweep_ms = tm.ms(5, 6);
        }
        st.tsqr_kernel = tall ? ctx->last_kernel : TTSVD_K_NONE;
        st.svd_sweeps = sweeps;
        out->steps.push_back(st);
        out->sigmas.push_back(sig);
        cur = WorkView{Y, out_rows, out_cols, ldy};
        which ^= 1;
        r = rnew;
    }
    // T^(1): the final 1 x (n_1 r_1) work matrix (tt_svd.hpp:193-197)
    std::vector<double> first((size_t)(dims[0] * r));
    if (cur.rows == 1) {
        // row 0 of every column: stride ld
        std::vector<double> tmp((size_t)cur.cols);
        TT_TRY(ensure_host(ctx->host_stage, (size_t)cur.cols * 8));
        TT_CUDA(cudaMemcpy2DAsync(ctx->host_stage.p, 8, cur.data, cur.ld * 8, 8, cur.cols, cudaMemcpyDeviceToHost,
                                  ctx->stream));
        TT_CUDA(cudaStreamSynchronize(ctx->stream));
        std::memcpy(first.data(), ctx->host_stage.p, (size_t)cur.cols * 8);
    } else {
        for (int64_t l = 0; l < dims[0] * r; ++l) {
            double v;
            TT_TRY(d2h(ctx, &v, cur.data + (l / cur.rows) * cur.ld + l % cur.rows, 1));
            first[l] = v;
        }
    }
    TT_CUDA(cudaStreamSynchronize(ctx->stream));
    if (!spec_steps.empty()) {
        // the device's ranks against the predictions those steps ran with
        const double* base = as<double>(ctx->host_sig);
        for (const SpecStep& ss : spec_steps) {
            const double* hs = base + ss.off;
            if ((int64_t)hs[ss.nsig] != ss.pred) {
                pending.clear();
                return kMispredict;
            }
            out->sigmas[ss.step].assign(hs, hs + ss.nsig);
        }
    }
    if (delta_io && delta >= 0.0) *delta_io = delta;
    flush_cores();
    out->cores[0] = std::move(first);
    out->ranks[0] = 1;
    out->ranks[1] = r;
    out->ranks[d] = 1;
    return TTSVD_OK;
}

int run_chain(ttsvd_cu_ctx* ctx, WorkView cur, const std::vector<int64_t>& dims, int64_t r_max, double eps,
              int64_t d_for_delta, ttsvd_cu_tt* out, double* delta_io = nullptr,
              double* first_sigma_norm_out = nullptr, ColSplit cs0 = ColSplit{0, 0},
              const double* R_first = nullptr) {
    const double delta_in = delta_io ? *delta_io : -1.0;
    // timing reads its events step by step, so a timed chain runs step by step
    const bool spec = !ctx->timing && (delta_in < 0.0 ? eps == 0.0 : delta_in == 0.0);
    if (spec) {
        const int rc = run_chain_impl(ctx, cur, dims, r_max, eps, d_for_delta, out, delta_io, first_sigma_norm_out, true, cs0, R_first);
        if (rc != kMispredict) return rc;
        if (delta_io) *delta_io = delta_in;
        R_first = nullptr;  // its buffer has been reused by the later steps: factor again
    }
    return run_chain_impl(ctx, cur, dims, r_max, eps, d_for_delta, out, delta_io, first_sigma_norm_out, false, cs0,
                          R_first);
}

// tsmm.hpp:84-126 transpose_reorder: Y (out_rows x out_cols, ld ldy) <- the
// flat order of W^T; padding rows zeroed.
int transpose_reorder_device(ttsvd_cu_ctx* ctx, const double* W, int64_t n, int64_t m, int64_t ldw, double* Y,
                             int64_t out_rows, int64_t out_cols, int64_t ldy) {
    const int64_t tiles = ((n + 31) / 32) * ((m + 31) / 32);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)ctx->num_sms * 8));
    transpose_reorder_kernel<<<(unsigned)grid, dim3(32, 8), 0, ctx->stream>>>(W, n, m, ldw, Y, out_rows, ldy);
    TT_TRY(check_launch(ctx, "transpose_reorder_kernel"));
    if (ldy > out_rows) {
        const int64_t pad = (ldy - out_rows) * out_cols;
        const int blocks = (int)std::min<int64_t>((pad + 255) / 256, 1024);
        zero_padding_kernel<<<std::max(blocks, 1), 256, 0, ctx->stream>>>(Y, out_rows, ldy, out_cols);
        TT_TRY(check_launch(ctx, "zero_padding_kernel"));
    }
    return TTSVD_OK;
}

// The first `count` flat (column-major) entries of a padded device matrix
// (rows x ?, ld) on the host: core_from_padded (tt_svd.hpp:140-147).
int flat_d2h(ttsvd_cu_ctx* ctx, const double* M, int64_t rows, int64_t ld, int64_t count, std::vector<double>& out) {
    const int64_t cols = (count + rows - 1) / rows;
    TT_TRY(ensure_host(ctx->host_stage, (size_t)rows * cols * 8));
    TT_CUDA(cudaMemcpy2DAsync(ctx->host_stage.p, (size_t)rows * 8, M, (size_t)ld * 8, (size_t)rows * 8, (size_t)cols,
                              cudaMemcpyDeviceToHost, ctx->stream));
    TT_CUDA(cudaStreamSynchronize(ctx->stream));
    out.assign(as<double>(ctx->host_stage), as<double>(ctx->host_stage) + count);
    return TTSVD_OK;
}

// Two-sided sweep (Alg. 4, tt_svd.hpp:402-512): steps alternate between the
// right end (core from V^T, as run_chain) and the left end (core from V);
// each step's TSMM output is re-laid out by transpose_reorder for the
// opposite end.  Same kernels as run_chain (K_TSQR, K_SVD, K_TSMM) plus the
// reorder.
int run_two_sided(ttsvd_cu_ctx* ctx, WorkView cur, const std::vector<int64_t>& dims, int64_t r_max, double eps,
                  ttsvd_cu_tt* out) {
    const int64_t d = (int64_t)dims.size();
    out->dims = dims;
    out->cores.assign(d, {});
    std::vector<int64_t> rl(d, 1), rr(d, 1);  // core shapes
    int64_t lo = 0, hi = d - 1, r_left = 1, r_right = 1, built = 0;
    bool right = true;
    double delta = -1.0;
    int which = 0;
    std::vector<double> sig, Vh, flat;
    Timer tm(ctx);
    while (built < d - 1) {
        ttsvd_cu_step st{};
        const int64_t m = cur.cols;
        st.rows = cur.rows;
        st.cols = m;
        const bool tall = cur.rows >= cur.cols;
        const int64_t nsig = tall ? m : cur.rows;
        TT_TRY(ensure(ctx->ws_sigma, (size_t)std::max<int64_t>(m, nsig) * 8));
        TT_TRY(ensure(ctx->ws_V, (size_t)m * std::max<int64_t>(nsig, 1) * 8));
        double* d_sigma = as<double>(ctx->ws_sigma);
        double* d_V = as<double>(ctx->ws_V);
        int sweeps = 0;
        tm.mark(0);
        if (tall) {
            TT_TRY(ensure(ctx->ws_X, (size_t)m * m * 8));
            double* R = as<double>(ctx->ws_X);
            TT_TRY(tsqr_device(ctx, cur.data, cur.rows, (int)m, cur.ld, R));
            tm.mark(1);
            TT_TRY(svd_work(ctx, R, m, m, m, true, false, d_sigma, d_V, &sweeps));
        } else {
            tm.mark(1);
            TT_TRY(svd_work(ctx, cur.data, cur.rows, cur.cols, cur.ld, true, false, d_sigma, d_V, &sweeps));
        }
        tm.mark(2);
        sig.resize(nsig);
        TT_TRY(d2h(ctx, sig.data(), d_sigma, nsig));
        if (delta < 0.0) {
            if (d < 2) return fail(TTSVD_ERR_DEGENERATE, "derive_delta: requires d >= 2");
            delta = eps / std::sqrt((double)(d - 1)) * sigma_norm_h(sig.data(), nsig);
        }
        const int64_t rnew = choose_rank_h(sig.data(), nsig, cur.cols, nsig, delta, r_max, cur.rows);
        TT_TRY(svd_vectors(ctx, rnew, d_sigma, d_V));
        Vh.resize((size_t)m * rnew);
        TT_TRY(d2h(ctx, Vh.data(), d_V, (size_t)m * rnew));
        st.nsig = nsig;
        st.rank = rnew;
        st.svd_sweeps = sweeps;
        st.tsqr_kernel = tall ? ctx->last_kernel : TTSVD_K_NONE;
        ++built;
        const bool last = built == d - 1;
        // the step's TSMM target (tsmm_reshape's out_rows) and, unless this
        // step finishes the train, the reorder's target shape
        int64_t p_rows, t_rows = 0, t_cols = 0;
        if (right) {
            const int64_t n_hi = dims[hi];
            std::vector<double> core((size_t)(rnew * n_hi * r_right));  // core_from_vt (tt_svd.hpp:121-128)
            for (int64_t b = 0; b < r_right; ++b)
                for (int64_t x = 0; x < n_hi; ++x)
                    for (int64_t a = 0; a < rnew; ++a) core[a + rnew * (x + n_hi * b)] = Vh[a * m + (x + n_hi * b)];
            out->cores[hi] = std::move(core);
            rl[hi] = rnew;
            rr[hi] = r_right;
            p_rows = r_left * dims[lo];
            if (!last) {
                t_rows = cur.rows * rnew / p_rows;
                t_cols = p_rows;
            }
        } else {
            const int64_t n_lo = dims[lo];
            std::vector<double> core((size_t)(r_left * n_lo * rnew));  // core_from_v (tt_svd.hpp:131-138)
            for (int64_t b = 0; b < rnew; ++b)
                for (int64_t x = 0; x < n_lo; ++x)
                    for (int64_t a = 0; a < r_left; ++a) core[a + r_left * (x + n_lo * b)] = Vh[b * m + (a + r_left * x)];
            out->cores[lo] = std::move(core);
            rl[lo] = r_left;
            rr[lo] = rnew;
            p_rows = cur.rows;
            if (last) {
                t_rows = rnew;
                t_cols = cur.rows;
            } else {
                t_cols = dims[hi] * r_right;
                t_rows = rnew * cur.rows / t_cols;
            }
        }
        const int64_t p_cols = cur.rows * rnew / p_rows, ldp = padded_stride_h(p_rows);
        TT_TRY(ensure(ctx->ws_thick[1], (size_t)ldp * p_cols * 8));
        double* P = as<double>(ctx->ws_thick[1]);
        tm.mark(3);
        TT_TRY(tsmm_device(ctx, cur.data, cur.rows, (int)m, cur.ld, d_V, m, (int)rnew, P, p_rows, p_cols, ldp));
        tm.mark(4);
        WorkView next{P, p_rows, p_cols, ldp};
        if (t_rows > 0) {
            const int64_t ldt = padded_stride_h(t_rows);
            TT_TRY(ensure(ctx->ws_work[which], (size_t)ldt * t_cols * 8));
            double* T = as<double>(ctx->ws_work[which]);
            TT_TRY(transpose_reorder_device(ctx, P, p_rows, p_cols, ldp, T, t_rows, t_cols, ldt));
            next = WorkView{T, t_rows, t_cols, ldt};
            which ^= 1;
        }
        tm.mark(7);
        if (tm.on) {
            st.t_tsqr_ms = tm.ms(0, 1);
            st.t_svd_ms = tm.ms(1, 2);
            st.t_tsmm_ms = tm.ms(3, 4);
            st.t_reorder_ms = tm.ms(4, 7);
        }
        out->steps.push_back(st);
        out->sigmas.push_back(sig);
        if (last) {
            // the remaining middle core, in place (tt_svd.hpp:440-449, 478-489)
            const int64_t j = right ? lo : hi;
            const int64_t a = right ? r_left : rnew, b = right ? rnew : r_right;
            TT_TRY(flat_d2h(ctx, next.data, next.rows, next.ld, a * dims[j] * b, flat));
            out->cores[j] = flat;
            rl[j] = a;
            rr[j] = b;
            break;
        }
        cur = next;
        if (right) {
            hi -= 1;
            r_right = rnew;
        } else {
            lo += 1;
            r_left = rnew;
        }
        right = !right;
    }
    out->ranks.assign(d + 1, 1);
    for (int64_t j = 0; j < d; ++j) {
        if (j > 0 && rr[j - 1] != rl[j]) return fail(TTSVD_ERR_DIMENSION_MISMATCH, "two-sided: rank chain broken");
        out->ranks[j + 1] = rr[j];
    }
    return TTSVD_OK;
}

}  // namespace

// =========================================================================
extern "C" {

const char* ttsvd_cu_version(void) { return "ttsvd_cu 0.1 (sm_100a)"; }
const char* ttsvd_cu_last_error(void) { return g_last_error.c_str(); }

int64_t ttsvd_cu_padded_stride(int64_t n) { return padded_stride_h(n); }

int ttsvd_cu_ctx_create(int device, void* stream, ttsvd_cu_ctx** out) {
    if (!out) return fail(TTSVD_ERR_INVALID, "null out");
    *out = nullptr;
    int count = 0;
    TT_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) return fail(TTSVD_ERR_DEVICE, "no such CUDA device");
    TT_CUDA(cudaSetDevice(device));
    auto* c = new ttsvd_cu_ctx();
    c->device = device;
    c->stream = static_cast<cudaStream_t>(stream);
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major < 10) {
        delete c;
        return fail(TTSVD_ERR_DEVICE, "ttsvd_cu requires an sm_100 (Blackwell) device");
    }
    c->num_sms = prop.multiProcessorCount;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_coop_kernel<kJacobiThreads>, kJacobiThreads, 0);
    c->coop_max_blocks = std::max(1, per_sm) * c->num_sms;
    for (auto& e : c->ev) cudaEventCreate(&e);
    *out = c;
    return TTSVD_OK;
}

int ttsvd_cu_ctx_destroy(ttsvd_cu_ctx* ctx) {
    if (!ctx) return TTSVD_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (DevBuf* b : {&ctx->ws_R, &ctx->ws_R2, &ctx->ws_P, &ctx->ws_Scr, &ctx->ws_G, &ctx->ws_Gp, &ctx->ws_A, &ctx->ws_V, &ctx->ws_Vacc, &ctx->ws_U, &ctx->ws_sigma, &ctx->ws_flags, &ctx->ws_work[0],
                      &ctx->ws_work[1], &ctx->ws_X, &ctx->ws_send, &ctx->ws_recv, &ctx->ws_thick[0], &ctx->ws_thick[1], &ctx->ws_gs, &ctx->ws_bd})
        if (b->p) cudaFree(b->p);
    for (DevBuf& b : ctx->ws_slab)
        if (b.p) cudaFree(b.p);
    if (ctx->host_stage.p) cudaFreeHost(ctx->host_stage.p);
    if (ctx->host_cores.p) cudaFreeHost(ctx->host_cores.p);
    if (ctx->host_sig.p) cudaFreeHost(ctx->host_sig.p);
    if (ctx->ws_gt_state.p) cudaFree(ctx->ws_gt_state.p);
    if (ctx->copy_ev) cudaEventDestroy(ctx->copy_ev);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->comm && nccl().ok) nccl().comm_destroy(ctx->comm);
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    delete ctx;
    return TTSVD_OK;
}

int ttsvd_cu_ctx_set_stream(ttsvd_cu_ctx* ctx, void* stream) {
    if (!ctx) return fail(TTSVD_ERR_INVALID, "null context");
    ctx->stream = static_cast<cudaStream_t>(stream);
    return TTSVD_OK;
}

int ttsvd_cu_synchronize(ttsvd_cu_ctx* ctx) {
    TT_TRY(set_device(ctx));
    TT_CUDA(cudaStreamSynchronize(ctx->stream));
    return TTSVD_OK;
}

int64_t ttsvd_cu_ctx_launches(const ttsvd_cu_ctx* ctx) { return ctx ? ctx->launches : -1; }

int ttsvd_cu_ctx_set_timing(ttsvd_cu_ctx* ctx, int on) {
    if (!ctx) return fail(TTSVD_ERR_INVALID, "null context");
    ctx->timing = on != 0;
    return TTSVD_OK;
}

int ttsvd_cu_tsqr(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int64_t m, int64_t ldx, double* R) {
    TT_TRY(set_device(ctx));
    if (m < 1) return fail(TTSVD_ERR_DIMENSION, "tsqr: needs at least one column");
    if (n < m) return fail(TTSVD_ERR_DIMENSION, "tsqr: requires n >= m");
    if (m > 4096) return fail(TTSVD_ERR_DIMENSION, "tsqr: m > 4096 not supported");
    if (!X || !R || ldx < n) return fail(TTSVD_ERR_INVALID, "tsqr: bad pointer or leading dimension");
    return tsqr_device(ctx, X, n, (int)m, ldx, R);
}

int ttsvd_cu_reduce_block(ttsvd_cu_ctx* ctx, const double* M, int64_t rows, int64_t m, int64_t ldm,
                          const double* R_in, int64_t r_m, double* R_out) {
    TT_TRY(set_device(ctx));
    if (r_m != m) return fail(TTSVD_ERR_DIMENSION_MISMATCH, "reduce_block: R.m != M.cols");
    if (m < 1 || rows < 0 || !R_in || !R_out || (rows > 0 && (!M || ldm < rows)))
        return fail(TTSVD_ERR_INVALID, "reduce_block: bad arguments");
    // one job: the running R starts at R_in and the rows of M are folded in
    // (tsqr.hpp:208-224 is a single reduce_into as well)
    if (rows == 0) {
        TT_CUDA(cudaMemcpyAsync(R_out, R_in, (size_t)m * m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
        return TTSVD_OK;
    }
    return tsqr_device(ctx, M, rows, (int)m, ldm, R_out, R_in);
}

int ttsvd_cu_combine_factors(ttsvd_cu_ctx* ctx, const double* parts, int64_t P, int64_t m, double* R) {
    TT_TRY(set_device(ctx));
    if (P < 1) return fail(TTSVD_ERR_DIMENSION_MISMATCH, "combine_factors: empty list");
    if (m < 1 || !parts || !R) return fail(TTSVD_ERR_INVALID, "combine_factors: bad arguments");
    TT_TRY(ensure(ctx->ws_recv, (size_t)P * m * m * 8));
    double* buf = as<double>(ctx->ws_recv);
    TT_CUDA(cudaMemcpyAsync(buf, parts, (size_t)P * m * m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    return merge_tree(ctx, buf, P, (int)m, R);
}

int ttsvd_cu_small_svd(ttsvd_cu_ctx* ctx, const double* R, int64_t m, double* sigma, double* V) {
    TT_TRY(set_device(ctx));
    if (m > 4096) return fail(TTSVD_ERR_DIMENSION_MISMATCH, "small_svd: m exceeds 4096");
    if (m < 1 || !R || !sigma || !V) return fail(TTSVD_ERR_INVALID, "small_svd: bad arguments");
    int sweeps = 0;
    TT_TRY(svd_work(ctx, R, m, m, m, false, true, sigma, V, &sweeps));
    TT_CUDA(cudaStreamSynchronize(ctx->stream));
    return TTSVD_OK;
}

int ttsvd_cu_jacobi_svd(ttsvd_cu_ctx* ctx, const double* A, int64_t n, int64_t m, int64_t lda, double* sigma,
                        double* V, double* U) {
    TT_TRY(set_device(ctx));
    if (n < m) return fail(TTSVD_ERR_DIMENSION, "jacobi_svd: requires n >= m");
    if (m < 1 || !A || !sigma || !V || lda < n) return fail(TTSVD_ERR_INVALID, "jacobi_svd: bad arguments");
    TT_TRY(ensure(ctx->ws_A, (size_t)n * m * 8));
    TT_TRY(ensure(ctx->ws_X, (size_t)m * m * 8));
    double* W = as<double>(ctx->ws_A);
    double* Vacc = as<double>(ctx->ws_X);
    TT_CUDA(cudaMemcpy2DAsync(W, n * 8, A, lda * 8, n * 8, m, cudaMemcpyDeviceToDevice, ctx->stream));
    TT_TRY(jacobi_device(ctx, W, (int)n, (int)m, Vacc));
    int sweeps = 0;
    TT_TRY(jacobi_status(ctx, &sweeps));
    double* Uout = U;
    if (!Uout) {
        TT_TRY(ensure(ctx->ws_V, (size_t)n * m * 8));
        Uout = as<double>(ctx->ws_V);
    }
    TT_TRY(finalize_device(ctx, W, (int)n, (int)m, Vacc, sigma, Uout, V));
    TT_CUDA(cudaStreamSynchronize(ctx->stream));
    return TTSVD_OK;
}

int ttsvd_cu_driver_svd(ttsvd_cu_ctx* ctx, const double* A, int64_t n, int64_t m, int64_t lda, int64_t r,
                        double* sigma, double* V, int32_t* path_out) {
    TT_TRY(set_device(ctx));
    if (!A || !sigma || !V || m < 1 || n < m || lda < n || r < 0 || r > m)
        return fail(TTSVD_ERR_INVALID, "driver_svd: needs n >= m >= 1, lda >= n, 0 <= r <= m");
    int sweeps = 0;
    TT_TRY(ensure(ctx->ws_V, (size_t)n * m * 8));
    double* Vw = as<double>(ctx->ws_V);
    TT_TRY(svd_work(ctx, A, n, m, lda, false, false, sigma, Vw, &sweeps));
    if (path_out) *path_out = ctx->bd_pending ? 1 : 0;
    TT_TRY(svd_vectors(ctx, r, sigma, Vw));
    if (r > 0) TT_CUDA(cudaMemcpyAsync(V, Vw, (size_t)n * r * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    TT_CUDA(cudaStreamSynchronize(ctx->stream));
    return TTSVD_OK;
}

int ttsvd_cu_select_rank(ttsvd_cu_ctx* ctx, const double* sigma, int64_t m, double delta, int64_t r_max,
                         int64_t* rank_host) {
    TT_TRY(set_device(ctx));
    if (!sigma || !rank_host || m < 0) return fail(TTSVD_ERR_INVALID, "select_rank: bad arguments");
    std::vector<double> s((size_t)std::max<int64_t>(m, 1));
    if (m > 0) TT_TRY(d2h(ctx, s.data(), sigma, (size_t)m));
    *rank_host = select_rank_h(s.data(), m, delta, r_max);
    return TTSVD_OK;
}

int64_t ttsvd_cu_select_rank_host(const double* sigma, int64_t m, double delta, int64_t r_max) {
    if (!sigma || m < 0) return -1;
    return select_rank_h(sigma, m, delta, r_max);
}

int ttsvd_cu_derive_delta(double norm_source, double eps, int64_t d, double* delta_host) {
    if (d < 2) return fail(TTSVD_ERR_DEGENERATE, "derive_delta: requires d >= 2");
    if (!delta_host) return fail(TTSVD_ERR_INVALID, "derive_delta: null out");
    *delta_host = eps / std::sqrt((double)(d - 1)) * norm_source;
    return TTSVD_OK;
}

int ttsvd_cu_tsmm_reshape(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int64_t m, int64_t ldx, const double* V,
                          int64_t k, int64_t ldv, double* Y, int64_t out_rows, int64_t out_cols, int64_t ldy) {
    TT_TRY(set_device(ctx));
    if (k > m) return fail(TTSVD_ERR_SHAPE, "tsmm_reshape: k > m (kernel only shrinks)");
    if (out_rows < 1 || out_cols < 1 || n * k != out_rows * out_cols)
        return fail(TTSVD_ERR_SHAPE, "tsmm_reshape: out shape does not hold n*k elements");
    if (!X || !V || !Y || ldx < n || ldv < m || ldy < out_rows || k < 1)
        return fail(TTSVD_ERR_INVALID, "tsmm_reshape: bad pointer or leading dimension");
    if ((size_t)m * 8 > (size_t)kTsmmSmem) return fail(TTSVD_ERR_SHAPE, "tsmm_reshape: m too large");
    return tsmm_device(ctx, X, n, (int)m, ldx, V, ldv, (int)k, Y, out_rows, out_cols, ldy);
}

} // extern "C"

namespace {
int tt_svd_impl(ttsvd_cu_ctx* ctx, const double* X, const int64_t* dims, int64_t d, int64_t ldx, int64_t r_max,
                double eps, ttsvd_cu_tt** out, const double* R_first);
}

extern "C" {

int ttsvd_cu_tt_svd(ttsvd_cu_ctx* ctx, const double* X, const int64_t* dims, int64_t d, int64_t ldx, int64_t r_max,
                    double eps, ttsvd_cu_tt** out) {
    return tt_svd_impl(ctx, X, dims, d, ldx, r_max, eps, out, nullptr);
}

} // extern "C"

namespace {
int tt_svd_impl(ttsvd_cu_ctx* ctx, const double* X, const int64_t* dims, int64_t d, int64_t ldx, int64_t r_max,
                double eps, ttsvd_cu_tt** out, const double* R_first) {
    TT_TRY(set_device(ctx));
    if (!out || !dims || !X) return fail(TTSVD_ERR_INVALID, "tt_svd: null argument");
    *out = nullptr;
    if (d < 2) return fail(TTSVD_ERR_DEGENERATE, "tt_svd_tsqr: requires d >= 2");
    int64_t total = 1;
    for (int64_t i = 0; i < d; ++i) {
        if (dims[i] < 1) return fail(TTSVD_ERR_DIMENSION, "Shape: extents must be >= 1");
        total *= dims[i];
    }
    const int64_t rows = total / dims[d - 1];
    if (ldx < rows) return fail(TTSVD_ERR_LAYOUT, "tt_svd: leading stride below the row count");
    auto* tt = new ttsvd_cu_tt();
    std::vector<int64_t> dv(dims, dims + d);
    int rc = run_chain(ctx, WorkView{X, rows, dims[d - 1], ldx}, dv, r_max, eps, d, tt, nullptr, nullptr,
                       ColSplit{0, 0}, R_first);
    if (rc != TTSVD_OK) {
        delete tt;
        return rc;
    }
    *out = tt;
    return TTSVD_OK;
}
} // namespace

extern "C" {

int ttsvd_cu_run_chain(ttsvd_cu_ctx* ctx, const double* W, int64_t rows, int64_t cols, int64_t ldw, const int64_t* dims,
                       int64_t d, int64_t r_max, double eps, int64_t d_for_delta, double* delta_io,
                       double* first_sigma_norm_out, ttsvd_cu_tt** out) {
    TT_TRY(set_device(ctx));
    if (!out || !dims || !W || !delta_io) return fail(TTSVD_ERR_INVALID, "run_chain: null argument");
    *out = nullptr;
    if (d < 2) return fail(TTSVD_ERR_DEGENERATE, "run_chain: requires d >= 2");
    int64_t total = 1;
    for (int64_t i = 0; i < d; ++i) {
        if (dims[i] < 1) return fail(TTSVD_ERR_DIMENSION, "Shape: extents must be >= 1");
        total *= dims[i];
    }
    if (cols != dims[d - 1] || rows * cols != total) return fail(TTSVD_ERR_SHAPE, "run_chain: W is not the last-mode matricization");
    if (ldw < rows) return fail(TTSVD_ERR_LAYOUT, "run_chain: leading stride below the row count");
    auto* tt = new ttsvd_cu_tt();
    double fsn = 0.0;
    int rc = run_chain(ctx, WorkView{W, rows, cols, ldw}, std::vector<int64_t>(dims, dims + d), r_max, eps, d_for_delta,
                       tt, delta_io, &fsn);
    if (rc != TTSVD_OK) {
        delete tt;
        return rc;
    }
    if (first_sigma_norm_out) *first_sigma_norm_out = fsn;
    *out = tt;
    return TTSVD_OK;
}

int ttsvd_cu_tt_svd_two_sided(ttsvd_cu_ctx* ctx, const double* X, const int64_t* dims, int64_t d, int64_t ldx,
                              int64_t r_max, double eps, ttsvd_cu_tt** out) {
    TT_TRY(set_device(ctx));
    if (!out || !dims || !X) return fail(TTSVD_ERR_INVALID, "tt_svd_two_sided: null argument");
    *out = nullptr;
    if (d < 2) return fail(TTSVD_ERR_DEGENERATE, "tt_svd_two_sided: requires d >= 2");
    int64_t total = 1;
    for (int64_t i = 0; i < d; ++i) {
        if (dims[i] < 1) return fail(TTSVD_ERR_DIMENSION, "Shape: extents must be >= 1");
        total *= dims[i];
    }
    const int64_t rows = total / dims[d - 1];
    if (ldx < rows) return fail(TTSVD_ERR_LAYOUT, "tt_svd_two_sided: leading stride below the row count");
    auto* tt = new ttsvd_cu_tt();
    int rc = run_two_sided(ctx, WorkView{X, rows, dims[d - 1], ldx}, std::vector<int64_t>(dims, dims + d), r_max, eps, tt);
    if (rc != TTSVD_OK) {
        delete tt;
        return rc;
    }
    *out = tt;
    return TTSVD_OK;
}

int ttsvd_cu_transpose_reorder(ttsvd_cu_ctx* ctx, const double* W, int64_t n, int64_t m, int64_t ldw, double* Y,
                               int64_t out_rows, int64_t out_cols, int64_t ldy) {
    TT_TRY(set_device(ctx));
    if (out_rows < 1 || out_cols < 1 || out_rows * out_cols != n * m)
        return fail(TTSVD_ERR_SHAPE, "transpose_reorder: out shape does not hold n*m elements");
    if (!W || !Y || n < 1 || m < 1 || ldw < n || ldy < out_rows)
        return fail(TTSVD_ERR_INVALID, "transpose_reorder: bad pointer or leading dimension");
    return transpose_reorder_device(ctx, W, n, m, ldw, Y, out_rows, out_cols, ldy);
}

int ttsvd_cu_choose_combined_dims(const int64_t* dims, int64_t d, int64_t m_min, double f1_min, const int64_t* r_tilde,
                                  int64_t n_r_tilde, int64_t r_max, int64_t* k_out, int64_t* m_out) {
    if (!dims || !k_out || !m_out) return fail(TTSVD_ERR_INVALID, "choose_combined_dims: null argument");
    if (d < 2) return fail(TTSVD_ERR_DEGENERATE, "choose_combined_dims: requires d >= 2");
    if (m_min < 1 || !(f1_min > 0.0) || f1_min > 1.0)
        return fail(TTSVD_ERR_DIMENSION_MISMATCH, "choose_combined_dims: invalid parameters");
    int64_t total = 1;
    for (int64_t i = 0; i < d; ++i) total *= dims[i];
    // ThickBoundsParams::estimate_at (tt_svd.hpp:298-309)
    auto estimate_at = [&](int64_t pos) {
        int64_t lead = 1;
        for (int64_t i = 0; i < pos; ++i) lead *= dims[i];
        const int64_t cap = std::min(lead, total / lead);
        int64_t rt = r_max;
        if (r_tilde && n_r_tilde > 0) rt = r_tilde[std::min(pos - 1, n_r_tilde - 1)];
        return std::min(rt, cap);
    };
    int64_t trail = 1;
    for (int64_t k = 1; k < d; ++k) {
        trail *= dims[d - k];
        const double need = std::max((double)m_min, (double)estimate_at(d - k) / f1_min);
        if ((double)trail >= need) {
            *k_out = k;
            *m_out = trail;
            return TTSVD_OK;
        }
    }
    *k_out = d - 1;
    *m_out = total / dims[0];
    return TTSVD_OK;
}

} // extern "C"

namespace {
// X: device tensor (padded layout).  X_host != nullptr: X is still empty and
// the tensor is at X_host (same layout): when the merged first step runs on
// the tall-tile kernel, X arrives in row chunks of the merged matricization
// on a second stream and tsqr_t128 folds every chunk as soon as it has landed
// (the first TSQR under the H2D); otherwise it is copied whole first.
int thick_impl(ttsvd_cu_ctx* ctx, const double* X, const double* X_host, const int64_t* dims, int64_t d, int64_t ldx,
               int64_t r_max, double eps, int64_t m_min, double f1_min, const int64_t* r_tilde, int64_t n_r_tilde,
               ttsvd_cu_tt** out) {
    TT_TRY(set_device(ctx));
    if (!out || !dims || !X) return fail(TTSVD_ERR_INVALID, "tt_svd_thick: null argument");
    *out = nullptr;
    if (d < 2) return fail(TTSVD_ERR_DEGENERATE, "tt_svd_thick_bounds: requires d >= 2");
    int64_t total = 1;
    for (int64_t i = 0; i < d; ++i) {
        if (dims[i] < 1) return fail(TTSVD_ERR_DIMENSION, "Shape: extents must be >= 1");
        total *= dims[i];
    }
    const int64_t rows0 = total / dims[d - 1];
    if (ldx < rows0) return fail(TTSVD_ERR_LAYOUT, "tt_svd_thick: leading stride below the row count");
    int64_t k = 1, m = dims[d - 1];
    TT_TRY(ttsvd_cu_choose_combined_dims(dims, d, m_min, f1_min, r_tilde, n_r_tilde, r_max, &k, &m));
    if (k == 1) {
        if (X_host) return ttsvd_cu_tt_svd_host(ctx, X_host, dims, d, ldx, r_max, eps, out);
        return ttsvd_cu_tt_svd(ctx, X, dims, d, ldx, r_max, eps, out);
    }

    // merged tensor (n_1, ..., n_{d-k}, m): column x of its matricization is the
    // contiguous run of X's column x / q starting at row (x mod q) (N/m),
    // q = m / n_d — a split-column view of X that K_TSQR and K_TSMM read in
    // place (ColSplit).  Only when the first step's kernels cannot (short or
    // narrow shapes) is it copied into its own padded layout (copy_logical,
    // storage.hpp:158-172; tt_svd.hpp:347-348).
    const int64_t rows_m = total / m, q = m / dims[d - 1];
    std::vector<int64_t> mdims(dims, dims + d - k);
    mdims.push_back(m);
    const int64_t dm = (int64_t)mdims.size();
    ttsvd_cu_tt main_tt;
    double delta = -1.0, fsn = 0.0;
    const double* R_first = nullptr;
    if (X_host) {
        double* dX = const_cast<double*>(X);
        const int64_t unit = (int64_t)ctx->num_sms * 256;  // a 256-row tile per CTA
        if (t128_eligible(ctx, rows_m, (int)m) && rows_m >= 8 * unit && !ctx->timing) {
            if (!ctx->copy_stream) {
                TT_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
                TT_CUDA(cudaEventCreateWithFlags(&ctx->copy_ev, cudaEventDisableTiming));
            }
            TT_TRY(ensure(ctx->ws_X, (size_t)m * m * 8));
            double* R = as<double>(ctx->ws_X);
            TT_CUDA(cudaEventRecord(ctx->copy_ev, ctx->stream));
            TT_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_ev, 0));
            const int64_t n_d = dims[d - 1];
            auto before = [&](int64_t r_lo, int64_t r_hi) -> int {
                // rows [r_lo, r_hi) of the merged matricization: q runs in each of X's n_d columns
                for (int64_t id = 0; id < n_d; ++id)
                    TT_CUDA(cudaMemcpy2DAsync(dX + id * ldx + r_lo, (size_t)rows_m * 8, X_host + id * ldx + r_lo,
                                              (size_t)rows_m * 8, (size_t)(r_hi - r_lo) * 8, (size_t)q,
                                              cudaMemcpyHostToDevice, ctx->copy_stream));
                TT_CUDA(cudaEventRecord(ctx->copy_ev, ctx->copy_stream));
                TT_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->copy_ev, 0));
                return TTSVD_OK;
            };
            const int64_t chunk = std::max<int64_t>(1, rows_m / (8 * unit)) * unit;
            const int rc_q = tsqr_t128_run(ctx, dX, rows_m, (int)m, ldx, R, ColSplit{(int)q, rows_m}, chunk, before);
            if (rc_q != TTSVD_OK) return rc_q;
            R_first = R;
        } else {
            TT_CUDA(cudaMemcpyAsync(dX, X_host, (size_t)ldx * dims[d - 1] * 8, cudaMemcpyHostToDevice, ctx->stream));
        }
    }
    int rc_main = run_chain(ctx, WorkView{X, rows_m, m, ldx}, mdims, r_max, eps, dm, &main_tt, &delta, &fsn,
                            ColSplit{(int)q, rows_m}, R_first);
    if (rc_main == kNoView) {
        const int64_t ldm = padded_stride_h(rows_m);
        TT_TRY(ensure(ctx->ws_thick[0], (size_t)ldm * m * 8));
        double* W = as<double>(ctx->ws_thick[0]);
        for (int64_t id = 0; id < dims[d - 1]; ++id)
            TT_CUDA(cudaMemcpy2DAsync(W + id * q * ldm, (size_t)ldm * 8, X + id * ldx, (size_t)rows_m * 8,
                                      (size_t)rows_m * 8, (size_t)q, cudaMemcpyDeviceToDevice, ctx->stream));
        delta = -1.0;
        rc_main = run_chain(ctx, WorkView{W, rows_m, m, ldm}, mdims, r_max, eps, dm, &main_tt, &delta, &fsn);
    }
    if (rc_main != TTSVD_OK) return rc_main;

    // recovery: TT-SVD of the combined core T_bar (r_b x m) as the (k+1)-mode
    // tensor (r_b, n_{d-k+1}, ..., n_d) (tt_svd.hpp:350-371)
    const std::vector<double>& tbar = main_tt.cores[dm - 1];
    const int64_t rb = main_tt.ranks[dm - 1];
    std::vector<int64_t> rdims{rb};
    for (int64_t i = d - k; i < d; ++i) rdims.push_back(dims[i]);
    const int64_t rrows = rb * m / dims[d - 1], ldr = padded_stride_h(rrows);
    std::vector<double> hr((size_t)ldr * dims[d - 1], 0.0);
    double tnorm = 0.0;
    for (int64_t l = 0; l < rb * m; ++l) {
        hr[(size_t)((l / rrows) * ldr + l % rrows)] = tbar[(size_t)l];
        tnorm += tbar[(size_t)l] * tbar[(size_t)l];
    }
    TT_TRY(ensure(ctx->ws_thick[1], hr.size() * 8));
    double* Rw = as<double>(ctx->ws_thick[1]);
    TT_CUDA(cudaMemcpyAsync(Rw, hr.data(), hr.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    double rdelta = delta * std::sqrt(tnorm) / (fsn > 0.0 ? fsn : 1.0);
    ttsvd_cu_tt rec_tt;
    TT_TRY(run_chain(ctx, WorkView{Rw, rrows, dims[d - 1], ldr}, rdims, r_max, eps, (int64_t)rdims.size(), &rec_tt,
                     &rdelta, nullptr));

    // absorb the dummy-mode core theta (1 x r_b x rho) into its neighbour
    // (tt_svd.hpp:373-398)
    std::vector<double> theta = rec_tt.cores[0];
    const int64_t rho = rec_tt.ranks[1];
    const std::vector<double>& c1 = rec_tt.cores[1];
    const int64_t n1 = rdims[1], r2 = rec_tt.ranks[2];
    auto* tt = new ttsvd_cu_tt();
    tt->dims.assign(dims, dims + d);
    tt->cores.assign(main_tt.cores.begin(), main_tt.cores.end() - 1);
    if (rb == 1 && rho == 1) {
        const double sc = theta[0];
        for (auto& v : tt->cores[0]) v *= sc;
        theta[0] = 1.0;
    }
    std::vector<double> boundary((size_t)(rb * n1 * r2), 0.0);
    for (int64_t b = 0; b < r2; ++b)
        for (int64_t x = 0; x < n1; ++x)
            for (int64_t a = 0; a < rb; ++a) {
                double acc = 0.0;
                for (int64_t l = 0; l < rho; ++l) acc += theta[(size_t)(a + rb * l)] * c1[(size_t)(l + rho * (x + n1 * b))];
                boundary[(size_t)(a + rb * (x + n1 * b))] = acc;
            }
    tt->cores.push_back(std::move(boundary));
    for (size_t j = 2; j < rec_tt.cores.size(); ++j) tt->cores.push_back(rec_tt.cores[j]);
    tt->ranks.assign(main_tt.ranks.begin(), main_tt.ranks.begin() + dm);  // r_0 .. r_{dm-1} = r_b
    for (size_t j = 2; j < rec_tt.ranks.size(); ++j) tt->ranks.push_back(rec_tt.ranks[j]);
    tt->steps = main_tt.steps;
    tt->steps.insert(tt->steps.end(), rec_tt.steps.begin(), rec_tt.steps.end());
    tt->sigmas = main_tt.sigmas;
    tt->sigmas.insert(tt->sigmas.end(), rec_tt.sigmas.begin(), rec_tt.sigmas.end());
    *out = tt;
    return TTSVD_OK;
}
} // namespace

extern "C" {

int ttsvd_cu_tt_svd_thick(ttsvd_cu_ctx* ctx, const double* X, const int64_t* dims, int64_t d, int64_t ldx,
                          int64_t r_max, double eps, int64_t m_min, double f1_min, const int64_t* r_tilde,
                          int64_t n_r_tilde, ttsvd_cu_tt** out) {
    return thick_impl(ctx, X, nullptr, dims, d, ldx, r_max, eps, m_min, f1_min, r_tilde, n_r_tilde, out);
}

int ttsvd_cu_tt_svd_thick_host(ttsvd_cu_ctx* ctx, const double* X_host, const int64_t* dims, int64_t d, int64_t ldx,
                               int64_t r_max, double eps, int64_t m_min, double f1_min, const int64_t* r_tilde,
                               int64_t n_r_tilde, ttsvd_cu_tt** out) {
    TT_TRY(set_device(ctx));
    if (!X_host || !dims || d < 1) return fail(TTSVD_ERR_INVALID, "tt_svd_thick_host: null argument");
    for (int64_t i = 0; i < d; ++i)
        if (dims[i] < 1) return fail(TTSVD_ERR_DIMENSION, "Shape: extents must be >= 1");
    TT_TRY(ensure(ctx->ws_recv, (size_t)ldx * dims[d - 1] * 8));
    return thick_impl(ctx, as<double>(ctx->ws_recv), X_host, dims, d, ldx, r_max, eps, m_min, f1_min, r_tilde,
                      n_r_tilde, out);
}

int ttsvd_cu_tt_svd_host(ttsvd_cu_ctx* ctx, const double* X_host, const int64_t* dims, int64_t d, int64_t ldx,
                         int64_t r_max, double eps, ttsvd_cu_tt** out) {
    TT_TRY(set_device(ctx));
    if (!X_host || !dims || d < 1) return fail(TTSVD_ERR_INVALID, "tt_svd_host: null argument");
    int64_t total = 1;
    for (int64_t i = 0; i < d; ++i) total *= dims[i];
    const size_t bytes = (size_t)ldx * dims[d - 1] * 8;
    (void)total;
    TT_TRY(ensure(ctx->ws_recv, bytes));
    double* dX = as<double>(ctx->ws_recv);
    const int64_t rows = d >= 2 && dims[d - 1] > 0 ? total / dims[d - 1] : 0;
    const int m1 = (int)dims[d - 1];
    // First step on the TMA-staged stream kernel and tall enough: X arrives
    // in row chunks on a second stream and every chunk is folded as soon as it
    // has landed (the streams' running factors carried between the launches),
    // so the first TSQR hides under the H2D.  Same bits as the device entry.
    if (d >= 2 && ldx >= rows && gt_eligible(ctx, dX, rows, m1, ldx) &&
        rows >= (int64_t)ctx->num_sms * kGtMaxWarps * 64 * 8 && !ctx->timing) {
        if (!ctx->copy_stream) {
            TT_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
            TT_CUDA(cudaEventCreateWithFlags(&ctx->copy_ev, cudaEventDisableTiming));
        }
        TT_TRY(ensure(ctx->ws_X, (size_t)m1 * m1 * 8));
        double* R = as<double>(ctx->ws_X);
        // the copies must not overtake earlier work on the context's stream that still reads the buffer
        TT_CUDA(cudaEventRecord(ctx->copy_ev, ctx->stream));
        TT_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_ev, 0));
        auto before = [&](int64_t r_lo, int64_t r_hi) -> int {
            TT_CUDA(cudaMemcpy2DAsync(dX + r_lo, (size_t)ldx * 8, X_host + r_lo, (size_t)ldx * 8, (size_t)(r_hi - r_lo) * 8,
                                      (size_t)m1, cudaMemcpyHostToDevice, ctx->copy_stream));
            TT_CUDA(cudaEventRecord(ctx->copy_ev, ctx->copy_stream));
            TT_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->copy_ev, 0));
            return TTSVD_OK;
        };
        int rc_q;
        if (m1 <= 16) rc_q = tsqr_gt_chunked<16, 4, 8>(ctx, dX, rows, m1, ldx, R, 8, before);
        else rc_q = tsqr_gt_chunked<32, 8, 8>(ctx, dX, rows, m1, ldx, R, 8, before);
        if (rc_q != TTSVD_OK) return rc_q;
        return tt_svd_impl(ctx, dX, dims, d, ldx, r_max, eps, out, R);
    }
    TT_CUDA(cudaMemcpyAsync(dX, X_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
    return ttsvd_cu_tt_svd(ctx, dX, dims, d, ldx, r_max, eps, out);
}

int ttsvd_cu_tt_svd_distributed(ttsvd_cu_ctx* ctx, const double* const* slabs, int64_t n_slabs, int64_t part0,
                                int64_t P_total, const int64_t* ldims, int64_t d_local, int64_t ld_slab,
                                int64_t r_max, double eps, ttsvd_cu_exchange_fn exchange, void* user,
                                ttsvd_cu_tt** out) {
    TT_TRY(set_device(ctx));
    if (!out || !slabs || !ldims || n_slabs < 1 || d_local < 1) return fail(TTSVD_ERR_PARTITION, "tt_svd_distributed: no partitions");
    *out = nullptr;
    if (P_total < n_slabs || part0 < 0 || part0 + n_slabs > P_total || P_total % n_slabs != 0)
        return fail(TTSVD_ERR_PARTITION, "tt_svd_distributed: inconsistent partition counts");
    // the exchange: a caller's callback, else the context's NCCL communicator
    // (ranks own consecutive partitions: rank k holds k*n_slabs ..), else
    // none (every partition in this process, the reference's in-process form)
    const bool use_nccl = !exchange && ctx->comm;
    if (use_nccl && (P_total != n_slabs * ctx->comm_size || part0 != (int64_t)ctx->comm_rank * n_slabs))
        return fail(TTSVD_ERR_PARTITION, "tt_svd_distributed: partitions do not match the communicator's ranks");
    if (n_slabs != P_total && !exchange && !use_nccl)
        return fail(TTSVD_ERR_INVALID, "tt_svd_distributed: an exchange (callback or NCCL communicator) is required across processes");
    const bool exchanged = exchange || use_nccl;
    auto all_gather = [&](const double* send, double* recv, int64_t count) -> int {
        if (use_nccl) {
            TT_NCCL(nccl().all_gather(send, recv, (size_t)count, ncclDouble, ctx->comm, ctx->stream));
            return TTSVD_OK;
        }
        if (exchange(user, send, recv, count, (void*)ctx->stream) != 0)
            return fail(TTSVD_ERR_DEVICE, "tt_svd_distributed: exchange failed");
        return TTSVD_OK;
    };
    const int64_t d = d_local + 1;
    int64_t total = 1;
    for (int64_t i = 0; i < d_local; ++i) total *= ldims[i];
    auto* tt = new ttsvd_cu_tt();
    std::vector<int64_t> gdims(d);
    gdims[0] = P_total;
    for (int64_t i = 0; i < d_local; ++i) gdims[i + 1] = ldims[i];
    auto done = [&](int rc) -> int {
        if (rc != TTSVD_OK) {
            delete tt;
            return rc;
        }
        *out = tt;
        return (int)TTSVD_OK;
    };
    if (P_total == 1) {  // one partition: tt_svd_tsqr of (1, n_1, ...) (tt_svd.hpp:530-541)
        gdims[0] = 1;
        const int64_t rows = d_local == 1 ? 1 : total / ldims[d_local - 1];
        return done(run_chain(ctx, WorkView{slabs[0], rows, ldims[d_local - 1], ld_slab}, gdims, r_max, eps, d, tt));
    }
    // per-slab state: grow-only ping-pong workspaces of the context (nothing
    // is allocated or freed per call once they have grown)
    std::vector<WorkView> cur(n_slabs);
    if (ctx->ws_slab.size() < (size_t)(2 * n_slabs)) ctx->ws_slab.resize((size_t)(2 * n_slabs));
    std::vector<DevBuf>& bufs = ctx->ws_slab;
    for (int64_t p = 0; p < n_slabs; ++p) {
        if (d_local == 1) cur[p] = WorkView{slabs[p], 1, ldims[0], ld_slab};
        else cur[p] = WorkView{slabs[p], total / ldims[d_local - 1], ldims[d_local - 1], ld_slab};
    }
    tt->dims = gdims;
    tt->cores.assign(d, {});
    tt->ranks.assign(d + 1, 1);
    double delta = -1.0;
    int64_t r = 1;
    int flip = 0;
    std::vector<double> sig;
    // the steps' V blocks go to the pinned core arena asynchronously and the
    // cores are built after the sweep (as run_chain: one host round trip per
    // step, for the sigmas the rank rule needs)
    struct Pending {
        int64_t i, m, rnew, n_i, r;
        size_t off;
    };
    std::vector<Pending> pending;
    size_t core_off = 0;
    auto flush = [&]() {
        const double* base = as<double>(ctx->host_cores);
        for (const Pending& pc : pending) {
            std::vector<double> core((size_t)(pc.rnew * pc.n_i * pc.r));
            for (int64_t b = 0; b < pc.r; ++b)
                for (int64_t x = 0; x < pc.n_i; ++x)
                    for (int64_t a = 0; a < pc.rnew; ++a)
                        core[a + pc.rnew * (x + pc.n_i * b)] = base[pc.off + a * pc.m + (x + pc.n_i * b)];
            tt->cores[pc.i + 1] = std::move(core);
        }
        pending.clear();
        core_off = 0;
    };
    int rc = TTSVD_OK;
    for (int64_t i = d_local - 1; i >= 0 && rc == TTSVD_OK; --i) {
        const int64_t n_i = ldims[i];
        const int64_t m = n_i * r;
        const size_t mm = (size_t)m * m;
        if ((rc = ensure(ctx->ws_send, n_slabs * mm * 8)) != TTSVD_OK) break;
        if ((rc = ensure(ctx->ws_recv, P_total * mm * 8)) != TTSVD_OK) break;
        double* send = as<double>(ctx->ws_send);
        double* recv = exchanged ? as<double>(ctx->ws_recv) : send;
        // gram_triangular per local partition (tt_svd.hpp:204-210, 573)
        for (int64_t p = 0; p < n_slabs && rc == TTSVD_OK; ++p)
            rc = tsqr_device(ctx, cur[p].data, cur[p].rows, (int)m, cur[p].ld, send + p * mm);
        if (rc != TTSVD_OK) break;
        if (exchanged && (rc = all_gather(send, recv, (int64_t)(n_slabs * mm))) != TTSVD_OK) break;
        // pinned-order combine over all partitions (tt_svd.hpp:575)
        if ((rc = ensure(ctx->ws_X, mm * 8)) != TTSVD_OK) break;
        double* R = as<double>(ctx->ws_X);
        if ((rc = ensure(ctx->ws_R2, ((P_total + 1) / 2) * mm * 8)) != TTSVD_OK) break;
        if ((rc = merge_tree(ctx, recv, P_total, (int)m, R)) != TTSVD_OK) break;
        // duplicated small SVD (tt_svd.hpp:579-606): identical on every process
        if ((rc = ensure(ctx->ws_sigma, (size_t)m * 8)) != TTSVD_OK) break;
        if ((rc = ensure(ctx->ws_V, mm * 8)) != TTSVD_OK) break;
        double* d_sigma = as<double>(ctx->ws_sigma);
        double* d_V = as<double>(ctx->ws_V);
        int sweeps = 0;
        if ((rc = svd_work(ctx, R, m, m, m, true, false, d_sigma, d_V, &sweeps)) != TTSVD_OK) break;
        sig.resize(m);
        if ((rc = d2h(ctx, sig.data(), d_sigma, m)) != TTSVD_OK) break;
        const int64_t global_rows = cur[0].rows * P_total;
        const int64_t nsig = std::min(m, global_rows);
        if (delta < 0.0) delta = eps / std::sqrt((double)(d - 1)) * sigma_norm_h(sig.data(), m);
        const int64_t rnew = choose_rank_h(sig.data(), m, m, nsig, delta, r_max, global_rows);
        if ((rc = svd_vectors(ctx, rnew, d_sigma, d_V)) != TTSVD_OK) break;
        {
            const size_t need = (size_t)m * rnew;
            if (core_off + need > ctx->host_cores.bytes / 8) {
                cudaError_t e = cudaStreamSynchronize(ctx->stream);
                if (e != cudaSuccess) { rc = fail(TTSVD_ERR_DEVICE, cudaGetErrorString(e)); break; }
                flush();
                if ((rc = ensure_host(ctx->host_cores, std::max<size_t>(need, (size_t)1 << 20) * 8 * 2)) != TTSVD_OK) break;
            }
            cudaError_t e = cudaMemcpyAsync(as<double>(ctx->host_cores) + core_off, d_V, need * 8,
                                            cudaMemcpyDeviceToHost, ctx->stream);
            if (e != cudaSuccess) { rc = fail(TTSVD_ERR_DEVICE, cudaGetErrorString(e)); break; }
            pending.push_back(Pending{i, m, rnew, n_i, r, core_off});
            core_off += need;
        }
        tt->ranks[i + 1] = rnew;
        ttsvd_cu_step st{};
        st.rows = global_rows;
        st.cols = m;
        st.nsig = nsig;
        st.rank = rnew;
        tt->steps.push_back(st);
        tt->sigmas.emplace_back(sig.begin(), sig.begin() + nsig);
        for (int64_t p = 0; p < n_slabs && rc == TTSVD_OK; ++p) {
            const int64_t out_rows = i >= 1 ? cur[p].rows / ldims[i - 1] : 1;
            const int64_t out_cols = i >= 1 ? ldims[i - 1] * rnew : rnew;
            const int64_t ldy = padded_stride_h(out_rows);
            DevBuf& b = bufs[2 * p + flip];
            if ((rc = ensure(b, (size_t)ldy * out_cols * 8)) != TTSVD_OK) break;
            rc = tsmm_device(ctx, cur[p].data, cur[p].rows, (int)m, cur[p].ld, d_V, m, (int)rnew, as<double>(b),
                             out_rows, out_cols, ldy);
            cur[p] = WorkView{as<double>(b), out_rows, out_cols, ldy};
        }
        flip ^= 1;
        r = rnew;
    }
    if (rc == TTSVD_OK) {
        // gather T^(1) (tt_svd.hpp:616-621): row 0 of each partition's 1 x r matrix
        const size_t cnt = (size_t)n_slabs * r;
        rc = ensure(ctx->ws_send, cnt * 8);
        if (rc == TTSVD_OK) rc = ensure(ctx->ws_recv, (size_t)P_total * r * 8);
        double* send = as<double>(ctx->ws_send);
        for (int64_t p = 0; p < n_slabs && rc == TTSVD_OK; ++p) {
            cudaError_t e = cudaMemcpy2DAsync(send + p * r, 8, cur[p].data, cur[p].ld * 8, 8, r,
                                              cudaMemcpyDeviceToDevice, ctx->stream);
            if (e != cudaSuccess) rc = fail(TTSVD_ERR_DEVICE, cudaGetErrorString(e));
        }
        double* recv = send;
        if (rc == TTSVD_OK && exchanged) {
            recv = as<double>(ctx->ws_recv);
            rc = all_gather(send, recv, (int64_t)cnt);
        }
        std::vector<double> vals((size_t)P_total * r);
        if (rc == TTSVD_OK) rc = d2h(ctx, vals.data(), recv, vals.size());  // synchronises: the V blocks have landed
        if (rc == TTSVD_OK) {
            flush();
            std::vector<double> first((size_t)P_total * r);
            for (int64_t p = 0; p < P_total; ++p)
                for (int64_t b = 0; b < r; ++b) first[p + P_total * b] = vals[p * r + b];
            tt->cores[0] = std::move(first);
            tt->ranks[0] = 1;
            tt->ranks[1] = r;
            tt->ranks[d] = 1;
        }
    }
    cudaStreamSynchronize(ctx->stream);
    return done(rc);
}

int ttsvd_cu_comm_unique_id(void* id_out) {
    if (!id_out) return fail(TTSVD_ERR_INVALID, "comm_unique_id: null out");
    if (!nccl().ok) return fail(TTSVD_ERR_DEVICE, nccl().why);
    ncclUniqueId id;
    TT_NCCL(nccl().get_unique_id(&id));
    static_assert(sizeof(ncclUniqueId) == TTSVD_COMM_ID_BYTES, "NCCL unique id size");
    std::memcpy(id_out, &id, sizeof id);
    return TTSVD_OK;
}

int ttsvd_cu_ctx_comm_init(ttsvd_cu_ctx* ctx, const void* unique_id, int nranks, int rank) {
    TT_TRY(set_device(ctx));
    if (!unique_id || nranks < 1 || rank < 0 || rank >= nranks) return fail(TTSVD_ERR_INVALID, "comm_init: bad arguments");
    if (!nccl().ok) return fail(TTSVD_ERR_DEVICE, nccl().why);
    if (ctx->comm) nccl().comm_destroy(ctx->comm);
    ctx->comm = nullptr;
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof id);
    TT_NCCL(nccl().comm_init_rank(&ctx->comm, nranks, id, rank));
    ctx->comm_rank = rank;
    ctx->comm_size = nranks;
    return TTSVD_OK;
}

int ttsvd_cu_ctx_comm_init_all(ttsvd_cu_ctx* const* ctxs, int ndev) {
    if (!ctxs || ndev < 1) return fail(TTSVD_ERR_INVALID, "comm_init_all: bad arguments");
    if (!nccl().ok) return fail(TTSVD_ERR_DEVICE, nccl().why);
    std::vector<int> devs(ndev);
    for (int i = 0; i < ndev; ++i) {
        if (!ctxs[i]) return fail(TTSVD_ERR_INVALID, "comm_init_all: null context");
        devs[i] = ctxs[i]->device;
        if (ctxs[i]->comm) nccl().comm_destroy(ctxs[i]->comm);
        ctxs[i]->comm = nullptr;
    }
    std::vector<ncclComm_t> comms(ndev);
    TT_NCCL(nccl().comm_init_all(comms.data(), ndev, devs.data()));
    for (int i = 0; i < ndev; ++i) {
        ctxs[i]->comm = comms[i];
        ctxs[i]->comm_rank = i;
        ctxs[i]->comm_size = ndev;
    }
    return TTSVD_OK;
}

int ttsvd_cu_tt_svd_distributed_devices(ttsvd_cu_ctx* const* ctxs, int ndev, const double* const* slabs,
                                        int64_t slabs_per_device, const int64_t* ldims, int64_t d_local,
                                        int64_t ld_slab, int64_t r_max, double eps, ttsvd_cu_tt** out) {
    if (!ctxs || ndev < 1 || !slabs || slabs_per_device < 1 || !out)
        return fail(TTSVD_ERR_INVALID, "tt_svd_distributed_devices: bad arguments");
    *out = nullptr;
    for (int i = 0; i < ndev; ++i)
        if (!ctxs[i] || !ctxs[i]->comm || ctxs[i]->comm_size != ndev || ctxs[i]->comm_rank != i)
            return fail(TTSVD_ERR_INVALID, "tt_svd_distributed_devices: contexts need ttsvd_cu_ctx_comm_init_all");
    // one host thread per device (SURVEY §8 e topology); the shared cores come
    // out bitwise identical on every device, device 0's train is returned
    const int64_t P = (int64_t)ndev * slabs_per_device;
    std::vector<ttsvd_cu_tt*> res(ndev, nullptr);
    std::vector<int> rcs(ndev, TTSVD_OK);
    std::vector<std::string> msgs(ndev);
    std::vector<std::thread> pool;
    for (int i = 0; i < ndev; ++i)
        pool.emplace_back([&, i] {
            rcs[i] = ttsvd_cu_tt_svd_distributed(ctxs[i], slabs + (size_t)i * slabs_per_device, slabs_per_device,
                                                 (int64_t)i * slabs_per_device, P, ldims, d_local, ld_slab, r_max,
                                                 eps, nullptr, nullptr, &res[i]);
            if (rcs[i] != TTSVD_OK) msgs[i] = g_last_error;
        });
    for (auto& t : pool) t.join();
    for (int i = 1; i < ndev; ++i) ttsvd_cu_tt_free(res[i]);
    for (int i = 0; i < ndev; ++i)
        if (rcs[i] != TTSVD_OK) {
            ttsvd_cu_tt_free(res[0]);
            return fail(rcs[i], "device " + std::to_string(i) + ": " + msgs[i]);
        }
    *out = res[0];
    return TTSVD_OK;
}

int64_t ttsvd_cu_tt_d(const ttsvd_cu_tt* tt) { return tt ? (int64_t)tt->dims.size() : -1; }

int ttsvd_cu_tt_ranks(const ttsvd_cu_tt* tt, int64_t* ranks) {
    if (!tt || !ranks) return fail(TTSVD_ERR_INVALID, "tt_ranks: null");
    std::copy(tt->ranks.begin(), tt->ranks.end(), ranks);
    return TTSVD_OK;
}

int ttsvd_cu_tt_core(const ttsvd_cu_tt* tt, int64_t j, double* dst) {
    if (!tt || !dst || j < 0 || j >= (int64_t)tt->cores.size()) return fail(TTSVD_ERR_INVALID, "tt_core: bad index");
    std::copy(tt->cores[j].begin(), tt->cores[j].end(), dst);
    return TTSVD_OK;
}

int64_t ttsvd_cu_tt_nsteps(const ttsvd_cu_tt* tt) { return tt ? (int64_t)tt->steps.size() : -1; }

int ttsvd_cu_tt_step(const ttsvd_cu_tt* tt, int64_t s, ttsvd_cu_step* o) {
    if (!tt || !o || s < 0 || s >= (int64_t)tt->steps.size()) return fail(TTSVD_ERR_INVALID, "tt_step: bad index");
    *o = tt->steps[s];
    return TTSVD_OK;
}

int ttsvd_cu_tt_sigma(const ttsvd_cu_tt* tt, int64_t s, double* dst) {
    if (!tt || !dst || s < 0 || s >= (int64_t)tt->sigmas.size()) return fail(TTSVD_ERR_INVALID, "tt_sigma: bad index");
    std::copy(tt->sigmas[s].begin(), tt->sigmas[s].end(), dst);
    return TTSVD_OK;
}

void ttsvd_cu_tt_free(ttsvd_cu_tt* tt) { delete tt; }

int ttsvd_cu_gen_partition(ttsvd_cu_ctx* ctx, uint64_t seed, int kind, double scale, int64_t total, int64_t rows,
                           int64_t ld, int64_t nparts, int64_t part, double* X) {
    TT_TRY(set_device(ctx));
    if (!X || rows < 1 || ld < rows || total < 0 || nparts < 1 || part < 0 || part >= nparts || (kind != 0 && kind != 1))
        return fail(TTSVD_ERR_INVALID, "gen_partition: bad arguments");
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)ctx->num_sms * 16);
    gen_partition_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, ctx->stream>>>(seed, kind, scale, total, rows,
                                                                                          ld, nparts, part, X);
    return check_launch(ctx, "gen_partition_kernel");
}

int ttsvd_cu_gen_uniform(ttsvd_cu_ctx* ctx, uint64_t seed, int64_t total, int64_t rows, int64_t ld, double* X) {
    TT_TRY(set_device(ctx));
    if (!X || rows < 1 || ld < rows || total < 0) return fail(TTSVD_ERR_INVALID, "gen_uniform: bad arguments");
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)ctx->num_sms * 16);
    gen_uniform_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, ctx->stream>>>(seed, total, rows, ld, X);
    return check_launch(ctx, "gen_uniform_kernel");
}

}  // extern "C"
