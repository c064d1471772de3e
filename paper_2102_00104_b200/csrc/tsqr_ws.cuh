// K_TSQR for narrow work matrices (m <= 32): warp streams.
//
// Every SW lanes of a warp (SW = 16 for m <= 16, else 32) form an independent
// stream that owns a contiguous row range and its own R (m x m, shared
// memory).  Lane c of a stream keeps column c of the current 32-row tile in
// registers; the structured [R; tile] QR is one panel, so a tile costs m
// reflectors and no trailing update — the pivot column is published in
// shared memory, each lane takes its dot product with it, derives the
// reflector (LAPACK dlarfg normalisation, zero rules of tsqr.hpp:120-160, as
// la_panel) and updates its column.  Thousands of streams per GPU hide the
// reflector latency.  Each stream writes its R into rows [s m, (s+1) m) of a
// stacked (S m) x m matrix, which the next level factors the same way with
// fewer streams (the flat-then-tree structure of tsqr.hpp:247-292).
#pragma once

#include <cfloat>
#include <cstdint>

namespace ttsvd_b200 {

constexpr int kWsThreads = 256;

struct WsArgs {
    const double* X;
    int64_t n, ld;
    int m;
    int64_t S;    // streams
    double* out;  // stacked factors (S m x m, ld ldo), or R (m x m, ld m) when S == 1
    int64_t ldo;
};

template <int SW>
__host__ __device__ constexpr int ws_rld() {
    return SW + 1;
}

constexpr int kWsSld = 34;  // column stride of a stream's staged tile (32 rows, 16-byte aligned)

template <int SW>
inline size_t ws_smem_bytes() {
    return (size_t)(kWsThreads / 32) * (32 / SW) * (32 + SW * ws_rld<SW>() + SW * kWsSld) * sizeof(double);
}

template <int SW>
__global__ void __launch_bounds__(kWsThreads, 2) tsqr_ws_kernel(WsArgs a) {
    extern __shared__ __align__(16) double sm[];
    constexpr int SPW = 32 / SW;  // streams per warp
    constexpr int RLD = ws_rld<SW>();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane / SW, sl = lane % SW;
    const int64_t s = ((int64_t)blockIdx.x * (kWsThreads / 32) + warp) * SPW + sub;
    const bool live = s < a.S;
    double* pv = sm + (size_t)(warp * SPW + sub) * (32 + SW * RLD + SW * kWsSld);
    double* Rs = pv + 32;
    double* stg = Rs + SW * RLD;  // the tile, column-major (ld kWsSld), staged by coalesced loads
    const int m = a.m;
    for (int e = sl; e < SW * RLD; e += SW) Rs[e] = 0.0;
    int64_t row0 = 0, row1 = 0;
    if (live) {
        const int64_t base = a.n / a.S, rem = a.n % a.S;
        row0 = s * base + (s < rem ? s : rem);
        row1 = row0 + base + (s < rem ? 1 : 0);
    }
    // every stream of the warp runs the same number of tiles (idle tiles are zero)
    int64_t my_tiles = (row1 - row0 + 31) / 32, tiles = my_tiles;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const int64_t t = __shfl_xor_sync(kFull, tiles, o);
        tiles = t > tiles ? t : tiles;
    }
    const unsigned s_pv = (unsigned)__cvta_generic_to_shared(pv);
    const unsigned s_rcol = (unsigned)__cvta_generic_to_shared(Rs + sl * RLD);
    const unsigned s_r = (unsigned)__cvta_generic_to_shared(Rs);
    __syncwarp();
    for (int64_t t = 0; t < tiles; ++t) {
        const int64_t r0 = row0 + 32 * t;
        const int rows = (t < my_tiles) ? (int)((row1 - r0) < 32 ? (row1 - r0) : 32) : 0;
        // coalesced: the stream's lanes walk down each column (32 rows = SW lanes x 32/SW)
        for (int c = 0; c < m; ++c) {
            const double* col = a.X + (int64_t)c * a.ld + r0;
#pragma unroll
            for (int h = 0; h < 32 / SW; ++h) {
                const int i = sl + SW * h;
                stg[c * kWsSld + i] = (i < rows) ? __ldcs(col + i) : 0.0;
            }
        }
        __syncwarp();
        double x[32];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            const double2 v = (sl < m) ? *reinterpret_cast<const double2*>(stg + sl * kWsSld + i) : make_double2(0.0, 0.0);
            x[i] = v.x;
            x[i + 1] = v.y;
        }
        for (int j = 0; j < m; ++j) {
            const bool piv = (sl == j);
#pragma unroll
            for (int i = 0; i < 32; i += 2) sts2_if(piv, s_pv + 8 * i, x[i], x[i + 1]);
            __syncwarp();
            double acc[8];
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const double2 p0 = lds2(s_pv + 8 * i);
                if (i < 16) {
                    acc[i / 2] = p0.x * x[i];
                    acc[i / 2] = fma(p0.y, x[i + 1], acc[i / 2]);
                } else {
                    acc[(i - 16) / 2] = fma(p0.x, x[i], acc[(i - 16) / 2]);
                    acc[(i - 16) / 2] = fma(p0.y, x[i + 1], acc[(i - 16) / 2]);
                }
            }
            const double d = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
            const double sp = __shfl_sync(kFull, d, sub * SW + j);
            const double u0 = lds1(s_r + 8 * j * (RLD + 1));
            const double rjc = lds1(s_rcol + 8 * j);
            const double nrm2 = u0 * u0 + sp;
            const double inv = rsqrt(nrm2);
            const double nr = nrm2 * inv;
            const double au = fabs(u0);
            const double sg = (u0 > 0.0) ? 1.0 : -1.0;
            double alpha = -sg * nr;
            double tj = 1.0 + au * inv;
            double scale = sg * __drcp_rn(au + nr);
            if (sp == 0.0 && u0 != 0.0) {  // H = I
                alpha = u0;
                tj = 0.0;
                scale = 0.0;
            }
            if (nrm2 == 0.0) {  // all-zero u
                alpha = sqrt(2.0 * DBL_MIN);
                tj = 2.0;
                scale = 0.0;
            }
            const bool upd = sl > j;
            const double g = tj * (rjc + scale * d);
            const double f = upd ? g * scale : 0.0;
            __syncwarp();
            sts1_if(upd, s_rcol + 8 * j, rjc - g);
            sts1_if(piv, s_r + 8 * j * (RLD + 1), alpha);
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const double2 p0 = lds2(s_pv + 8 * i);
                x[i] = fma(-f, p0.x, x[i]);
                x[i + 1] = fma(-f, p0.y, x[i + 1]);
            }
            __syncwarp();
        }
    }
    if (live && sl < m) {
        double* o = a.out + (int64_t)sl * a.ldo + (a.S == 1 ? 0 : s * m);
        for (int i = 0; i < m; ++i) o[i] = (i <= sl) ? Rs[sl * RLD + i] : 0.0;
    }
}

}  // namespace ttsvd_b200
