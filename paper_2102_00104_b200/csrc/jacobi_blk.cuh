// K_SVD, m > ~96 without accumulation (the TT-SVD driver's Jacobi on R^T or
// W^T): block one-sided Jacobi, cluster resident, inner work on the FP64
// tensor cores.
//
// The n x m matrix is cut into blocks of 4 columns and lives in the shared
// memory of one thread-block cluster (C <= 16 CTAs).  A round pairs every
// block with one other block (round-robin tournament over block pairs, the
// block analogue of circle_pair); per block pair (8 columns B, 4 warps):
//
//   1. G = B^T B (8 x 8) by DMMA m8n8k4, the k dimension running over rows;
//   2. the rotations one-sided Jacobi would take on B's columns, computed
//      from the Gram entries (two-sided updates G <- J^T G J, Q <- Q J;
//      small_svd.hpp:84-96: skip rule |gamma| <= 1e2 eps sqrt(alpha beta),
//      zeta/t/c/s, pair oriented p < q by global column index): the 16 cross
//      pairs in 4 disjoint sub-rounds at every visit, the 12 pairs inside
//      the two blocks in 3 more sub-rounds at the first round of a sweep;
//   3. B <- B Q by DMMA (skipped when no pair rotated).
//
// Between rounds the slot of every block pair moves (top row one slot right,
// bottom row one slot left; top[h-1] -> bot[h-1], bot[0] -> top[1]); moves
// inside a CTA relabel buffers, the two blocks that cross a CTA boundary are
// copied into the neighbour's inbox through distributed shared memory (the
// inbox indices are pushed ahead by the receiver), one cluster barrier per
// round.  A sweep is
// nblk_pad - 1 rounds, so every column pair meets at least once per sweep;
// the matrix has converged after a sweep in which no pair rotated (Gram
// entries are recomputed from the columns at every visit, so the stopping
// test is the reference's), at most max_sweeps.
//
// Compared with the pairwise kernels this moves each column through shared
// memory 3x per round for 4 columns' worth of pairs (Gram read, apply read +
// write) and replaces 511 latency-bound rounds per sweep (m = 512) by 127.
#pragma once

#include <cfloat>
#include <cstdint>

namespace ttsvd_b200 {

struct BjArgs {
    double* A;  // n x m, ld n (global); overwritten with the orthogonalised columns
    int n, m;
    int n8;   // rows rounded up to 8 (zero rows in shared memory)
    int ldc;  // shared-memory column stride (n8 rounded to 16, + 4: conflict-free fragments)
    int C;    // CTAs in the cluster
    int* status;
    int max_sweeps;
    long long* prof;  // optional (diagnostics): CTA 0 cycle sums [gram, solve, apply, moves + cluster barrier],
                      // then block-pair visits that rotated, per sweep (all CTAs) [4 + sweep]
};

constexpr int kBjThreads = 512;

__device__ __forceinline__ long long bj_clock() {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
    return t;
}
constexpr int kBjWpg = 4;                               // warps per block pair
constexpr int kBjSlots = kBjThreads / (32 * kBjWpg);   // block-pair slots per CTA

inline int bj_ldc(int n8) { return ((n8 + 15) / 16) * 16 + 4; }
inline size_t bj_smem_bytes(int ldc) { return (size_t)(2 * kBjSlots + 2) * 4 * ldc * sizeof(double); }

__device__ __forceinline__ void bj_group_sync(int grp) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(kBjWpg * 32) : "memory");
}

// a block that leaves the CTA unchanged: copy it into the neighbour's inbox
// (the 4 warps of its group; no-op for blocks that stay)
__device__ __forceinline__ void bj_copy_block(const double* src, double* dst, int bsz, int t) {
    if (src == dst) return;
    const double2* s2 = reinterpret_cast<const double2*>(src);
    double2* d2 = reinterpret_cast<double2*>(dst);
    for (int i = t; i < bsz / 2; i += kBjWpg * 32) d2[i] = s2[i];
}

// One visit of a block pair (8 columns: blocks bt | bb, 4 columns each, ld
// ldc, rows n8): Gram by DMMA over the group's warps, the rotations on the
// Gram matrix by the solver warp, B <- B Q by DMMA.  Returns (in the solver
// warp) whether any pair rotated.
__device__ __forceinline__ bool bj_visit(double* bt, double* bb, int blt, int blb, bool first_round, int m, int n8,
                                         int ldc, double (*gpart)[64], double* Gs, double* Qs, int* grp_rot, int grp,
                                         int wg, bool solver, int lane, double* dt, double* db, int bsz,
                                         long long* pf = nullptr) {
    const long long tv0 = pf ? bj_clock() : 0;
    const double tol = 1e2 * DBL_EPSILON;
    bool rotated = false;
    // ---- 1. Gram partials: lane l reads column l/4, rows 4q + l%4 ----
    {
        const int c = lane >> 2;
        const double* col = (c < 4 ? bt + c * ldc : bb + (c - 4) * ldc) + (lane & 3);
        double acc0[2] = {0.0, 0.0}, acc1[2] = {0.0, 0.0};
        const int nq = n8 >> 2;
        int q = wg;
        for (; q + kBjWpg < nq; q += 2 * kBjWpg) {
            const double v0 = col[4 * q], v1 = col[4 * (q + kBjWpg)];
            dmma884(acc0, v0, v0);
            dmma884(acc1, v1, v1);
        }
        if (q < nq) {
            const double v0 = col[4 * q];
            dmma884(acc0, v0, v0);
        }
        double* gp = gpart[wg];
        gp[(lane >> 2) * 8 + 2 * (lane & 3)] = acc0[0] + acc1[0];
        gp[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = acc0[1] + acc1[1];
    }
    bj_group_sync(grp);
    const long long tv1 = pf ? bj_clock() : 0;
    // ---- 2. rotations on the Gram matrix (the solver warp) ----
    if (solver) {
        double* G = Gs;
        double* Q = Qs;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = lane + 32 * h, i = e >> 3, j = e & 7;
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < kBjWpg; ++w) s += gpart[w][e];
            G[i * 9 + j] = s;
            Q[i * 9 + j] = (i == j) ? 1.0 : 0.0;
        }
        int any = 0;
        __syncwarp();
        // sub-rounds 0..3: the 16 cross pairs (top i, bottom (i + s) mod 4);
        // sub-rounds 4..6 (first round of a sweep only): the 12 pairs
        // inside the two blocks, so every pair meets once per sweep
        const int nsub = first_round ? 7 : 4;
        const int kp = lane & 3;
        for (int s = 0; s < nsub; ++s) {
            int x, y;
            if (s < 4) {
                x = kp;
                y = 4 + ((kp + s) & 3);
            } else {
                const int base = kp < 2 ? 0 : 4, j = kp & 1, t = s - 4;
                x = base + (t == 0 ? 2 * j : j);
                y = base + (t == 0 ? 2 * j + 1 : (t == 1 ? j + 2 : 3 - j));
            }
            const int gx = x < 4 ? 4 * blt + x : 4 * blb + x - 4;
            const int gy = y < 4 ? 4 * blt + y : 4 * blb + y - 4;
            const int p = gx < gy ? x : y, q = gx < gy ? y : x;
            // every lane computes the rotation of pair kp (no broadcast round trip)
            const double al = G[p * 9 + p], be = G[q * 9 + q], ga = G[p * 9 + q];
            double c = 1.0, sn = 0.0;
            if (ga * ga > (tol * tol) * (al * be)) {
                // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (be - al) / (2 ga),
                // rewritten without the first division: t = sign(dd) h / (|dd| + sqrt(dd^2 + h^2))
                const double dd = be - al, h = 2.0 * ga;
                const double t = (dd == 0.0) ? 1.0
                                             : ((dd > 0.0) ? h : -h) * __drcp_rn(fabs(dd) + sqrt(fma(dd, dd, h * h)));
                c = rsqrt(fma(t, t, 1.0));
                sn = c * t;
                any = 1;
            }
            {
                // columns: (x_p, x_q) <- (c x_p - s x_q, s x_p + c x_q) on G and Q
                const int i = lane >> 2;
                const double gp = G[i * 9 + p], gq = G[i * 9 + q];
                const double qp = Q[i * 9 + p], qq = Q[i * 9 + q];
                __syncwarp();
                G[i * 9 + p] = c * gp - sn * gq;
                G[i * 9 + q] = sn * gp + c * gq;
                Q[i * 9 + p] = c * qp - sn * qq;
                Q[i * 9 + q] = sn * qp + c * qq;
            }
            __syncwarp();
            {
                // rows of G: J^T (G J); lane -> (pair lane >> 3, column lane & 7)
                const int src = lane >> 3;
                const double c2 = __shfl_sync(0xffffffffu, c, src);
                const double s2 = __shfl_sync(0xffffffffu, sn, src);
                const int p2 = __shfl_sync(0xffffffffu, p, src), q2 = __shfl_sync(0xffffffffu, q, src);
                const int j = lane & 7;
                const double gp = G[p2 * 9 + j], gq = G[q2 * 9 + j];
                G[p2 * 9 + j] = c2 * gp - s2 * gq;
                G[q2 * 9 + j] = s2 * gp + c2 * gq;
            }
            __syncwarp();
        }
        any = __any_sync(0xffffffffu, any);
        if (lane == 0) *grp_rot = any;
        rotated = any;
    }
    bj_group_sync(grp);
    const long long tv2 = pf ? bj_clock() : 0;
    // ---- 3. B <- B Q (DMMA; 8-row tiles) ----
    if (*grp_rot) {
        const double* Q = Qs;
        const double q0 = Q[(lane & 3) * 9 + (lane >> 2)];
        const double q1 = Q[(4 + (lane & 3)) * 9 + (lane >> 2)];
        const int ce = 2 * (lane & 3);
        double* o0 = ce < 4 ? dt + ce * ldc : db + (ce - 4) * ldc;  // a block leaving the CTA goes straight to its inbox
#pragma unroll 4
        for (int t = wg; t < (n8 >> 3); t += kBjWpg) {
            const int rr = 8 * t + (lane >> 2);
            const double a0 = bt[(lane & 3) * ldc + rr];
            const double a1 = bb[(lane & 3) * ldc + rr];
            double d[2] = {0.0, 0.0};
            dmma884(d, a0, q0);
            dmma884(d, a1, q1);
            o0[rr] = d[0];
            o0[ldc + rr] = d[1];
        }
    } else {
        bj_copy_block(bt, dt, bsz, wg * 32 + lane);
        bj_copy_block(bb, db, bsz, wg * 32 + lane);
    }
    if (pf) {
        const long long tv3 = bj_clock();
        pf[0] += tv1 - tv0;
        pf[1] += tv2 - tv1;
        pf[2] += tv3 - tv2;
    }
    return rotated;
}

__global__ void __launch_bounds__(kBjThreads, 1) jacobi_bj_kernel(BjArgs a) {
    constexpr int S = kBjSlots;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double smem[];
    __shared__ int top_buf[S], bot_buf[S], top_blk[S], bot_blk[S];
    __shared__ int inbox_idx[2][2], inbox_blk[2][2], rot[2];
    __shared__ int rdst[2], ldst[2];  // neighbours' inbox buffers for my sends (pushed by them)
    __shared__ int grp_rot[S];
    __shared__ double gpart[S][kBjWpg][64];
    __shared__ double Gs[S][8 * 9], Qs[S][8 * 9];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int grp = warp / kBjWpg, wg = warp % kBjWpg;
    const int n = a.n, m = a.m, n8 = a.n8, ldc = a.ldc, C = a.C;
    const int bsz = 4 * ldc;
    const int k = (int)cl.block_rank();
    if (tid < S) {
        const int g = k * S + tid;
        top_buf[tid] = tid;
        bot_buf[tid] = S + tid;
        top_blk[tid] = 2 * g;  // blocks past the last hold zero columns: their pairs never rotate
        bot_blk[tid] = 2 * g + 1;
    }
    if (tid == 0) {
        inbox_idx[0][0] = 2 * S;
        inbox_idx[0][1] = 2 * S + 1;
        rdst[0] = 2 * S;
        ldst[0] = 2 * S + 1;
        rot[0] = rot[1] = 0;
    }
    __syncthreads();
    // stage the 2S blocks of this CTA (zero columns beyond m, zero rows beyond n)
    for (int e = tid; e < 2 * S * 4 * n8; e += kBjThreads) {
        const int slot = e / (4 * n8), rem = e % (4 * n8), c = rem / n8, i = rem % n8;
        const int blk = slot < S ? top_blk[slot] : bot_blk[slot - S];
        const int buf = slot < S ? top_buf[slot] : bot_buf[slot - S];
        const int col = blk * 4 + c;
        smem[(int64_t)buf * bsz + c * ldc + i] = (col < m && i < n) ? a.A[(int64_t)col * n + i] : 0.0;
    }
    cl.sync();
    const int rounds = 2 * S * C - 1;
    int sweep = 0, par = 0;
    bool converged = (m < 2);
    for (; sweep < a.max_sweeps && !converged; ++sweep) {
        if (tid == 0) rot[sweep & 1] = 0;
        __syncthreads();
        for (int r = 0; r < rounds; ++r, par ^= 1) {
            const int blt = top_blk[grp], blb = bot_blk[grp];
            const bool active = 4 * blt < m || 4 * blb < m;
            double* bt = smem + (int64_t)top_buf[grp] * bsz;
            double* bb = smem + (int64_t)bot_buf[grp] * bsz;
            long long* pfv = (a.prof && blockIdx.x == 0 && tid == 0) ? a.prof : nullptr;
            const long long tr0 = pfv ? bj_clock() : 0;
            // the two blocks that leave the CTA this round are written straight
            // into the neighbours' inboxes (DSMEM) by their visit
            double* dt = bt;
            double* db = bb;
            if (k < C - 1 && grp == S - 1) dt = cl.map_shared_rank(smem, k + 1) + (int64_t)rdst[par] * bsz;
            if (k > 0 && grp == 0) db = cl.map_shared_rank(smem, k - 1) + (int64_t)ldst[par] * bsz;
            if (active) {
                if (bj_visit(bt, bb, blt, blb, r == 0, m, n8, ldc, gpart[grp], Gs[grp], Qs[grp], &grp_rot[grp], grp, wg,
                             wg == grp, lane, dt, db, bsz, pfv)) {
                    rot[sweep & 1] = 1;
                    if (a.prof && lane == 0 && sweep < 28) atomicAdd((unsigned long long*)&a.prof[4 + sweep], 1ull);
                }
            } else {
                bj_copy_block(bt, dt, bsz, wg * 32 + lane);
                bj_copy_block(bb, db, bsz, wg * 32 + lane);
            }
            const long long tr1 = pfv ? bj_clock() : 0;
            __syncthreads();
            // ---- block moves: boundary blocks -> neighbours' inboxes ----
            if (tid == 0) {
                if (k < C - 1) *cl.map_shared_rank(&inbox_blk[par][0], k + 1) = top_blk[S - 1];
                if (k > 0) *cl.map_shared_rank(&inbox_blk[par][1], k - 1) = bot_blk[0];
            }
            if (tid == 0) {
                // the blocks just sent free their buffers: they become my inboxes for
                // the next round, and the neighbours that fill them are told now
                int in0 = -1, in1 = -1;
                if (k < C - 1) (k > 0 ? in0 : in1) = top_buf[S - 1];
                if (k > 0) (k < C - 1 ? in1 : in0) = bot_buf[0];
                if (in0 >= 0) {
                    inbox_idx[par ^ 1][0] = in0;
                    if (k > 0) *cl.map_shared_rank(&rdst[par ^ 1], k - 1) = in0;
                }
                if (in1 >= 0) {
                    inbox_idx[par ^ 1][1] = in1;
                    if (k < C - 1) *cl.map_shared_rank(&ldst[par ^ 1], k + 1) = in1;
                }
            }
            cl.sync();
            if (pfv) pfv[3] += bj_clock() - tr1;
            if (warp == 0) {
                const int j = lane < S ? lane : S - 1;
                const int tb = top_buf[j], tc = top_blk[j], bb_ = bot_buf[j], bc = bot_blk[j];
                const int tb_up = __shfl_up_sync(0xffffffffu, tb, 1), tc_up = __shfl_up_sync(0xffffffffu, tc, 1);
                const int bb_dn = __shfl_down_sync(0xffffffffu, bb_, 1), bc_dn = __shfl_down_sync(0xffffffffu, bc, 1);
                const int bb0 = __shfl_sync(0xffffffffu, bb_, 0), bc0 = __shfl_sync(0xffffffffu, bc, 0);
                const int tbl = __shfl_sync(0xffffffffu, tb, S - 1), tcl = __shfl_sync(0xffffffffu, tc, S - 1);
                int ntb, ntc, nbb, nbc;
                if (j == 0) {
                    if (k == 0) ntb = tb, ntc = tc;
                    else ntb = inbox_idx[par][0], ntc = inbox_blk[par][0];
                } else if (j == 1 && k == 0) {
                    ntb = bb0, ntc = bc0;
                } else {
                    ntb = tb_up, ntc = tc_up;
                }
                if (j == S - 1) {
                    if (k == C - 1) nbb = tbl, nbc = tcl;
                    else nbb = inbox_idx[par][1], nbc = inbox_blk[par][1];
                } else {
                    nbb = bb_dn, nbc = bc_dn;
                }
                __syncwarp();
                if (lane < S) {
                    top_buf[j] = ntb;
                    top_blk[j] = ntc;
                    bot_buf[j] = nbb;
                    bot_blk[j] = nbc;
                }
            }
            __syncthreads();
        }
        int any = 0;
        for (int q = 0; q < C; ++q) any |= *(volatile int*)cl.map_shared_rank(&rot[sweep & 1], q);
        converged = (any == 0);
    }
    for (int e = tid; e < 2 * S * 4 * n; e += kBjThreads) {
        const int slot = e / (4 * n), rem = e % (4 * n), c = rem / n, i = rem % n;
        const int blk = slot < S ? top_blk[slot] : bot_blk[slot - S];
        const int buf = slot < S ? top_buf[slot] : bot_buf[slot - S];
        const int col = blk * 4 + c;
        if (col < m) a.A[(int64_t)col * n + i] = smem[(int64_t)buf * bsz + c * ldc + i];
    }
    if (k == 0 && tid == 0) *a.status = converged ? sweep : -1;
    cl.sync();  // no CTA leaves while a neighbour may still read its flags
}



}  // namespace ttsvd_b200
