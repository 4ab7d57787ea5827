// eigen_sbr.cu -- two-stage tridiagonalisation of the large Kronecker factors (Alg. 1 step 2,
// the eigendecomposition each owner runs per factor; the result feeds Eqs. 13-15).
//
// The one-stage Householder reduction (eigen_trd.cu, trd_panel) needs a symmetric mat-vec over the
// whole trailing matrix and two grid-wide reductions per column: a latency chain of n steps that
// bounds a lone d = 4609 factor at ~20 us per column.  Here the reduction is split (successive band
// reduction, Bischof-Lang-Sun; the dense -> band -> tridiagonal scheme of two-stage LAPACK/MAGMA
// eigensolvers, re-derived for this design in scripts/sbr_prototype.py):
//
//   stage 1  F -> B = Q1^T F Q1, lower bandwidth b = 16.  Per panel of 16 columns p .. p+15:
//            Householder QR of the m x 16 block below the band (m = n - p - 16) on one 8-CTA
//            cluster (the panel lives in distributed shared memory; one cluster reduction per
//            column), then the two-sided WY update of the trailing m x m matrix A22 with
//            Q = I - V T V^T:  X = A22 V T (symmetric product from the lower triangle, fp64 DMMA),
//            M = T^T V^T X, W = X - V M / 2, A22 -= V W^T + W V^T (rank-32 fp64 DMMA update of the
//            lower tiles).  Every factor of the batch advances one panel per launch (staggered so
//            all finish together).
//   stage 2  B -> T = Q2^T B Q2 tridiagonal by bulge chasing.  Sweep s annihilates column s below
//            its subdiagonal; its step k applies one 16-long reflector H to rows
//            R_k = [s+1+16k, s+16+16k]: generated from column s (k = 0) or from the first column of
//            the bulge the previous step left (k >= 1), applied from the left to the 15 remaining
//            bulge columns, two-sided to the diagonal block, and from the right to the 16 rows
//            below (which creates the next bulge).  Band plus bulge are 32 entries per row.  One
//            cluster of up to 8 CTAs per factor holds the band in distributed shared memory
//            (rows split in contiguous chunks); a step runs on a warp of the CTA owning its first
//            row.  Step (s, k) waits for (s, k-1) and (s-1, k+2) (steps of sweeps three apart
//            commute; checked exactly in the prototype), so ~3n steps are on the critical path,
//            each a few hundred cycles of shared-memory work.
//   Q2       E = Q2 Z for the eigenvectors Z of T: the reflectors of sweeps 16j .. 16j+15 at step k
//            form block G(j, k) (a 31-row window).  Valid order: j descending, k ascending
//            (prototype); one CTA per 32 columns of Z, lane = column, a warp per pass j with the
//            31-row window in registers, passes pipelined one block apart.
//
// All arithmetic is fp64 (the preconditioner amplifies eigenvector errors by up to Lambda/damping,
// DESIGN.md §8); every reduction runs in a fixed order (bitwise repeatable).
#include "eigen_trd.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

namespace cg = cooperative_groups;

#define SBR_TRY(expr)                        \
    do {                                     \
        kfac_status_t _st = (expr);          \
        if (_st != KFAC_OK) return _st;      \
    } while (0)

namespace kfac {
namespace sbr {
namespace {

constexpr int B = kSbrBw;                  // 16
constexpr int kMaxJobs = 256;              // factors per launch descriptor table
// stage 1 panel QR
constexpr int kQrCl = 8;                   // CTAs per cluster
constexpr int kQrThreads = 512;
constexpr int kQrRows = (kSbrMaxN + kQrCl - 1) / kQrCl;        // panel rows per CTA (max)
constexpr int kQrSlot = 2 * B;             // per-CTA partial slot: 16 column sums + pivot row
// stage 1 products
constexpr int kTm = 64;                    // rows of X per CTA (symmetric product, W)
constexpr int kKc = 32;                    // K chunk of the symmetric product
// stage 2
#ifndef KFAC_SBR_CHASE_WARPS
#define KFAC_SBR_CHASE_WARPS 8
#endif
constexpr int kChaseWarps = KFAC_SBR_CHASE_WARPS;
#ifndef KFAC_SBR_CHASE_ROWS
#define KFAC_SBR_CHASE_ROWS 320
#endif
constexpr int kChaseRows = KFAC_SBR_CHASE_ROWS;   // target band rows per CTA (32 doubles each)
constexpr int kChaseMaxCs = 16;            // CTAs per cluster (non-portable above 8)
constexpr int kBandLd = 2 * B;             // band row: A[i][i - t], t = 0 .. 31
// Q2
constexpr int kQ2Warps = 8;

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp16(void *smem, const void *gmem, bool valid) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// number of stage-1 panels of an n x n factor: p = 0, 16, ... while the block below the band has
// at least two rows (m = n - p - 16 >= 2)
__host__ __device__ inline int num_panels(int n) { return n >= B + 2 ? (n - B - 2) / B + 1 : 0; }

// ================================================================ stage 1: panel QR (cluster) ==
struct PanelSet {
    const TrdJob *jobs;
    int count;
    int job[kMaxJobs];
    int p0[kMaxJobs];
    int tile_begin[kMaxJobs + 1];        // 64-row tiles of X (symmetric product / W kernels)
};

__device__ __forceinline__ int find_item(const PanelSet &S, int tile) {
    int lo = 0, hi = S.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (S.tile_begin[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Householder QR (LAPACK dgeqr2 order) of the m x 16 panel P = A[q:n, p:p+16], q = p + 16, rows
// split over the cluster's CTAs.  Column j: every CTA sums x_r P[r][c] over its rows r > j (x = P[:, j];
// c = j gives ||x_{j+1:}||^2), the cluster adds the 8 partials in rank order, and with the pivot row
// P[j][:] every CTA forms beta, tau and w_c = tau v^T P[:, c] = tau (S_c / (alpha - beta) + P[j][c])
// and updates its rows: P[r][c] -= v_r w_c, v_r = x_r / (alpha - beta).  The update of column j+1
// and the next column's partial sums are fused (each warp owns whole rows, so a __syncwarp orders
// its reads before its writes); column j itself keeps x and is scaled to v at the end.  Writes R
// into A, the reflectors into Vd (column p + j, unit entry at row q + j), tau, and the WY factor T
// (dlarft from the Gram matrix V^T V, reduced over the cluster the same way).
__global__ void __cluster_dims__(kQrCl, 1, 1) __launch_bounds__(kQrThreads, 1)
    sbr_panel_qr(const __grid_constant__ PanelSet S) {
    extern __shared__ __align__(16) double qsm[];
    double *P = qsm;                                   // [kQrRows][16]
    double *slot = P + kQrRows * B;                    // [2][kQrSlot]  (read by the whole cluster)
    double *gram = slot + 2 * kQrSlot;                 // [256]         (read by the whole cluster)
    double *red = gram + B * B;                        // [warps][16]
    double *coef = red + (kQrThreads / 32) * B;        // [32]: column sums, pivot row
    double *Tsm = coef + 2 * B;                        // [16][17]
    double *Gf = Tsm + B * 17;                         // [256]: the cluster's Gram matrix (rank 0)
    __shared__ double tau_s[B], scale_s[B], beta_s[B];
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int item = blockIdx.x / kQrCl;
    const TrdJob &J = S.jobs[S.job[item]];
    const int n = J.n, ldw = J.ldw, p = S.p0[item], q = p + B, m = n - q;
    const int lo = (int)((long long)m * rank / kQrCl), hi = (int)((long long)m * (rank + 1) / kQrCl);
    const int rows = hi - lo;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    constexpr int kWarps = kQrThreads / 32;
    const int c = lane & (B - 1), h = lane >> 4;        // warp rows 2 warp + h + 2 kWarps it, column c

    for (int e = t; e < rows * B; e += kQrThreads) {
        const int r = e >> 4, cc = e & (B - 1);
        P[e] = J.Ad[(size_t)(q + lo + r) * ldw + p + cc];
    }
    __syncthreads();
    const int nr = min(B, m);
    // partial sums of column 0
    double acc = 0.0;
    for (int r0 = 2 * warp; r0 < rows; r0 += 2 * kWarps) {
        const int r = r0 + h;
        if (r < rows && lo + r > 0) acc = fma(P[r * B], P[r * B + c], acc);
    }
    for (int j = 0; j < nr; ++j) {
        double *my = slot + (j & 1) * kQrSlot;
        acc += __shfl_xor_sync(0xffffffffu, acc, 16);
        if (lane < B) red[warp * B + lane] = acc;
        __syncthreads();
        if (t < B) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) s += red[w * B + t];
            my[t] = s;
        } else if (t < 2 * B) {
            if (lo <= j && j < hi) my[t] = P[(j - lo) * B + (t - B)];
        }
        cluster.sync();
        if (t < 2 * B) {
            double v = 0.0;
            if (t < B) {
                double pv[kQrCl];
#pragma unroll
                for (int rk = 0; rk < kQrCl; ++rk) pv[rk] = cluster.map_shared_rank(my, rk)[t];
#pragma unroll
                for (int rk = 0; rk < kQrCl; ++rk) v += pv[rk];
            } else {
                int owner = 0;
                for (int rk = 0; rk < kQrCl; ++rk)
                    if ((long long)m * rk / kQrCl <= j) owner = rk;
                v = cluster.map_shared_rank(my, owner)[t];
            }
            coef[t] = v;
        }
        __syncthreads();
        const double alpha = coef[B + j], xn2 = coef[j];
        double beta = alpha, tau = 0.0, scale = 0.0;
        if (xn2 > 0.0) {
            beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
            tau = (beta - alpha) / beta;
            scale = 1.0 / (alpha - beta);
        }
        if (t == 0) {
            tau_s[j] = tau;
            scale_s[j] = scale;
            beta_s[j] = beta;
        }
        const double wc = (c > j) ? tau * (coef[c] * scale + coef[B + c]) : 0.0;
        const double wn = (j + 1 < B) ? tau * (coef[j + 1] * scale + coef[B + j + 1]) : 0.0;
        // rows r > j: P[r][c] -= x_r scale w_c; pivot row: P[j][c] -= w_c.  Fused: partial sums of
        // column j+1 over rows r > j+1 from the updated values (computed locally for column j+1).
        acc = 0.0;
        for (int r0 = 2 * warp; r0 < rows; r0 += 2 * kWarps) {
            const int r = r0 + h, gi = lo + r;
            double pc = 0.0, pn = 0.0, xj = 0.0;
            const bool ok = r < rows;
            if (ok) {
                pc = P[r * B + c];
                xj = P[r * B + j];
                if (j + 1 < B) pn = P[r * B + j + 1];
            }
            __syncwarp();
            if (ok && gi >= j) {
                const double f = gi > j ? xj * scale : 1.0;
                if (c > j) {
                    pc = fma(-f, wc, pc);
                    P[r * B + c] = pc;
                }
                pn = fma(-f, wn, pn);
                if (gi > j + 1) acc = fma(pn, pc, acc);
            }
        }
        __syncthreads();
    }
    for (int j = nr + t; j < B; j += kQrThreads) {
        tau_s[j] = 0.0;
        scale_s[j] = 0.0;
    }
    __syncthreads();
    // columns j < nr: rows > j hold x (scale to v), row j gets beta
    for (int e = t; e < rows * B; e += kQrThreads) {
        const int r = e >> 4, cc = e & (B - 1), gi = lo + r;
        if (cc < nr) {
            if (gi > cc) P[e] *= scale_s[cc];
            else if (gi == cc) P[e] = beta_s[cc];
        }
    }
    __syncthreads();
    // write back R (rows < 16 of the panel, on/above the diagonal), V (unit lower trapezoid), tau
    for (int e = t; e < rows * B; e += kQrThreads) {
        const int r = e >> 4, cc = e & (B - 1), gi = lo + r;
        const size_t row = (size_t)(q + gi) * ldw;
        if (gi <= cc) J.Ad[row + p + cc] = P[e];
        if (cc < nr) J.Vd[row + p + cc] = gi > cc ? P[e] : (gi == cc ? 1.0 : 0.0);
    }
    if (rank == 0 && t < B) J.tau[p + t] = tau_s[t];
    // Gram matrix G = V^T V over this CTA's rows, then over the cluster (rank order)
    if (t < B * B) {
        const int a = t >> 4, b2 = t & (B - 1);
        double gacc = 0.0;
        for (int r = 0; r < rows; ++r) {
            const int gi = lo + r;
            const double va = gi > a ? P[r * B + a] : (gi == a ? 1.0 : 0.0);
            const double vb = gi > b2 ? P[r * B + b2] : (gi == b2 ? 1.0 : 0.0);
            gacc = fma(va, vb, gacc);
        }
        gram[t] = gacc;
    }
    cluster.sync();
    if (rank == 0) {
        if (t < B * B) {
            double G = 0.0;
            for (int rk = 0; rk < kQrCl; ++rk) G += cluster.map_shared_rank(gram, rk)[t];
            Gf[t] = G;
        }
        for (int e = t; e < B * 17; e += kQrThreads) Tsm[e] = 0.0;
        __syncthreads();
        // dlarft (forward, columnwise): T_jj = tau_j, T[0:j, j] = -tau_j T[0:j, 0:j] G[0:j, j]
        for (int j = 0; j < B; ++j) {
            double a2 = 0.0;
            if (t < j)
                for (int l = t; l < j; ++l) a2 += Tsm[t * 17 + l] * Gf[l * B + j];
            __syncthreads();
            if (t < j) Tsm[t * 17 + j] = -tau_s[j] * a2;
            if (t == j) Tsm[j * 17 + j] = tau_s[j];
            __syncthreads();
        }
        if (t < B * B) J.Ts[t] = Tsm[(t >> 4) * 17 + (t & 15)];
    }
    cluster.sync();                                     // keep this CTA's shared memory alive
}

// ============================================================ stage 1: X = A22 V (split over K) ==
// One CTA per (64 rows of X, K range): 4 warps x 16 rows, K in chunks of 32 through two cp.async
// stages.  A22 is read from its lower triangle only: chunks left of the tile read A[i][k]
// (k-contiguous), chunks right of it read A[k][i] (the mirrored element, i-contiguous), the two
// chunks crossing the diagonal load both and pick per element.  Products on the fp64 tensor cores
// (DMMA m8n8k4); each CTA writes its K-range partial of X (summed in a fixed order by sbr_xt).
constexpr int kAsLd = kKc + 2, kAtLd = kTm + 4, kVsLd = B + 2;
constexpr int kSymmStage = kTm * kAsLd + kKc * kAtLd + kKc * kVsLd;       // doubles per stage
constexpr int kSymmSmem = 2 * kSymmStage * 8;
constexpr int kMaxSplit = 8;

__global__ void __launch_bounds__(128) sbr_symm(const __grid_constant__ PanelSet S, int splits) {
    extern __shared__ __align__(16) double ssm[];
    const int unit = blockIdx.x / splits, sp = blockIdx.x % splits;
    const int item = find_item(S, unit);
    const TrdJob &J = S.jobs[S.job[item]];
    const int n = J.n, ldw = J.ldw, p = S.p0[item], q = p + B, m = n - q;
    const int tile = unit - S.tile_begin[item], i0 = tile * kTm;
    const double *A = J.Ad + (size_t)q * ldw + q;      // A22 origin
    const double *V = J.Vd + (size_t)q * ldw + p;      // V[i][c] = V[i * ldw + c]
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, g = lane >> 2, qd = lane & 3;

    const int nk_all = (m + kKc - 1) / kKc;
    const int kt0 = (int)((long long)nk_all * sp / splits), kt1 = (int)((long long)nk_all * (sp + 1) / splits);
    auto ctype = [&](int k0) { return (k0 + kKc <= i0) ? 0 : (k0 >= i0 + kTm ? 1 : 2); };
    auto issue = [&](int kt, int buf) {
        if (kt < kt1) {
            double *st = ssm + buf * kSymmStage;
            double *As = st, *At = st + kTm * kAsLd, *Vs = At + kKc * kAtLd;
            const int k0 = kt * kKc, ty = ctype(k0);
            if (ty != 1) {                                 // As[i][k] = A[i0+i][k0+k]
                for (int ch = t; ch < kTm * (kKc / 2); ch += 128) {
                    const int i = ch / (kKc / 2), k = (ch % (kKc / 2)) * 2;
                    const bool ok = (i0 + i < m) && (k0 + k < m);
                    cp16(As + i * kAsLd + k, ok ? A + (size_t)(i0 + i) * ldw + k0 + k : A, ok);
                }
            }
            if (ty != 0) {                                 // At[k][i] = A[k0+k][i0+i]
                for (int ch = t; ch < kKc * (kTm / 2); ch += 128) {
                    const int k = ch / (kTm / 2), i = (ch % (kTm / 2)) * 2;
                    const bool ok = (k0 + k < m) && (i0 + i < m);
                    cp16(At + k * kAtLd + i, ok ? A + (size_t)(k0 + k) * ldw + i0 + i : A, ok);
                }
            }
            for (int ch = t; ch < kKc * (B / 2); ch += 128) {   // Vs[k][c] = V[k0+k][c]
                const int k = ch / (B / 2), cc = (ch % (B / 2)) * 2;
                const bool ok = k0 + k < m;
                cp16(Vs + k * kVsLd + cc, ok ? V + (size_t)(k0 + k) * ldw + cc : V, ok);
            }
        }
        cp_commit();
    };
    double acc[2][2][2] = {};
    issue(kt0, 0);
    for (int kt = kt0; kt < kt1; ++kt) {
        const int buf = (kt - kt0) & 1;
        issue(kt + 1, buf ^ 1);
        cp_wait<1>();
        __syncthreads();
        const double *st = ssm + buf * kSymmStage;
        const double *As = st, *At = st + kTm * kAsLd, *Vs = At + kKc * kAtLd;
        const int k0 = kt * kKc, ty = ctype(k0);
#pragma unroll
        for (int kk = 0; kk < kKc; kk += 4) {
            const int k = kk + qd;
            double a[2], b[2];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) {
                const int i = warp * 16 + mi * 8 + g;
                const bool low = ty == 0 || (ty == 2 && k0 + k <= i0 + i);
                a[mi] = low ? As[i * kAsLd + k] : At[k * kAtLd + i];
            }
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) b[ni] = Vs[k * kVsLd + ni * 8 + g];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi)
#pragma unroll
                for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
        __syncthreads();
    }
    cp_wait<0>();
    double *Xp = J.Xs + (size_t)(1 + sp) * J.n * B;    // partial sp (slot 0 holds X')
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
            const int i = i0 + warp * 16 + mi * 8 + g, cc = ni * 8 + 2 * qd;
            if (i < m) *reinterpret_cast<double2 *>(Xp + (size_t)i * B + cc) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
        }
}

// ========================================== stage 1: X' = (sum of partials) T, V^T X' partials ==
__global__ void __launch_bounds__(256) sbr_xt(const __grid_constant__ PanelSet S, int splits) {
    __shared__ double Xt[kTm * 17], Tsm[B * 17], Vt[kTm * 17];
    const int item = find_item(S, blockIdx.x);
    const TrdJob &J = S.jobs[S.job[item]];
    const int n = J.n, ldw = J.ldw, p = S.p0[item], q = p + B, m = n - q;
    const int tile = blockIdx.x - S.tile_begin[item], i0 = tile * kTm;
    const int t = threadIdx.x;
    const double *V = J.Vd + (size_t)q * ldw + p;
    for (int e = t; e < kTm * B; e += 256) {
        const int i = e >> 4, cc = e & 15;
        double x = 0.0, v = 0.0;
        if (i0 + i < m) {
            for (int sp = 0; sp < splits; ++sp) x += J.Xs[(size_t)(1 + sp) * n * B + (size_t)(i0 + i) * B + cc];
            v = V[(size_t)(i0 + i) * ldw + cc];
        }
        Xt[i * 17 + cc] = x;
        Vt[i * 17 + cc] = v;
    }
    Tsm[(t >> 4) * 17 + (t & 15)] = J.Ts[t];
    __syncthreads();
    double xp[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {                      // X' rows (t >> 4) + 16 u, column t & 15
        const int i = (t >> 4) + 16 * u, cc = t & 15;
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < B; ++l) s = fma(Xt[i * 17 + l], Tsm[l * 17 + cc], s);
        xp[u] = (i0 + i < m) ? s : 0.0;
        if (i0 + i < m) J.Xs[(size_t)(i0 + i) * B + cc] = s;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) Xt[((t >> 4) + 16 * u) * 17 + (t & 15)] = xp[u];
    __syncthreads();
    {
        const int a = t >> 4, cc = t & 15;
        double s = 0.0;
        for (int i = 0; i < kTm; ++i) s = fma(Vt[i * 17 + a], Xt[i * 17 + cc], s);
        J.Ps[(size_t)tile * B * B + t] = s;
    }
}

// ======================================= stage 1: M = T^T V^T X', W = X' - V M / 2, [V|W], [W|V] ==
__global__ void __launch_bounds__(256) sbr_make_w(const __grid_constant__ PanelSet S) {
    __shared__ double Ssm[B * 17], Msm[B * 17], Tsm[B * 17];
    const int item = find_item(S, blockIdx.x);
    const TrdJob &J = S.jobs[S.job[item]];
    const int n = J.n, ldw = J.ldw, p = S.p0[item], q = p + B, m = n - q;
    const int tile = blockIdx.x - S.tile_begin[item], i0 = tile * kTm;
    const int ntiles = S.tile_begin[item + 1] - S.tile_begin[item];
    const int t = threadIdx.x, a = t >> 4, cc = t & 15;
    double s = 0.0;
    for (int u = 0; u < ntiles; ++u) s += J.Ps[(size_t)u * B * B + t];     // fixed order
    Ssm[a * 17 + cc] = s;
    Tsm[a * 17 + cc] = J.Ts[t];
    __syncthreads();
    double mv = 0.0;
#pragma unroll
    for (int l = 0; l < B; ++l) mv = fma(Tsm[l * 17 + a], Ssm[l * 17 + cc], mv);      // (T^T S)[a][cc]
    Msm[a * 17 + cc] = mv;
    __syncthreads();
    const double *V = J.Vd + (size_t)q * ldw + p;
    for (int e = t; e < kTm * B; e += 256) {
        const int i = i0 + e / B, c2 = e % B;
        if (i >= m) continue;
        double w = J.Xs[(size_t)i * B + c2];
        double vm = 0.0;
#pragma unroll
        for (int l = 0; l < B; ++l) vm = fma(V[(size_t)i * ldw + l], Msm[l * 17 + c2], vm);
        w -= 0.5 * vm;
        const double v = V[(size_t)i * ldw + c2];
        J.VWs[(size_t)i * 2 * B + c2] = v;
        J.VWs[(size_t)i * 2 * B + B + c2] = w;
        J.WVs[(size_t)i * 2 * B + c2] = w;
        J.WVs[(size_t)i * 2 * B + B + c2] = v;
    }
}

// ====================================================================== stage 2: bulge chasing ==
#ifndef KFAC_SBR_TIMING
#define KFAC_SBR_TIMING 0
#endif
#if KFAC_SBR_TIMING
// Diagnostic build only (-DKFAC_SBR_TIMING=1): %globaltimer stamps (wait begin, step begin, step
// end) of the steps of sweeps s < kTimS of the first factor; read with kfac_debug_sbr_timing.
constexpr int kTimS = 256, kTimK = 360;
__device__ unsigned long long g_sbr_tim[kTimS][kTimK][4];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif
struct ChaseSet {
    const TrdJob *jobs;
    int count;
    int job[kMaxJobs];
};

__device__ __forceinline__ void fence_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
// Shared-memory-only cluster fences (PTX 8.6): release of this CTA's own shared-memory writes to a
// neighbour that reads them remotely (MEMBAR.CTA, no GPU-scope membar), and the matching acquire.
__device__ __forceinline__ void fence_release_own_smem() {
    asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_acquire_cluster_smem() {
    asm volatile("fence.acquire.sync_restrict::shared::cluster.cluster;" ::: "memory");
}
__device__ __forceinline__ int ld_volatile(const int *p) { return *reinterpret_cast<const volatile int *>(p); }
__device__ __forceinline__ void st_volatile(int *p, int v) { *reinterpret_cast<volatile int *>(p) = v; }

// Event counter of one warp (shared memory): cnt = steps completed so far (monotone) and an mbarrier
// with one arrival per step.  A waiting warp sleeps in mbarrier.try_wait (no polling traffic that
// would slow the warps doing work); the counter resolves which phase to wait for, and the bounded
// suspend re-checks it if the producer ran two phases ahead in between.  ev_signal is called by one
// lane; ev_wait by the whole warp (a lone sleeping lane with the rest parked in __syncwarp costs
// ~10 us to reconverge, measured).
__device__ __forceinline__ void ev_init(unsigned long long *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void ev_signal(unsigned long long *bar, int *cnt, int v) {
    __threadfence_block();
    st_volatile(cnt, v);
    asm volatile("{ .reg .b64 st; mbarrier.arrive.release.cta.shared::cta.b64 st, [%0]; }" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void ev_wait(unsigned long long *bar, const int *cnt, int target) {
    const uint32_t addr = (uint32_t)__cvta_generic_to_shared(bar);
    for (;;) {
        const int c = ld_volatile(cnt);
        if (c >= target) break;
        uint32_t done;
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(addr), "r"((uint32_t)(c & 1)), "r"(2000u)
            : "memory");
    }
    __threadfence_block();
}

__device__ __forceinline__ int chase_steps(int n, int s) { return (n - 2 - s) / B + 1; }   // a_k <= n - 1

// Householder reflector of x (LAPACK dlarfg) from alpha = x_0 and sq = ||x_{1:}||^2, with one
// division: d = alpha - beta, inv = 1 / (beta d)  ->  tau = (beta - alpha) / beta = -d^2 inv,
// scale = 1 / (alpha - beta) = beta inv.
__device__ __forceinline__ void house(double alpha, double sq, double &beta, double &tau, double &scale) {
    beta = alpha;
    tau = 0.0;
    scale = 0.0;
    if (sq > 0.0) {
        beta = -copysign(sqrt(fma(alpha, alpha, sq)), alpha);
        const double d = alpha - beta, inv = 1.0 / (beta * d);
        tau = -d * d * inv;
        scale = beta * inv;
    }
}

// Interior step (every row a .. a+31 in this CTA and inside the matrix; most steps): the same
// arithmetic as chase_step below with compile-time shared-memory offsets.
__device__ __forceinline__ double chase_interior(double *rowa, int k, int lane, double &vout) {
    const int ac = k ? B : 1;                                      // a - c
    const int L = lane & (B - 1);
    const double x = rowa[L * (kBandLd + 1) + ac];                 // A[a + L][c]
    const double alpha = __shfl_sync(0xffffffffu, x, 0);
    double sq = L >= 1 ? x * x : 0.0;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    double beta, tau, scale;
    house(alpha, sq, beta, tau, scale);
    const double v = L == 0 ? 1.0 : x * scale;
    vout = lane < B ? v : 0.0;
    if (tau == 0.0) return 0.0;
    double vr[B];
#pragma unroll
    for (int i = 0; i < B; ++i) vr[i] = __shfl_sync(0xffffffffu, v, i);
    double *p;
    int stride;
    if (lane >= B) { p = rowa + lane * (kBandLd + 1); stride = -1; }
    else if (lane == B - 1) { p = rowa + ac; stride = kBandLd + 1; }
    else { p = rowa + (B - 1 - lane); stride = kBandLd + 1; }
    const bool act = lane >= B - 1 || k > 0;
    double e1[B], d3[B];
#pragma unroll
    for (int l = 0; l < B; ++l) e1[l] = act ? p[l * stride] : 0.0;
#pragma unroll
    for (int m = 0; m < B; ++m) d3[m] = rowa[(kBandLd + 1) * max(L, m) - min(L, m)];
    double q1[4] = {0.0, 0.0, 0.0, 0.0}, q3[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int l = 0; l < B; ++l) {
        q1[l & 3] = fma(vr[l], e1[l], q1[l & 3]);
        q3[l & 3] = fma(vr[l], d3[l], q3[l & 3]);
    }
    const double w1 = ((q1[0] + q1[1]) + (q1[2] + q1[3])) * tau;
    const double y = (q3[0] + q3[1]) + (q3[2] + q3[3]);
    if (act) {
        const bool colc = lane == B - 1;
#pragma unroll
        for (int l = 0; l < B; ++l) p[l * stride] = colc ? (l == 0 ? beta : 0.0) : fma(-vr[l], w1, e1[l]);
    }
    double vy = v * y;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) vy += __shfl_xor_sync(0xffffffffu, vy, o);
    const double w = tau * y - 0.5 * tau * tau * vy * v;
    double wr[B];
#pragma unroll
    for (int i = 0; i < B; ++i) wr[i] = __shfl_sync(0xffffffffu, w, i);
    __syncwarp();                    // lanes 16..31 read these rows (d3) before lanes 0..15 write them
    if (lane < B) {
        double *Rr = rowa + L * (kBandLd + 1);
#pragma unroll
        for (int m = 0; m < B; ++m)
            if (m <= L) Rr[-m] = d3[m] - fma(v, wr[m], w * vr[m]);
    }
    return tau;
}

// One step (s, k) of the bulge chase by one warp; rows a .. a+31 are lanes 0 .. 31.  Returns tau
// (for Rq), with v_lane in vout (v_0 = 1).  Straight-line: lanes 16..31 duplicate lanes 0..15 for
// the reflector and the diagonal block (so the 16-lane reductions need no broadcast and nothing
// diverges); v and w are broadcast into every lane's registers by shuffles; phase 1 is one strided
// 16-element run per lane: bulge column a-15+lane (lanes 0..14, k > 0), column c (lane 15: set to
// beta e_0), row a+lane (lanes 16..31, band offsets lane - l).  Band row a + l is R(l):
//   REMOTE: rows >= hi (l >= lh = hi - a) live in the next CTA (cluster window `nxt`);
//   END:    rows > n - 1 do not exist (read as zero, never written).
template <bool REMOTE, bool END>
__device__ __forceinline__ double chase_step(double *rowa, double *nxt, int lh, int lv, int s, int k, int lane,
                                             double &vout) {
    const int ac = k ? B : 1;                                      // a - c
    const int L = lane & (B - 1);
    auto R = [&](int l) -> double * {
        if (REMOTE && l >= lh) return nxt + (size_t)(l - lh) * kBandLd;
        return rowa + (size_t)l * kBandLd;
    };
    auto ok = [&](int l) { return !END || l < lv; };               // row a + l inside the matrix
    const double x = ok(L) ? R(L)[L + ac] : 0.0;                   // A[a + L][c]
    const double alpha = __shfl_sync(0xffffffffu, x, 0);
    double sq = L >= 1 ? x * x : 0.0;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    double beta, tau, scale;
    house(alpha, sq, beta, tau, scale);
    const double v = L == 0 ? 1.0 : x * scale;
    vout = lane < B ? v : 0.0;
    if (tau == 0.0) return 0.0;
    double vr[B];
#pragma unroll
    for (int i = 0; i < B; ++i) vr[i] = __shfl_sync(0xffffffffu, v, i);
    // phase 1 element l: row lane (lanes >= 16, offset lane - l) or row l (offset l + 15 - lane;
    // lane 15: l + ac)
    const bool act = lane >= B ? ok(lane) : (lane == B - 1 || k > 0);
    const int off1 = lane == B - 1 ? ac : B - 1 - lane;
    double *own = lane >= B ? R(lane) : nullptr;
    double e1[B], d3[B];
#pragma unroll
    for (int l = 0; l < B; ++l) {
        double *q = lane >= B ? own + (lane - l) : R(l) + (l + off1);
        e1[l] = (act && (lane >= B || ok(l))) ? *q : 0.0;
    }
    double *mine = R(L);
#pragma unroll
    for (int m = 0; m < B; ++m) {
        if (REMOTE) d3[m] = ok(max(L, m)) ? (m <= L ? mine[L - m] : R(m)[m - L]) : 0.0;
        else d3[m] = ok(max(L, m)) ? rowa[(kBandLd + 1) * max(L, m) - min(L, m)] : 0.0;
    }
    double q1[4] = {0.0, 0.0, 0.0, 0.0}, q3[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int l = 0; l < B; ++l) {
        q1[l & 3] = fma(vr[l], e1[l], q1[l & 3]);
        q3[l & 3] = fma(vr[l], d3[l], q3[l & 3]);
    }
    const double w1 = ((q1[0] + q1[1]) + (q1[2] + q1[3])) * tau;
    const double y = (q3[0] + q3[1]) + (q3[2] + q3[3]);
    if (act) {
        const bool colc = lane == B - 1;
#pragma unroll
        for (int l = 0; l < B; ++l) {
            double *q = lane >= B ? own + (lane - l) : R(l) + (l + off1);
            if (lane >= B || ok(l)) *q = colc ? (l == 0 ? beta : 0.0) : fma(-vr[l], w1, e1[l]);
        }
    }
    double vy = v * y;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) vy += __shfl_xor_sync(0xffffffffu, vy, o);
    const double w = tau * y - 0.5 * tau * tau * vy * v;
    double wr[B];
#pragma unroll
    for (int i = 0; i < B; ++i) wr[i] = __shfl_sync(0xffffffffu, w, i);
    __syncwarp();
    if (lane < B && ok(L)) {
#pragma unroll
        for (int m = 0; m < B; ++m)
            if (m <= L) mine[L - m] = d3[m] - fma(v, wr[m], w * vr[m]);
    }
    return tau;
}

// Shared memory: band rows [lo, hi) x 32 doubles, one event counter per warp, prog[n].
// Warp w runs the segments (steps in this chunk) of sweeps s = w, w + NW, ...  Step (s, k) waits
// for (s, k-1) -- the same warp, or for the segment's first step the previous CTA -- and for
// (s-1, k+2): warp w-1 of this CTA (its event counter: the target count is known from the segment
// lengths both warps walk through) or, near the chunk end, the next CTA.  Cross-CTA dependencies go
// through prog[] (the producer writes the neighbour's copy) with a cluster-scope fence; they occur
// only in the first and last steps of a segment.
__global__ void __launch_bounds__(kChaseWarps * 32, 1) sbr_chase(const __grid_constant__ ChaseSet S) {
    extern __shared__ __align__(16) double csm[];
    __shared__ unsigned long long ev_bar[kChaseWarps];
    __shared__ int ev_cnt[kChaseWarps];
    cg::cluster_group cluster = cg::this_cluster();
    const int CS = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
    const TrdJob &J = S.jobs[S.job[blockIdx.x / CS]];
    const int n = J.n, ldw = J.ldw;
    const int Lr = (n + CS - 1) / CS, lo = min(n, rank * Lr), hi = min(n, lo + Lr);
    double *band = csm;                                          // [Lr][32]
    int *prog = reinterpret_cast<int *>(band + (size_t)Lr * kBandLd);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

    for (int e = t; e < (hi - lo) * kBandLd; e += blockDim.x) {
        const int i = lo + e / kBandLd, tt = e % kBandLd;
        band[e] = (tt <= B && i - tt >= 0) ? J.Ad[(size_t)i * ldw + i - tt] : 0.0;
    }
    for (int e = t; e < n; e += blockDim.x) prog[e] = 0;
    if (t < kChaseWarps) {
        ev_init(&ev_bar[t]);
        ev_cnt[t] = 0;
    }
    cluster.sync();
    double *band_next = rank + 1 < CS ? cluster.map_shared_rank(band, rank + 1) : nullptr;
    int *prog_prev = rank > 0 ? cluster.map_shared_rank(prog, rank - 1) : nullptr;
    int *prog_next = rank + 1 < CS ? cluster.map_shared_rank(prog, rank + 1) : nullptr;
    double *rq_prev = nullptr, tau_prev = 0.0, v_prev = 0.0;
    auto seg_lo = [&](int s) { return lo > s + 1 ? (lo - s - 1 + B - 1) / B : 0; };
    auto seg_hi = [&](int s) { return min(chase_steps(n, s) - 1, (hi - 2 - s) / B); };   // s + 1 < hi
    const int pw = (warp + kChaseWarps - 1) % kChaseWarps;      // warp of sweep s - 1
    int mycnt = 0, pbase = 0;

    for (int s = warp; s < n - 2; s += kChaseWarps) {
        if (s + 1 >= hi) break;                                   // later sweeps start beyond this chunk too
        const int k_lo = seg_lo(s), k_hi = seg_hi(s);
        const int pns = s > 0 ? chase_steps(n, s - 1) : 0;
        const int pk_lo = s > 0 ? seg_lo(s - 1) : 0, pk_hi = s > 0 ? seg_hi(s - 1) : -1;
        for (int k = k_lo; k <= k_hi; ++k) {
            const int a = s + 1 + B * k;
#if KFAC_SBR_TIMING
            const bool tim = blockIdx.x < CS && s < kTimS && k < kTimK && lane == 0;
            if (tim) { g_sbr_tim[s][k][0] = gtime(); g_sbr_tim[s][k][3] = rank; }
#endif
            {                                                     // the whole warp waits (no divergence)
                bool remote = false;
                if (k == k_lo && k > 0) {                         // (s, k-1) ran on the previous CTA
                    while (ld_volatile(prog + s) < k) __nanosleep(32);
                    remote = true;
                }
                if (s > 0) {
                    const int k2 = min(k + 2, pns - 1);           // (s-1, k2) must be complete
                    if (k2 <= pk_hi) {
                        ev_wait(&ev_bar[pw], &ev_cnt[pw], pbase + (k2 - pk_lo) + 1);
                    } else {
                        while (ld_volatile(prog + s - 1) < k2 + 1) __nanosleep(32);
                        remote = true;
                    }
                }
                if (remote) fence_acquire_cluster_smem();
            }
            __syncwarp();
#if KFAC_SBR_TIMING
            if (tim) g_sbr_tim[s][k][1] = gtime();
#endif
            // the previous step's reflector goes out now, after this step's acquire: a cluster-scope
            // fence waits for the warp's outstanding global stores
#ifndef KFAC_SBR_EXP_NORQ
            if (rq_prev && lane < B) rq_prev[lane] = lane == 0 ? tau_prev : v_prev;
#endif
            const bool full = a + 2 * B - 1 < hi, end = a + 2 * B - 1 > n - 1;
            double *rowa = band + (size_t)(a - lo) * kBandLd;
            const int lh = hi - a, lv = n - a;
            double v, tau;
            if (full && !end) tau = chase_interior(rowa, k, lane, v);
            else if (full) tau = chase_step<false, true>(rowa, band_next, lh, lv, s, k, lane, v);
            else if (!end) tau = chase_step<true, false>(rowa, band_next, lh, lv, s, k, lane, v);
            else tau = chase_step<true, true>(rowa, band_next, lh, lv, s, k, lane, v);
            __syncwarp();
            if (lane == 0) {
                // consumers: (s+1, k-2) on warp w+1 (event) or the previous CTA (row a - 31),
                // (s, k+1) on this warp or the next CTA (row a + 16); rows written in the next CTA
                // to_next: this step wrote rows of the next CTA (remote stores): full cluster release.
                // to_prev only: the previous CTA's consumer reads our rows: own-shared-memory release.
                const bool to_prev = prog_prev && a - 2 * B + 1 < lo;
                const bool to_next = prog_next && !full;
#ifdef KFAC_SBR_EXP_CHEAP_PUSH_FENCE                              // timing experiment only (unsound)
                if (to_next || to_prev) fence_release_own_smem();
#else
                if (to_next) fence_cluster();
                else if (to_prev) fence_release_own_smem();
#endif
                if (to_prev) st_volatile(prog_prev + s, k + 1);
                if (to_next) st_volatile(prog_next + s, k + 1);
                ev_signal(&ev_bar[warp], &ev_cnt[warp], ++mycnt);
            }
            rq_prev = J.Rq + ((size_t)k * n + s) * B;
            tau_prev = tau;
            v_prev = v;
#if KFAC_SBR_TIMING
            if (tim) g_sbr_tim[s][k][2] = gtime();
#endif
        }
        if (s > 0) pbase += max(0, pk_hi - pk_lo + 1);
    }
    if (rq_prev && lane < B) rq_prev[lane] = lane == 0 ? tau_prev : v_prev;
    cluster.sync();
    for (int i = lo + t; i < hi; i += blockDim.x) {
        J.d[i] = band[(size_t)(i - lo) * kBandLd];
        if (i >= 1) J.e[i - 1] = band[(size_t)(i - lo) * kBandLd + 1];
    }
    if (rank == CS - 1 && t == 0) J.e[n - 1] = 0.0;
    cluster.sync();
}

// ========================================================================== Q2 application ==
struct Q2Set {
    const TrdJob *jobs;
    int count;
    int job[kMaxJobs];
    int slab_begin[kMaxJobs + 1];
};

__device__ __forceinline__ int find_slab(const Q2Set &S, int b) {
    int lo = 0, hi = S.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (S.slab_begin[mid] <= b) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Z <- Q2 Z on 32 columns (lane = column).  Pass j applies the blocks G(j, 0), G(j, 1), ... (sweeps
// 16j .. 16j+15, each block in reverse product order s = 16j+15 .. 16j) and its block k waits for
// pass j+1's block k (the only earlier blocks it overlaps).  Block k's window is rows r0 .. r0+30
// (r0 = 16j + 1 + 16k) in registers: its last 15 rows are the next block's first 15, so a block
// loads 16 new rows and stores the 16 rows it leaves behind; the next block's reflectors are
// prefetched into shared memory (cp.async) while this one is applied.
__global__ void __launch_bounds__(kQ2Warps * 32, 1) sbr_q2(const __grid_constant__ Q2Set S) {
    __shared__ __align__(16) double rs[kQ2Warps][2][B * B];
    __shared__ unsigned long long ev_bar[kQ2Warps];
    __shared__ int ev_cnt[kQ2Warps];
    const int item = find_slab(S, blockIdx.x);
    const TrdJob &J = S.jobs[S.job[item]];
    const int n = J.n, ldw = J.ldw;
    const int c0 = (blockIdx.x - S.slab_begin[item]) * 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int col = c0 + lane;
    const bool colok = col < n;
    double *Z = final_z(J) + col;
    const int npass = (n - 3) / B + 1;                           // sweeps 0 .. n-3
    if (threadIdx.x < kQ2Warps) {
        ev_init(&ev_bar[threadIdx.x]);
        ev_cnt[threadIdx.x] = 0;
    }
    __syncthreads();
    const int pw = (warp + kQ2Warps - 1) % kQ2Warps;             // warp of pass j + 1
    int mycnt = 0, pbase = 0;
    auto prefetch = [&](int j, int k, int buf) {                 // reflectors of block (j, k)
        const double *src = J.Rq + ((size_t)k * n + B * j) * B;
        const int nvalid = min(B, n - 2 - B * j);
#pragma unroll
        for (int u = 0; u < B * B / 2 / 32; ++u) {
            const int e = (u * 32 + lane) * 2;                   // two doubles per 16-byte copy
            cp16(&rs[warp][buf][e], src + e, e / B < nvalid);
        }
        cp_commit();
    };
    for (int j = npass - 1 - warp; j >= 0; j -= kQ2Warps) {
        const int kmax = (n - 2 - B * j) / B;                     // last step of sweep 16j
        const int kmax_next = j + 1 < npass ? (n - 2 - B * (j + 1)) / B : -1;
        const int nvalid = min(B, n - 2 - B * j);                 // sweeps 16j + i <= n - 3
        double z[2 * B - 1];
        prefetch(j, 0, 0);
        for (int k = 0; k <= kmax; ++k) {
            if (j + 1 < npass) ev_wait(&ev_bar[pw], &ev_cnt[pw], pbase + min(k + 1, kmax_next + 1));
            __syncwarp();
            const int r0 = B * j + 1 + B * k;
            if (k == 0) {
#pragma unroll
                for (int i = 0; i < 2 * B - 1; ++i)
                    z[i] = (colok && r0 + i < n) ? __ldcg(Z + (size_t)(r0 + i) * ldw) : 0.0;
            } else {
#pragma unroll
                for (int i = B - 1; i < 2 * B - 1; ++i)
                    z[i] = (colok && r0 + i < n) ? __ldcg(Z + (size_t)(r0 + i) * ldw) : 0.0;
            }
            if (k < kmax) prefetch(j, k + 1, (k + 1) & 1);
            else cp_commit();
            cp_wait<1>();
            __syncwarp();
            const double *R = rs[warp][k & 1];
#pragma unroll
            for (int i = B - 1; i >= 0; --i) {
                // sweep 16j + i exists at step k iff its rows start inside the matrix
                if (i < nvalid && r0 + i <= n - 1) {
                    const double tau = R[i * B];
                    double d4[4] = {z[i], 0.0, 0.0, 0.0};     // four partial sums: short FMA chains
#pragma unroll
                    for (int l = 1; l < B; ++l) d4[l & 3] = fma(R[i * B + l], z[i + l], d4[l & 3]);
                    const double d = ((d4[0] + d4[1]) + (d4[2] + d4[3])) * tau;
                    z[i] -= d;
#pragma unroll
                    for (int l = 1; l < B; ++l) z[i + l] = fma(-d, R[i * B + l], z[i + l]);
                }
            }
            const bool last = k == kmax;
#pragma unroll
            for (int i = 0; i < 2 * B - 1; ++i)
                if ((i < B || last) && colok && r0 + i < n) Z[(size_t)(r0 + i) * ldw] = z[i];
#pragma unroll
            for (int i = 0; i < B - 1; ++i) z[i] = z[i + B];
            __syncwarp();
            if (lane == 0) ev_signal(&ev_bar[warp], &ev_cnt[warp], ++mycnt);
        }
        cp_wait<0>();
        __syncwarp();
        if (j + 1 < npass) pbase += kmax_next + 1;
    }
}

}  // namespace

// ------------------------------------------------------------------------------------- host --
// Default routing (no KFAC_EIG_*_STAGE flag): the two-stage reduction takes a factor only where it
// shortens the call -- when the factor carries at least kAutoShare of the call's d^3 (its one-stage
// column chain is then the critical path: a lone factor, one rank's share at W >= 4; with many
// factors the one-stage panels share the HBM stream across factors and win) and its size is one the
// two-stage path measures faster at (profiles/r02_*_sbr_*).
#ifndef KFAC_SBR_SHARE
#define KFAC_SBR_SHARE 0.5
#endif
#ifndef KFAC_SBR_MAXN
#define KFAC_SBR_MAXN 4000
#endif
constexpr double kAutoShare = KFAC_SBR_SHARE;
constexpr int kAutoMaxN = KFAC_SBR_MAXN;

std::vector<char> route(const int32_t *dims, int count, uint32_t flags) {
    std::vector<char> r(count, 0);
    if (flags & KFAC_EIG_ONE_STAGE) return r;
    if (flags & KFAC_EIG_TWO_STAGE) {
        for (int i = 0; i < count; ++i) r[i] = eligible(dims[i]);
        return r;
    }
    double total = 0.0;
    for (int i = 0; i < count; ++i) total += (double)dims[i] * dims[i] * dims[i];
    for (int i = 0; i < count; ++i) {
        const double d3 = (double)dims[i] * dims[i] * dims[i];
        r[i] = eligible(dims[i]) && dims[i] <= kAutoMaxN && d3 >= kAutoShare * total;
    }
    return r;
}

size_t extra_bytes(int n, int ldw) {
    size_t cur = 0;
    TrdJob J{};
    J.n = n;
    J.ldw = ldw;
    plan_fields(J, cur);
    return cur;
}

void plan_fields(TrdJob &J, size_t &cur) {
    auto take = [&](size_t bytes) {
        cur = round_up(cur, 256);
        const size_t r = cur;
        cur += bytes;
        return r;
    };
    const size_t n = (size_t)J.n, ldw = (size_t)J.ldw;
    J.Ad = reinterpret_cast<double *>(take(8 * n * ldw));
    J.Xs = reinterpret_cast<double *>(take(8 * n * B * (1 + kMaxSplit)));   // X' | K-split partials of X
    J.VWs = reinterpret_cast<double *>(take(8 * n * 2 * B));
    J.WVs = reinterpret_cast<double *>(take(8 * n * 2 * B));
    J.Ts = reinterpret_cast<double *>(take(8 * B * B));
    J.Ms = reinterpret_cast<double *>(take(8 * B * B));
    J.Ps = reinterpret_cast<double *>(take(8 * (size_t)(cdiv(J.n, kTm) + 1) * B * B));
    J.Rq = reinterpret_cast<double *>(take(8 * ((size_t)(J.n / B) + 2) * n * B));
}

void rebase_fields(TrdJob &J, char *base) {
    auto rb = [&](double *&p) {
        if (p) p = reinterpret_cast<double *>(base + reinterpret_cast<uintptr_t>(p));
    };
    rb(J.Ad); rb(J.Xs); rb(J.VWs); rb(J.WVs); rb(J.Ts); rb(J.Ms); rb(J.Ps); rb(J.Rq);
}

namespace {
constexpr size_t kQrSmem = sizeof(double) * ((size_t)kQrRows * B + 2 * kQrSlot + B * B + (kQrThreads / 32) * B + 2 * B + B * 17 + B * B);

size_t chase_smem(int n, int cs) {
    const int Lr = cdiv(n, cs);
    return sizeof(double) * (size_t)Lr * kBandLd + sizeof(int) * (size_t)n;
}
int chase_cs(int n) { return std::min(kChaseMaxCs, std::max(1, cdiv(n, kChaseRows))); }
}  // namespace

kfac_status_t reduce(const TrdJob *djobs, const std::vector<TrdJob> &jobs, const std::vector<int> &ids,
                     cudaStream_t s) {
    const kfac_status_t st = stage1(djobs, jobs, ids, s);
    if (st != KFAC_OK) return st;
    return chase(djobs, jobs, ids, s);
}

kfac_status_t stage1(const TrdJob *djobs, const std::vector<TrdJob> &jobs, const std::vector<int> &ids,
                     cudaStream_t s) {
    KFAC_CUDA_TRY(set_smem_attr((const void *)sbr_panel_qr, (int)kQrSmem));
    KFAC_CUDA_TRY(set_smem_attr((const void *)sbr_symm, kSymmSmem));
    // ---- stage 1: one panel of every active factor per launch, staggered to finish together ----
    int pmax = 0;
    for (int i : ids) pmax = std::max(pmax, num_panels(jobs[i].n));
    thread_local PanelSet PS;
    std::vector<Gemm64Desc> gd;
    for (int tp = 0; tp < pmax; ++tp) {
        std::vector<int> act;
        for (int i : ids)
            if (tp - (pmax - num_panels(jobs[i].n)) >= 0) act.push_back(i);
        for (size_t c0 = 0; c0 < act.size(); c0 += kMaxJobs) {
            const int na = (int)std::min(act.size() - c0, (size_t)kMaxJobs);
            PS.jobs = djobs;
            PS.count = na;
            int tiles = 0;
            gd.clear();
            for (int u = 0; u < na; ++u) {
                const int i = act[c0 + u];
                const TrdJob &J = jobs[i];
                const int p = B * (tp - (pmax - num_panels(J.n)));
                const int q = p + B, m = J.n - q;
                PS.job[u] = i;
                PS.p0[u] = p;
                PS.tile_begin[u] = tiles;
                tiles += cdiv(m, kTm);
                Gemm64Desc g{};                            // A22 -= [V W] [W V]^T  (lower tiles)
                g.M = m; g.N = m; g.K = 2 * B;
                g.A = J.VWs; g.ta = DT_F64; g.lda = 2 * B;
                g.B = J.WVs; g.tb = DT_F64; g.ldb = 2 * B; g.trans_b = 1;
                g.C = J.Ad + (size_t)q * J.ldw + q; g.tc = DT_F64; g.ldc = J.ldw;
                g.epi = EPI_SUB;
                g.lower = 1;
                gd.push_back(g);
            }
            PS.tile_begin[na] = tiles;
            sbr_panel_qr<<<na * kQrCl, kQrThreads, kQrSmem, s>>>(PS);
            KFAC_LAUNCHED();
            // K split so that the launch fills the GPU twice over (fixed per launch: the partials
            // are summed in split order by sbr_xt)
            const int splits = std::max(1, std::min(kMaxSplit, cdiv(2 * num_sms(), tiles)));
            sbr_symm<<<tiles * splits, 128, kSymmSmem, s>>>(PS, splits);
            KFAC_LAUNCHED();
            sbr_xt<<<tiles, 256, 0, s>>>(PS, splits);
            KFAC_LAUNCHED();
            sbr_make_w<<<tiles, 256, 0, s>>>(PS);
            KFAC_LAUNCHED();
            SBR_TRY(gemm64_grouped(gd.data(), (int)gd.size(), s));
        }
    }
    return KFAC_OK;
}

int chase_ctas(const std::vector<TrdJob> &jobs, const std::vector<int> &ids) {
    int c = 0;
    for (int i : ids) c += chase_cs(jobs[i].n);
    return c;
}

kfac_status_t chase(const TrdJob *djobs, const std::vector<TrdJob> &jobs, const std::vector<int> &ids,
                    cudaStream_t s) {
    // ---- stage 2: one cluster per factor, grouped by cluster size ----
    KFAC_CUDA_TRY(cudaFuncSetAttribute((const void *)sbr_chase, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int cs = 1; cs <= kChaseMaxCs; ++cs) {
        std::vector<int> grp;
        for (int i : ids)
            if (chase_cs(jobs[i].n) == cs) grp.push_back(i);
        for (size_t c0 = 0; c0 < grp.size(); c0 += kMaxJobs) {
            thread_local ChaseSet CSet;
            const int na = (int)std::min(grp.size() - c0, (size_t)kMaxJobs);
            CSet.jobs = djobs;
            CSet.count = na;
            size_t smem = 0;
            for (int u = 0; u < na; ++u) {
                CSet.job[u] = grp[c0 + u];
                smem = std::max(smem, chase_smem(jobs[grp[c0 + u]].n, cs));
            }
            KFAC_CUDA_TRY(set_smem_attr((const void *)sbr_chase, (int)smem));
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(na * cs);
            cfg.blockDim = dim3(kChaseWarps * 32);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = cs;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            KFAC_CUDA_TRY(cudaLaunchKernelEx(&cfg, sbr_chase, CSet));
            KFAC_LAUNCHED();
        }
    }
    return KFAC_OK;
}

kfac_status_t apply_q2(const TrdJob *djobs, const std::vector<TrdJob> &jobs, const std::vector<int> &ids,
                       cudaStream_t s) {
    thread_local Q2Set QS;
    for (size_t c0 = 0; c0 < ids.size(); c0 += kMaxJobs) {
        const int na = (int)std::min(ids.size() - c0, (size_t)kMaxJobs);
        QS.jobs = djobs;
        QS.count = na;
        int slabs = 0;
        for (int u = 0; u < na; ++u) {
            const int i = ids[c0 + u];
            QS.job[u] = i;
            QS.slab_begin[u] = slabs;
            slabs += cdiv(jobs[i].n, 32);
        }
        QS.slab_begin[na] = slabs;
        sbr_q2<<<slabs, kQ2Warps * 32, 0, s>>>(QS);
        KFAC_LAUNCHED();
    }
    return KFAC_OK;
}

}  // namespace sbr
}  // namespace kfac

#if KFAC_SBR_TIMING
extern "C" int kfac_debug_sbr_timing(unsigned long long *out, int count) {
    const size_t want = sizeof(unsigned long long) * kfac::sbr::kTimS * kfac::sbr::kTimK * 4;
    if ((size_t)count * sizeof(unsigned long long) < want) return KFAC_ERR_INVALID_VALUE;
    return cudaMemcpyFromSymbol(out, kfac::sbr::g_sbr_tim, want) == cudaSuccess ? KFAC_OK : KFAC_ERR_CUDA;
}
#endif
