// eigen_trd.cu -- eigendecomposition of the large Kronecker factors (Alg. 1, Eqs. 13-15)
// by the classical three-phase dense symmetric eigensolver, re-designed for B200:
//
//   (1) Householder tridiagonalisation F = H T H^T, H = H_0 H_1 ... H_{n-2}
//       (Golub & Van Loan Alg. 8.3.1; blocked as in LAPACK dsytrd/dlatrd with panels of 32):
//       a persistent cooperative kernel per panel in which every factor of the batch owns a group
//       of CTAs (sized by its remaining work) synchronised by its own global-memory barrier -- two
//       barriers per column; the rank-64 trailing update A -= V W^T + W V^T runs inside the same
//       kernel on the fp64 tensor cores (DMMA).  Working matrix fp32, every reduction in fp64,
//       (d, e, tau) in fp64.  Factors the router sends to the two-stage reduction (eigen_sbr.cu:
//       dense -> band 16 -> tridiagonal) skip these panels.
//   (2) Cuppen's divide and conquer on T (fp64 arithmetic and fp64 eigenvector storage):
//       leaves of <= kLeaf (16) rows by implicit QL (one warp each); each merge solves
//       D + rho z z^T with LAPACK-style deflation (small z_i, and close d_i by a Givens rotation),
//       a bracketed rational-Newton secular solver (one warp per root), the Gu-Eisenstat
//       recomputed z-hat (orthogonal eigenvectors without extra precision), and the
//       eigenvector update Q_nd S as grouped fp64 GEMMs (DMMA, or the Ozaki int8 engine for the
//       large ones) whose N and K are the device-side count of non-deflated roots.
//   (3) back-transformation X = H Z in blocks of 512 reflectors with the compact WY form
//       H_b...H_{b+511} = I - V T V^T (LAPACK dlarft by kTs = 64-blocks joined recursively), three
//       grouped fp64 GEMMs per block (for two-stage factors after Q2, with reflector offset 16).
//
// One-sided block Jacobi (eigen.cu) remains the solver for factors below 64 and warm starts.
#include "eigen_trd.cuh"

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <optional>
#include <vector>

#define RET_OK(expr)                         \
    do {                                     \
        kfac_status_t _st = (expr);          \
        if (_st != KFAC_OK) return _st;      \
    } while (0)

namespace kfac {

size_t trd_workspace_bytes(const int32_t *dims, int count);
kfac_status_t trd_run(const float *const *F, const int32_t *dims, const int32_t *ldF, int count,
                      float *const *Q, const int32_t *ldQ, float *const *evals, int32_t *info, uint32_t flags,
                      void *ws, cudaStream_t s);

namespace {

constexpr int kNb = 32;                 // panel width (reflectors per syr2k)
#ifndef KFAC_TRD_THREADS
#define KFAC_TRD_THREADS 512
#endif
constexpr int kTrdThreads = KFAC_TRD_THREADS;   // 512 (256 with two CTAs per SM measured slower)
constexpr int kTrdCtasPerSm = 512 / kTrdThreads;
constexpr int kTrdWarps = kTrdThreads / 32;
constexpr int kPart = 2 * kNb + 2;      // per-CTA partials: V^T v, W^T v, ||x||^2, w^T v
constexpr int kMaxGroupCtas = 512;
#ifndef KFAC_LEAF
#define KFAC_LEAF 16
#endif
constexpr int kLeaf = KFAC_LEAF;        // D&C leaf size (16: mlp 9.39 -> 9.21 ms, r32 10.14 -> 10.01 ms, r50 within noise)
#ifndef KFAC_SBR_OVERLAP
#define KFAC_SBR_OVERLAP 1
#endif
#ifndef KFAC_SYMV_ROWS
#define KFAC_SYMV_ROWS 32
#endif
constexpr int kSymvR = KFAC_SYMV_ROWS;  // symv tile rows (lower triangle only), multiple of 8
// Rows per warp half of the finer symv unit geometry, the alternative each launch may take (the
// host picks per launch the geometry whose busiest warp pair streams the fewest rows; measured:
// lone d = 4609 116 -> 107 ms with 24 rows throughout, session r2q).
constexpr int kSymvRLone = 24;
constexpr int kSymvRMin = kSymvRLone < kSymvR ? kSymvRLone : kSymvR;   // sizes the TP partials
constexpr int kSymvC = 128;             // symv tile columns (one float4 per lane)
constexpr int kPairR = 2 * kSymvR;       // rows per column partial (a warp pair's two half tiles)
constexpr int kMaxRb = (16384 / kPairR + 31) / 32 * 32;   // super blocks for n <= 16384
#ifndef KFAC_SYMV_FP32
#define KFAC_SYMV_FP32 1                  // fp32 products with 4/8-term fp32 partial sums, fp64 beyond (R23)
#endif
constexpr int kBt = 512;                // reflectors per back-transformation block
constexpr int kTs = 64;                 // dlarft sub-block (T built recursively from 64-blocks: 33 KB of
                                        // shared memory, several CTAs per SM; 128-blocks ran the first
                                        // back-transformation step in 3 waves of one CTA per SM)
constexpr double kEps = 1.1102230246251565e-16;   // 2^-53, LAPACK dlamch('E')


template <class T>
__device__ __forceinline__ T ldcg(const T *p) { return __ldcg(p); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Barrier among the `nc` CTAs of one factor's group (counter zeroed before each launch).  The
// CTA's writes are ordered before thread 0's release add by bar.sync (cumulativity), and its
// acquire poll orders the other CTAs' writes before everything after the closing bar.sync.
__device__ __forceinline__ void group_barrier(unsigned *bar, unsigned &target, int nc) {
    __syncthreads();
    target += (unsigned)nc;
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        while (ld_acquire(bar) < target) {
        }
    }
    __syncthreads();
}

// Block-wide fixed-order sum of one double per thread; result valid in every thread.
__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x / 32); ++i) s += sh[i];
    return s;
}

// Fixed-order sum over the group's CTAs of one partial column, by one warp (lane-strided partial
// sums, then a butterfly): independent loads instead of a chain of nc dependent L2 round trips.
__device__ __forceinline__ double warp_part_sum(const double *part, int col, int nc, int lane) {
    double s = 0.0;
#pragma unroll 4
    for (int q = lane; q < nc; q += 32) s += ldcg(part + (size_t)q * kPart + col);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

__device__ __forceinline__ void part_range(int r0, int n, int c, int nc, int &lo, int &hi) {
    const long long len = n - r0;
    lo = r0 + (int)(len * c / nc);
    hi = r0 + (int)(len * (c + 1) / nc);
}

// ------------------------------------------- small factors: cluster-resident dsytd2 --
// For a call whose factors are all small (d <= ~880: the MLP and ResNet-32 configurations) the
// panel kernel's grid-wide barriers dominate: a d = 785 factor pays ~20 us per column for ~1 us of
// mat-vec bytes.  Here one thread-block cluster of CL <= 16 CTAs holds the factor's lower triangle
// in fp64 in distributed shared memory (row r on CTA r % CL) and runs unblocked Householder
// tridiagonalisation (LAPACK dsytd2, lower; Golub & Van Loan Alg. 8.3.1) with three cluster barriers
// per column and every matrix access local:
//   1  x = A[k+1:n, k] all-gathered (each CTA stores its rows' entries into every CTA's copy);
//   -  every CTA forms the same reflector from the full x (fixed-order sums: bit-identical);
//   2  y = A22 v: row sums of the CTA's rows + column sums over its rows (the mirrored upper triangle),
//      exchanged through shared memory and summed in rank order for each owned row; v^T A v from
//      the CTA's own rows (= sum_r v_r (2 rowsum_r - A_rr v_r));
//   3  w = tau y - (tau^2/2)(v^T A v) v all-gathered;  A22 -= v w^T + w v^T on the own rows.
// Outputs as the panel kernel's: d, e, tau (fp64) and the reflectors in Vb (v_k[k+1] = 1).
constexpr int kSmThreads = 512;
constexpr int kSmMaxCl = 16;
constexpr int kSmMaxJobs = 64;
constexpr size_t kSmSmemCap = 225 * 1024;

struct SmallSet {
    const TrdJob *jobs;
    int count;
    int job[kSmMaxJobs];
};

// local lower-triangle storage of CTA `rank` (rows r = rank + CL i): offset of local row i
__host__ __device__ inline long long sm_row_off(int i, int cl, int rank) {
    return (long long)cl * i * (i - 1) / 2 + (long long)i * (rank + 1);
}
// the same in 32-bit arithmetic (device: a CTA's triangle holds < 2^15 doubles)
__device__ __forceinline__ int sm_off(int i, int cl, int rank) { return (cl * i * (i - 1) >> 1) + i * (rank + 1); }
__host__ __device__ inline int sm_rows(int n, int cl, int rank) { return rank < n ? (n - rank + cl - 1) / cl : 0; }
// largest local triangle over the cluster's CTAs (doubles): every CTA uses the same layout
__host__ __device__ inline long long sm_tri_max(int n, int cl) {
    long long m = 0;
    for (int r = 0; r < cl; ++r) {
        const long long t = sm_row_off(sm_rows(n, cl, r), cl, r);
        m = t > m ? t : m;
    }
    return m;
}
constexpr int kSmBlk = 32;              // columns of outputs buffered in shared memory per flush
// dynamic shared memory of one CTA: triangle | x/v (2 buffers) | w | column sums | row sums | slots |
// output buffers (the own rows' reflector entries and d, e, tau of kSmBlk columns)
__host__ __device__ inline size_t sm_smem_bytes(int n, int cl) {
    const size_t nl0 = (size_t)sm_rows(n, cl, 0);
    return sizeof(double) * ((size_t)sm_tri_max(n, cl) + 4 * (size_t)n + nl0 + 64 + (kSmBlk * nl0 + 1) / 2 +
                             3 * kSmBlk);
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the small reduction's barrier: a CTA barrier when the cluster is one CTA (cl is uniform)
__device__ __forceinline__ void sm_sync(int cl) {
    if (cl == 1) __syncthreads();
    else cluster_sync_all();
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_nctas() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
// shared-memory address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(const void *p, uint32_t rank) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster(uint32_t addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_cluster(uint32_t addr) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}

// Block sum with the warp partials combined by shuffles in every warp (a fixed tree: every thread,
// and every CTA of the cluster, gets the same bits) instead of a serial pass over shared memory.
__device__ __forceinline__ double sm_block_sum(double v, double *sh) {
    constexpr int kW = kSmThreads / 32;
    static_assert(kW <= 32 && (kW & (kW - 1)) == 0, "warps per CTA");
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = lane < kW ? sh[lane] : 0.0;
    // butterfly over all 32 lanes (a pairwise sum is commutative, so partners hold the same bits and
    // every lane ends with the same total; a 16-lane butterfly left lanes 16..31 with 0)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

__global__ void __launch_bounds__(kSmThreads, 1) trd_small(const __grid_constant__ SmallSet S) {
    extern __shared__ __align__(16) double smd[];
    __shared__ double sh[kSmThreads / 32];
    const int cl = (int)cluster_nctas(), rank = (int)cluster_rank();
    const TrdJob &J = S.jobs[S.job[blockIdx.x / cl]];
    const int n = J.n, ldw = J.ldw;
    const int t = threadIdx.x, lane = t % 32, warp = t / 32, nwarp = kSmThreads / 32;
    const int nl = sm_rows(n, cl, rank);
    double *Al = smd;                                            // local lower triangle
    double *xv = Al + sm_tri_max(n, cl);                         // [2][n]: x, then v (by column parity)
    double *wv = xv + 2 * n;                                     // [n]: w
    double *cs = wv + n;                                         // [n]: column sums over own rows
    double *rs = cs + n;                                         // [nl]: row sums of own rows
    const int nl0 = sm_rows(n, cl, 0);
    double *slot = rs + nl0;                                     // [0]: partial v^T A v (same offset in
                                                                 // every CTA: read through the cluster)
    // outputs are buffered for kSmBlk columns and written together: a global store outstanding at a
    // cluster barrier's release would make that barrier wait for it
    float *vbuf = reinterpret_cast<float *>(slot + 64);          // [kSmBlk][nl0] own rows' v entries
    double *dbuf = slot + 64 + (kSmBlk * nl0 + 1) / 2;           // [3][kSmBlk]: d, e, tau
    auto flush = [&](int k0, int nb) {                           // columns k0 .. k0 + nb - 1
        __syncthreads();
        const int ib = (k0 + 1 - rank + cl - 1) / cl;
        for (int e = t; e < (nl - ib) * nb; e += kSmThreads) {
            const int i = ib + e / nb, j = e % nb;
            J.Vb[(size_t)(rank + cl * i) * ldw + k0 + j] = vbuf[j * nl0 + i];   // rows <= k0 + j: masked
        }
        for (int j = t; j < nb; j += kSmThreads) {
            if ((k0 + j) % cl == rank) J.d[k0 + j] = dbuf[j];
            if (rank == 0) {
                J.e[k0 + j] = dbuf[kSmBlk + j];
                J.tau[k0 + j] = dbuf[2 * kSmBlk + j];
            }
        }
    };
    // A = (F + F^T)/2 in fp64, own rows
    for (int i = warp; i < nl; i += nwarp) {
        const int r = rank + cl * i;
        double *row = Al + sm_off(i, cl, rank);
        for (int c = lane; c <= r; c += 32)
            row[c] = 0.5 * ((double)J.F[(size_t)r * J.ldF + c] + (double)J.F[(size_t)c * J.ldF + r]);
    }
    sm_sync(cl);
    for (int k = 0; k < n - 1; ++k) {
        double *x = xv + (k & 1) * n;
        const int jb = k % kSmBlk;
        // ---- 1: all-gather x = A[k+1:n, k]; d_k from row k's owner ----
        const int i0 = (k + 1 - rank + cl - 1) / cl;             // first own row >= k+1
        for (int i = i0 + t; i < nl; i += kSmThreads) {
            const int r = rank + cl * i;
            const double a = Al[sm_off(i, cl, rank) + k];
            for (int q = 0; q < cl; ++q) st_cluster(map_rank(x + r, q), a);
        }
        if (t == 0 && k % cl == rank) dbuf[jb] = Al[sm_off(k / cl, cl, rank) + k];
        sm_sync(cl);
        // ---- reflector (dlarfg), the same in every CTA ----
        double q2 = 0.0;
        for (int r = k + 2 + t; r < n; r += kSmThreads) q2 += x[r] * x[r];
        const double alpha = x[k + 1];                           // read before the block sum's barriers,
        const double nrm2 = sm_block_sum(q2, sh);                // which order it before x[k+1] = 1
        double tau = 0.0, beta = alpha, scale = 0.0;
        if (nrm2 > 0.0) {
            beta = -copysign(sqrt(alpha * alpha + nrm2), alpha);
            tau = (beta - alpha) / beta;
            scale = 1.0 / (alpha - beta);
        }
        if (rank == 0 && t == 0) {
            dbuf[kSmBlk + jb] = beta;
            dbuf[2 * kSmBlk + jb] = tau;
        }
        for (int r = k + 1 + t; r < n; r += kSmThreads) x[r] = r == k + 1 ? 1.0 : x[r] * scale;
        __syncthreads();
        for (int i = i0 + t; i < nl; i += kSmThreads) vbuf[jb * nl0 + i] = (float)x[rank + cl * i];
        if (jb == kSmBlk - 1 || k == n - 2) flush(k - jb, jb + 1);
        if (tau == 0.0) continue;                                // H_k = I (the same in every CTA)
        const double *v = x;
        // ---- 2: y = A22 v.  Row sums (warp per own row) ----
#ifndef KFAC_SM_NOWORK                                           // diagnostic: skip the matrix passes
#define KFAC_SM_NOWORK 0
#endif
        for (int i = i0 + warp; i < (KFAC_SM_NOWORK ? 0 : nl); i += nwarp) {
            const int r = rank + cl * i;
            const double *row = Al + sm_off(i, cl, rank);
            double a = 0.0, a2 = 0.0;
            int c = k + 1 + lane;
            for (; c + 32 <= r; c += 64) {
                a += row[c] * v[c];
                a2 += row[c + 32] * v[c + 32];
            }
            if (c <= r) a += row[c] * v[c];
            a += a2;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (lane == 0) rs[i] = a;
        }
        // column sums over own rows below the diagonal (thread per column)
        for (int c = k + 1 + t; c < (KFAC_SM_NOWORK ? 0 : n); c += kSmThreads) {
            double a = 0.0;
            int i = max(i0, (c + 1 - rank + cl - 1) / cl);
            int o = sm_off(i, cl, rank) + c, r = rank + cl * i;
            double a2 = 0.0;                                     // two chains (fixed order: even/odd rows)
            for (; i + 1 < nl; i += 2) {                         // row i + 1 starts r + 1 doubles later
                a += Al[o] * v[r];
                o += r + 1;
                a2 += Al[o] * v[r + cl];
                o += r + cl + 1;
                r += 2 * cl;
            }
            if (i < nl) a += Al[o] * v[r];
            a += a2;
            cs[c] = a;
        }
        __syncthreads();
        double pv = 0.0;                                         // v^T A v over own rows
        for (int i = i0 + t; i < nl; i += kSmThreads) {
            const int r = rank + cl * i;
            pv += v[r] * (2.0 * rs[i] - Al[sm_off(i, cl, rank) + r] * v[r]);
        }
        pv = sm_block_sum(pv, sh);
        if (t == 0) slot[0] = pv;
        sm_sync(cl);
        // ---- 3: w = tau y - (tau^2 / 2)(v^T A v) v on own rows, all-gathered ----
        // remote loads issued together, then summed in rank order (bit-identical in every CTA)
        double rp[kSmMaxCl];
#pragma unroll
        for (int q = 0; q < kSmMaxCl; ++q) rp[q] = q < cl ? ld_cluster(map_rank(slot, q)) : 0.0;
        double vav = 0.0;
#pragma unroll
        for (int q = 0; q < kSmMaxCl; ++q) vav += rp[q];
        const double alpha2 = -0.5 * tau * tau * vav;
        for (int i = i0 + t; i < nl; i += kSmThreads) {
            const int r = rank + cl * i;
#pragma unroll
            for (int q = 0; q < kSmMaxCl; ++q) rp[q] = q < cl ? ld_cluster(map_rank(cs + r, q)) : 0.0;
            double y = rs[i];
#pragma unroll
            for (int q = 0; q < kSmMaxCl; ++q) y += rp[q];
            const double w = tau * y + alpha2 * v[r];
            for (int q = 0; q < cl; ++q) st_cluster(map_rank(wv + r, q), w);
        }
        sm_sync(cl);
        // A22 -= v w^T + w v^T, own rows
        for (int i = i0 + warp; i < (KFAC_SM_NOWORK ? 0 : nl); i += nwarp) {
            const int r = rank + cl * i;
            double *row = Al + sm_off(i, cl, rank);
            const double vr = v[r], wr = wv[r];
#pragma unroll 2
            for (int c = k + 1 + lane; c <= r; c += 32) row[c] -= vr * wv[c] + wr * v[c];
        }
        __syncthreads();
    }
    if (t == 0 && (n - 1) % cl == rank) J.d[n - 1] = Al[sm_off((n - 1) / cl, cl, rank) + n - 1];
    sm_sync(cl);                                                 // no CTA exits while others read it
}

// ------------------------------------------------------------ init --
// A = (F + F^T)/2 in fp32 (pads zero), Vb = 0.
__global__ void trd_init(const TrdJob *jobs) {
    // 32 x 32 tiles (grid-stride over the tile grid of the factor): F's tile and its transposed
    // partner are both read row-wise (coalesced) through shared memory.
    __shared__ float tr[32][33];
    const TrdJob &J = jobs[blockIdx.y];
    const int n = J.n, ldw = J.ldw;
    const int tn = (ldw + 31) / 32, tiles = tn * tn;
    // two-stage factors: stage 1 writes tau only for the columns of its panels (0 .. 16 num_panels
    // - 1); the back-transformation walks reflectors 0 .. n - 2, so the rest are identities (tau = 0)
    // -- never workspace left over from an earlier call (tests/test_gpu_ws_poison.py)
    if (J.off != 1 && blockIdx.x == 0)
        for (int c = threadIdx.x; c < n; c += blockDim.x) J.tau[c] = 0.0;
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;      // 32 x 8 threads
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int r0 = (tile / tn) * 32, c0 = (tile % tn) * 32;
        __syncthreads();
        for (int y = ty; y < 32; y += 8) {          // F[c0 + y][r0 + tx] -> tr[y][tx]
            const int rr = c0 + y, cc = r0 + tx;
            tr[y][tx] = (rr < n && cc < n) ? J.F[(size_t)rr * J.ldF + cc] : 0.f;
        }
        __syncthreads();
        for (int y = ty; y < 32; y += 8) {
            const int r = r0 + y, c = c0 + tx;
            if (r >= n || c >= ldw) continue;
            if (J.off != 1) {                       // two-stage: fp64 working matrix, Vd = 0
                double a = 0.0;
                if (c < n) a = 0.5 * ((double)J.F[(size_t)r * J.ldF + c] + (double)tr[tx][y]);
                J.Ad[(size_t)r * ldw + c] = a;
                J.Vd[(size_t)r * ldw + c] = 0.0;
                continue;
            }
            float a = 0.f;
            if (c < n) a = 0.5f * (J.F[(size_t)r * J.ldF + c] + tr[tx][y]);
            J.A[(size_t)r * ldw + c] = a;             // (Vb above the reflectors is masked when read)
        }
    }
}

// ----------------------------------------------------- panel kernel --
#ifndef KFAC_TRD_TIMING
#define KFAC_TRD_TIMING 0
#endif
#if KFAC_TRD_TIMING
// Diagnostic build only (-DKFAC_TRD_TIMING=1): clock64 stamps of the phases of every column, taken
// by thread 0 of three CTAs (first, middle, last) of group 0; read with kfac_debug_trd_timing.
constexpr int kTimCols = 8192, kTimPts = 10;
__device__ unsigned long long g_trd_tim[3][kTimCols][kTimPts];
#define TRD_TS(col, pt)                                                              \
    do {                                                                             \
        if (tim_slot >= 0 && (col) < kTimCols) g_trd_tim[tim_slot][col][pt] = clock64(); \
    } while (0)
#else
#define TRD_TS(col, pt) \
    do {                \
    } while (0)
#endif

struct PanelLaunch {
    const TrdJob *jobs;
    int count;
    int job[kMaxGroupCtas];
    int p0[kMaxGroupCtas];                 // panel start of each group's factor (staggered)
    int cta_begin[kMaxGroupCtas + 1];
    int ring_off;                          // float offset of the symv prefetch ring in dynamic smem
    int use_xs;                            // x of the merged column kept in shared memory
};

// One panel of 32 columns (LAPACK dlatrd, lower) for every active factor.  Column k (i = k - p0):
//   A: c = A_p[k:n, k] - V[k:n, <i] W[k, <i]^T - W[k:n, <i] V[k, <i]^T;  d_k = c_k, x = c_{k+1:n}
//   B: reflector (dlarfg) of x: beta = -sign(x_0)||x||, tau = (beta - x_0)/beta, v = x/(x_0 - beta), v_0 = 1;
//      y = A_p[k+1:n, k+1:n] v  (A_p: matrix at the panel start), partial V^T v, W^T v
//   C: y -= W (V^T v) + V (W^T v);  w = tau y;  partial w^T v
//   D: W[:, i] = w - (tau/2)(w^T v) v
// so that after the panel A_p[q:n, q:n] - V W^T - W V^T is the reduced trailing matrix (q = p0+32).
template <int SYMV_ROWS>
__global__ void __launch_bounds__(kTrdThreads, kTrdCtasPerSm) trd_panel(const __grid_constant__ PanelLaunch L) {
    // the symv unit geometry of this instantiation (shadows the namespace defaults)
    constexpr int kSymvR = SYMV_ROWS;
    constexpr int kPairR = 2 * kSymvR;
    constexpr int kMaxRb = (16384 / kPairR + 31) / 32 * 32;
    extern __shared__ __align__(16) float vsm[];     // v, 4-aligned, zero padded
    __shared__ double sh[kTrdWarps];
    __shared__ double red[kTrdWarps][2 * kNb];
    __shared__ double ab[2 * kNb];                   // (V^T v, W^T v)
    __shared__ float rowV[kNb], rowW[kNb];           // V[k, <i], W[k, <i]
    __shared__ double scal[8];
    __shared__ int tpre[kMaxRb + 1];                 // symv unit prefix per 64-row super block
    __shared__ __align__(16) double pairbuf[(kTrdWarps / 2) * 2 * 2 * 32 * 2];   // pair column sums

    int g = 0;
    {
        int lo = 0, hi = L.count - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (L.cta_begin[mid] <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
        }
        g = lo;
    }
    const TrdJob &J = L.jobs[L.job[g]];
    const int c = blockIdx.x - L.cta_begin[g], nc = L.cta_begin[g + 1] - L.cta_begin[g];
    const int n = J.n, ldw = J.ldw, p0 = L.p0[g];
    const float *A = J.A;
    float *VW = J.VW, *WV = J.WV;
    double *part = J.part;
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    const int ring_off = L.ring_off;                 // floats: symv prefetch ring after v
    // x of the merged column (phase B), after the ring: 16-byte aligned doubles
    double *xs = reinterpret_cast<double *>(vsm + ring_off + kTrdWarps * 2 * 8 * 32 * 4);
    unsigned target = 0;
#if KFAC_TRD_TIMING
    const int tim_slot = (g != 0 || t != 0) ? -1 : c == 0 ? 0 : c == nc / 2 ? 1 : c == nc - 1 ? 2 : -1;
#endif
    float w_next = 0.f;                              // W[k, i-1], computed redundantly
    // Column k's phase A (its corrected column and diagonal) is folded into column k-1's phase C
    // whenever both lie in the same panel: there every row's c_r = f_r - v_r beta with f_r known
    // before the barrier and beta = w_k + 2 alpha after it (see phase C); ||x||^2 is then summed
    // by every CTA from the full x in phase B.  Columns 1..31 of a panel need two group barriers
    // instead of three.
    bool merged = false;
    double m_beta = 0.0;                             // beta of the merged column

    for (int i = 0; i < kNb; ++i) {
        const int k = p0 + i;
        if (k >= n) break;
        int lo, hi;
        TRD_TS(k, 0);
        // ---------------- phase A (rows [k, n)) ----------------
        if (!merged) {
        if (t < i) {
            rowV[t] = ldcg(VW + (size_t)k * 64 + t);
            rowW[t] = (t == i - 1) ? w_next : ldcg(VW + (size_t)k * 64 + kNb + t);
        }
        __syncthreads();
        part_range(k, n, c, nc, lo, hi);
        double s2 = 0.0;
        const int sub = lane >> 3, sl = lane & 7;          // 8 lanes per row, 4 rows per warp
        for (int r0 = lo + 4 * warp; r0 < hi; r0 += 4 * kTrdWarps) {
            // lane sl covers panel columns q = 4 sl .. 4 sl + 3 (< i) with one float4 of V and of W
            const int r = r0 + sub;
            double corr = 0.0;
            if (r < hi && 4 * sl < i) {
                const float4 vv = __ldcg(reinterpret_cast<const float4 *>(VW + (size_t)r * 64) + sl);
                const float4 ww = __ldcg(reinterpret_cast<const float4 *>(VW + (size_t)r * 64 + kNb) + sl);
                const float v4[4] = {vv.x, vv.y, vv.z, vv.w}, w4[4] = {ww.x, ww.y, ww.z, ww.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (4 * sl + u < i) corr += (double)v4[u] * rowW[4 * sl + u] + (double)w4[u] * rowV[4 * sl + u];
            }
            corr += __shfl_xor_sync(0xffffffffu, corr, 4);
            corr += __shfl_xor_sync(0xffffffffu, corr, 2);
            corr += __shfl_xor_sync(0xffffffffu, corr, 1);
            if (sl == 0 && r < hi) {
                const double cv = (double)A[(size_t)r * ldw + k] - corr;   // column k (lower triangle kept)
                if (r == k) J.d[k] = cv;
                else __stcg(J.x + r, cv);
                if (r >= k + 2) s2 += cv * cv;
            }
        }
        s2 = block_sum(s2, sh);
        if (t == 0) __stcg(part + (size_t)c * kPart + 2 * kNb, s2);
        group_barrier(J.bar, target, nc);
        }   // !merged
        TRD_TS(k, 1);
        if (k == n - 1) break;
        // ---------------- phase B (rows [k+1, n)) ----------------
        // x_r = J.x[r] (phase A), or f_r - v'_r beta with v' = V[:, i-1] (merged)
        // (with xs in shared memory, v' is still the previous column's v in vsm: no strided load)
        const int c0p = k & ~3;                      // previous column's v offset
        auto xval = [&](int r) -> double {
            if (!merged) return ldcg(J.x + r);
            const double vp = L.use_xs ? (double)vsm[r - c0p] : (double)ldcg(VW + (size_t)r * 64 + (i - 1));
            return ldcg(J.x + r) - m_beta * vp;
        };
        double m_nrm2 = 0.0;
        const double alpha_pre = warp == 0 ? xval(k + 1) : 0.0;      // issued before the q2 pass
        if (merged) {
            // ||x||^2 over rows k+2.. computed by every CTA from the full x (the same loads and the
            // same fixed-order reduction in every CTA, so all CTAs agree bit for bit); 8 loads in
            // flight per thread
            double q2 = 0.0;
            for (int r0 = k + 2 + t; r0 < n; r0 += 8 * kTrdThreads) {
                double fx[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) fx[u] = r0 + u * kTrdThreads < n ? ldcg(J.x + r0 + u * kTrdThreads) : 0.0;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int r = r0 + u * kTrdThreads;
                    if (r < n) {
                        const double vp = L.use_xs ? (double)vsm[r - c0p] : (double)ldcg(VW + (size_t)r * 64 + (i - 1));
                        const double xr = fx[u] - m_beta * vp;
                        if (L.use_xs) xs[r - (k + 2)] = xr;   // kept for the v fill below (no second load)
                        q2 += xr * xr;
                    }
                }
            }
            m_nrm2 = block_sum(q2, sh);
        }
        if (warp == 0) {
            const double nrm2 = merged ? m_nrm2 : warp_part_sum(part, 2 * kNb, nc, lane);
            const double alpha = alpha_pre;
            double tau = 0.0, beta = alpha, scale = 0.0;
            if (nrm2 > 0.0) {
                beta = -copysign(sqrt(alpha * alpha + nrm2), alpha);
                tau = (beta - alpha) / beta;
                scale = 1.0 / (alpha - beta);
            }
            if (lane == 0) {
                scal[0] = tau;
                scal[1] = scale;
                if (c == 0) {
                    J.e[k] = beta;
                    J.tau[k] = tau;
                }
            }
        }
        __syncthreads();
        TRD_TS(k, 2);
        const double tau = scal[0], scale = scal[1];
        const int c0 = (k + 1) & ~3;
        const int nvp = (n - c0 + kSymvC - 1) / kSymvC * kSymvC;   // v padded to whole column chunks
#pragma unroll 4
        for (int j = t; j < nvp; j += kTrdThreads) {
            const int col = c0 + j;
            float v = 0.f;
            if (col == k + 1) v = 1.f;
            else if (col > k + 1 && col < n) v = (float)((merged && L.use_xs ? xs[col - (k + 2)] : xval(col)) * scale);
            vsm[j] = v;
        }
        if (warp == 0) {
            // tile prefix of the symv: tpre[b] = number of 64 x 128 lower-triangle tiles in row
            // blocks < b (block b spans chunks c0 .. its last row), for the warps' tile cursors
            // (units: 64-row super blocks x 128-column chunks, each shared by a warp pair)
            const int r00 = k + 1, nrb = (n - r00 + kPairR - 1) / kPairR;
            int loc[kMaxRb / 32], run = 0;
#pragma unroll
            for (int u = 0; u < kMaxRb / 32; ++u) {
                const int b = lane * (kMaxRb / 32) + u;
                run += b < nrb ? (min(n, r00 + kPairR * (b + 1)) - 1 - c0) / kSymvC + 1 : 0;
                loc[u] = run;
            }
            int incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int excl = incl - run;
#pragma unroll
            for (int u = 0; u < kMaxRb / 32; ++u) {
                const int b = lane * (kMaxRb / 32) + u;
                if (b < nrb) tpre[b + 1] = excl + loc[u];
            }
            if (lane == 0) tpre[0] = 0;
        }
        __syncthreads();
        part_range(k + 1, n, c, nc, lo, hi);
        for (int r = lo + t; r < hi; r += kTrdThreads) {
            const float v = vsm[r - c0];
            J.Vb[(size_t)r * ldw + k] = v;
            VW[(size_t)r * 64 + i] = v;
            WV[(size_t)r * 64 + kNb + i] = v;
            J.VWd[(size_t)r * 64 + i] = v;
            J.WVd[(size_t)r * 64 + kNb + i] = v;
        }
        double pa, pb;
        TRD_TS(k, 3);
        // symmetric mat-vec over the lower triangle of A_p[k+1:n, k+1:n] in 64 x 128 tiles (one warp
        // per tile, every tile of the group's factor spread over its warps): each tile adds its
        // row sums to DP[row][chunk] and its column sums (the mirrored upper triangle) to
        // TP[column][block]; phase C sums both in a fixed order, so every element is read once.
        // The warp walks its tiles as a stream of 8-row octets; every lane prefetches its own
        // 16-byte chunk of the next octet with cp.async into a private two-stage ring (zero fill
        // above the diagonal and past the last row), so the loads of octet q+1 are in flight while
        // octet q is reduced.
        {
            const int r00 = k + 1, nrb = (n - r00 + kPairR - 1) / kPairR;
            const int total = tpre[nrb];
            const int W = nc * (kTrdWarps / 2);      // warp pairs of the group
            const int half = warp & 1, pair = warp >> 1;
            const float4 *v4 = reinterpret_cast<const float4 *>(vsm);
            float4 *ring = reinterpret_cast<float4 *>(vsm + ring_off) + (size_t)warp * (2 * 8 * 32) + lane;
            // octet cursor: unit it (64-row super block bq, chunk jq); this warp's 32-row half starts
            // at hs and every unit yields at least one (possibly fully masked) octet, so both warps of
            // a pair meet at the same per-unit combine
            int it = c * (kTrdWarps / 2) + pair, bq = 0, base = 0, jq = 0, rq = 0;
            auto locate = [&]() {                    // last super block with tpre[bq] <= it
                int lo2 = bq, hi2 = nrb - 1;
                while (lo2 < hi2) {
                    const int mid = (lo2 + hi2 + 1) >> 1;
                    if (tpre[mid] <= it) lo2 = mid; else hi2 = mid - 1;
                }
                bq = lo2;
                base = tpre[bq];
                jq = it - base;
                rq = r00 + kPairR * bq + kSymvR * half;
            };
            auto issue = [&](int stage) {
                const int rend = min(n, r00 + kPairR * bq + kSymvR * (half + 1));
                const int ccq = c0 + kSymvC * jq + 4 * lane;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int rr = rq + u;
                    const bool ok = rr < rend && ccq <= rr;
                    const float *src = ok ? A + (size_t)rr * ldw + ccq : A;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                                     (uint32_t)__cvta_generic_to_shared(ring + (stage * 8 + u) * 32)),
                                 "l"(src), "r"(ok ? 16u : 0u)
                                 : "memory");
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
            if (it < total) {
                locate();
                issue(0);
            }
            // panel dot partials over the owned rows (lane q -> panel column q), loads in flight
            // together with the first symv octet
            pa = 0.0;
            pb = 0.0;
            if (lane < i)
#pragma unroll 4
                for (int r = lo + warp; r < hi; r += kTrdWarps) {
                    const double vr = vsm[r - c0];
                    pa += (double)ldcg(VW + (size_t)r * 64 + lane) * vr;
                    pb += (double)ldcg(VW + (size_t)r * 64 + kNb + lane) * vr;
                }

            int stage = 0;
            double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
            double2 *pslot = reinterpret_cast<double2 *>(pairbuf) + (size_t)pair * (2 * 2 * 32);
            int unit_parity = 0;
            while (it < total) {
                // current octet
                const int b = bq, j = jq, r = rq;
                const int r0 = r00 + kPairR * b + kSymvR * half, r1 = min(n, r0 + kSymvR);
                const int cc = c0 + kSymvC * j + 4 * lane;
                // advance the cursor (a unit ends after the half's last octet, or after its single
                // masked octet when the half is empty) and prefetch the next octet
                rq += 8;
                const bool unit_end = rq >= r1;
                if (unit_end) {
                    it += W;
                    if (it < total) locate();
                }
                const bool more = it < total;
                if (more) {
                    issue(stage ^ 1);
                    asm volatile("cp.async.wait_group 1;" ::: "memory");
                } else {
                    asm volatile("cp.async.wait_group 0;" ::: "memory");
                }
                const float4 v = v4[(cc - c0) >> 2];
                float4 a[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) a[u] = ring[(stage * 8 + u) * 32];
                stage ^= 1;
                double p[8];
#if KFAC_SYMV_FP32
                // fp32 products and short fp32 partial sums (4 columns / 8 rows), fp64 beyond
                float tf0 = 0.f, tf1 = 0.f, tf2 = 0.f, tf3 = 0.f;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int rr = r + u;
                    const float ax = cc <= rr ? a[u].x : 0.f, ay = cc + 1 <= rr ? a[u].y : 0.f;
                    const float az = cc + 2 <= rr ? a[u].z : 0.f, aw = cc + 3 <= rr ? a[u].w : 0.f;
                    p[u] = (double)fmaf(ax, v.x, fmaf(ay, v.y, fmaf(az, v.z, aw * v.w)));
                    const float vr = rr < r1 ? vsm[rr - c0] : 0.f;
                    tf0 = fmaf(cc < rr ? ax : 0.f, vr, tf0);
                    tf1 = fmaf(cc + 1 < rr ? ay : 0.f, vr, tf1);
                    tf2 = fmaf(cc + 2 < rr ? az : 0.f, vr, tf2);
                    tf3 = fmaf(cc + 3 < rr ? aw : 0.f, vr, tf3);
                }
                t0 += (double)tf0;
                t1 += (double)tf1;
                t2 += (double)tf2;
                t3 += (double)tf3;
#else
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int rr = r + u;
                    const double ax = cc <= rr ? a[u].x : 0.0, ay = cc + 1 <= rr ? a[u].y : 0.0;
                    const double az = cc + 2 <= rr ? a[u].z : 0.0, aw = cc + 3 <= rr ? a[u].w : 0.0;
                    p[u] = ax * v.x + ay * v.y + az * v.z + aw * v.w;
                    const double vr = rr < r1 ? (double)vsm[rr - c0] : 0.0;
                    t0 += (cc < rr ? ax : 0.0) * vr;
                    t1 += (cc + 1 < rr ? ay : 0.0) * vr;
                    t2 += (cc + 2 < rr ? az : 0.0) * vr;
                    t3 += (cc + 3 < rr ? aw : 0.0) * vr;
                }
#endif
                // butterfly reduce-scatter of the 8 row partials (9 shuffles instead of 40)
                const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
                double q4[4], q2[2];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const double send = h16 ? p[u] : p[u + 4], keep = h16 ? p[u + 4] : p[u];
                    q4[u] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const double send = h8 ? q4[u] : q4[u + 2], keep = h8 ? q4[u + 2] : q4[u];
                    q2[u] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
                }
                double sd = (h4 ? q2[1] : q2[0]) + __shfl_xor_sync(0xffffffffu, h4 ? q2[0] : q2[1], 4);
                sd += __shfl_xor_sync(0xffffffffu, sd, 2);
                sd += __shfl_xor_sync(0xffffffffu, sd, 1);
                const int rs = r + (h16 ? 4 : 0) + (h8 ? 2 : 0) + (h4 ? 1 : 0);
                if ((lane & 3) == 0 && rs < r1) __stcg(J.DP + (size_t)rs * J.ldp + j, sd);
                if (unit_end) {                      // unit done: the pair's column sums
                    double2 *sl = pslot + unit_parity * (2 * 32);
                    if (half == 1) {
                        sl[lane] = make_double2(t0, t1);
                        sl[32 + lane] = make_double2(t2, t3);
                    }
                    asm volatile("bar.sync %0, 64;" ::"r"(1 + pair) : "memory");
                    if (half == 0) {
                        const double2 u01 = sl[lane], u23 = sl[32 + lane];
                        if (cc < n) __stcg(J.TP + (size_t)cc * J.ldtp + b, t0 + u01.x);
                        if (cc + 1 < n) __stcg(J.TP + (size_t)(cc + 1) * J.ldtp + b, t1 + u01.y);
                        if (cc + 2 < n) __stcg(J.TP + (size_t)(cc + 2) * J.ldtp + b, t2 + u23.x);
                        if (cc + 3 < n) __stcg(J.TP + (size_t)(cc + 3) * J.ldtp + b, t3 + u23.y);
                    }
                    unit_parity ^= 1;                // the other slot is free: its reader passed
                    t0 = t1 = t2 = t3 = 0.0;         // the barrier of the previous unit already
                }
            }
        }
        TRD_TS(k, 4);
        red[warp][lane] = pa;
        red[warp][kNb + lane] = pb;
        __syncthreads();
        if (t < 2 * kNb) {
            double s = 0.0;
            for (int w = 0; w < kTrdWarps; ++w) s += red[w][t];
            __stcg(part + (size_t)c * kPart + t, s);
        }
        TRD_TS(k, 5);
        group_barrier(J.bar, target, nc);
        TRD_TS(k, 6);
        // ---------------- phase C ----------------
        {   // (V^T v, W^T v): kTpc consecutive threads per panel column sum the group's CTA partials
            constexpr int kTpc = kTrdThreads / (2 * kNb);
            const int col = t / kTpc, sub = t % kTpc;
            double sum = 0.0;
            if ((col % kNb) < i)
                for (int q0 = sub; q0 < nc; q0 += 8 * kTpc) {     // 8 loads in flight, same order
                    double pv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        pv[u] = q0 + kTpc * u < nc ? ldcg(part + (size_t)(q0 + kTpc * u) * kPart + col) : 0.0;
#pragma unroll
                    for (int u = 0; u < 8; ++u) sum += pv[u];
                }
#pragma unroll
            for (int o = kTpc / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            if (sub == 0) ab[col] = sum;
        }
        // merge column k+1's phase A into this phase C (same panel, same row ownership)
        const bool mnext = (i + 1 < kNb) && (k + 1 < n);
        if (mnext && t < i) {          // V[k+1, q], W[k+1, q] (q < i: final since earlier barriers)
            rowV[t] = ldcg(VW + (size_t)(k + 1) * 64 + t);
            rowW[t] = ldcg(VW + (size_t)(k + 1) * 64 + kNb + t);
        }
        __syncthreads();
        double wv = 0.0;
        {
            const int nrb = (n - (k + 1) + kPairR - 1) / kPairR;
            const int sub = lane >> 3, sl = lane & 7;      // 8 lanes per row, 4 rows per warp
            for (int r0 = lo + 4 * warp; r0 < hi; r0 += 4 * kTrdWarps) {
                const int r = r0 + sub;
                double yr = 0.0, corr = 0.0;
                float a_next = 0.f;                        // A_p[r, k+1] for the merged column
                if (r < hi) {
                    const int b = (r - (k + 1)) / kPairR;          // TP: 64-row super blocks
                    const int nj = (min(n, k + 1 + kSymvR * ((r - (k + 1)) / kSymvR + 1)) - 1 - c0) / kSymvC + 1;
                    const int nt = nrb - b;
                    // every load of the row issued before any is used: V/W row, A_p[r, k+1], then
                    // DP and TP partials in batches of 8 + 8 per lane (one batch for n <= 8192)
                    float4 vv = make_float4(0.f, 0.f, 0.f, 0.f), ww = vv;
                    if (4 * sl < i) {
                        vv = __ldcg(reinterpret_cast<const float4 *>(VW + (size_t)r * 64) + sl);
                        ww = __ldcg(reinterpret_cast<const float4 *>(VW + (size_t)r * 64 + kNb) + sl);
                    }
                    if (mnext && sl == 0) a_next = A[(size_t)r * ldw + k + 1];
                    const double *dp = J.DP + (size_t)r * J.ldp, *tp = J.TP + (size_t)r * J.ldtp + b;
                    double y0 = 0.0, y1 = 0.0;
                    const int ntot = max(nj, nt);
                    for (int base = sl; base < ntot; base += 64) {
                        double pd[8], pt[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) pd[u] = base + 8 * u < nj ? ldcg(dp + base + 8 * u) : 0.0;
#pragma unroll
                        for (int u = 0; u < 8; ++u) pt[u] = base + 8 * u < nt ? ldcg(tp + base + 8 * u) : 0.0;
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            y0 += pd[u];
                            y1 += pt[u];
                        }
                    }
                    yr = y0 + y1;
                    if (4 * sl < i) {
                        const float v4[4] = {vv.x, vv.y, vv.z, vv.w}, w4[4] = {ww.x, ww.y, ww.z, ww.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (4 * sl + u < i) {
                                yr -= (double)w4[u] * ab[4 * sl + u] + (double)v4[u] * ab[kNb + 4 * sl + u];
                                corr += (double)v4[u] * rowW[4 * sl + u] + (double)w4[u] * rowV[4 * sl + u];
                            }
                    }
                }
                yr += __shfl_xor_sync(0xffffffffu, yr, 4);
                yr += __shfl_xor_sync(0xffffffffu, yr, 2);
                yr += __shfl_xor_sync(0xffffffffu, yr, 1);
                if (mnext) {
                    corr += __shfl_xor_sync(0xffffffffu, corr, 4);
                    corr += __shfl_xor_sync(0xffffffffu, corr, 2);
                    corr += __shfl_xor_sync(0xffffffffu, corr, 1);
                }
                if (sl == 0 && r < hi) {
                    const double w = tau * yr;
                    const double vr = (double)vsm[r - c0];
                    __stcg(J.y + r, w);
                    if (L.use_xs) xs[r - lo] = w;           // own rows, reused in phase D
                    wv += w * vr;
                    if (mnext) {
                        // column k+1 before its last correction term:
                        //   c_r = A_p[r, k+1] - sum_{q<i} (V[r,q] W[k+1,q] + W[r,q] V[k+1,q])
                        //         - (V[r,i] W[k+1,i] + W[r,i] V[k+1,i])
                        // with V[:, i] = v (v_{k+1} = 1) and W[:, i] = w + alpha v, the last term is
                        // w_r + v_r (w_{k+1} + 2 alpha), so c_r = f_r - v_r beta:
                        __stcg(J.x + r, (double)a_next - corr - w);
                    }
                }
            }
        }
        wv = block_sum(wv, sh);
        if (t == 0) __stcg(part + (size_t)c * kPart + 2 * kNb + 1, wv);
        TRD_TS(k, 7);
        group_barrier(J.bar, target, nc);
        TRD_TS(k, 8);
        // ---------------- phase D (+ the merged phase A of column k+1) ----------------
        // w^T v: one partial per thread (a single round trip), fixed-order block reduction, so
        // every CTA of the group gets the same alpha bit for bit
        double ps = 0.0;
        for (int q = t; q < nc; q += kTrdThreads) ps += ldcg(part + (size_t)q * kPart + 2 * kNb + 1);
        const double yk1 = ldcg(J.y + k + 1);                         // in flight with the partials
        const double alpha2 = -0.5 * tau * block_sum(ps, sh);
        if (mnext) {
            m_beta = yk1 + 2.0 * alpha2;                               // w_{k+1} + 2 alpha
            if (c == 0 && t == 0) J.d[k + 1] = ldcg(J.x + k + 1) - m_beta;   // f_{k+1} - v_{k+1} beta
        }
        merged = mnext;
        for (int r = lo + t; r < hi; r += kTrdThreads) {
            const float w = (float)((L.use_xs ? xs[r - lo] : ldcg(J.y + r)) + alpha2 * (double)vsm[r - c0]);
            VW[(size_t)r * 64 + kNb + i] = w;
            WV[(size_t)r * 64 + i] = w;
            J.VWd[(size_t)r * 64 + kNb + i] = w;
            J.WVd[(size_t)r * 64 + i] = w;
        }
        w_next = (float)(yk1 + alpha2);                 // row k+1: v = 1
        __syncthreads();
        TRD_TS(k, 9);
    }
    if (p0 + kNb < n) {
        // Fused rank-64 trailing update A[q0:n, q0:n] -= V W^T + W V^T (lower 64 x 64 tiles) on the
        // fp64 tensor cores, by the same group once every CTA has written its rows of the panel:
        // two teams of 8 warps per CTA, each tile's whole K = 64 of [V|W] and [W|V] (fp64 copies)
        // staged at once in shared memory (row stride 68 doubles), 16 DMMA k-steps, fp32 RMW.
        group_barrier(J.bar, target, nc);
        const int q0 = p0 + kNb, m = n - q0, nt = (m + 63) / 64, ntiles = nt * (nt + 1) / 2;
        const int team = warp / 8, tw = warp % 8, tt = t % 256;
        double *Ts = reinterpret_cast<double *>(vsm + ring_off) + (size_t)team * (2 * 64 * 68);
        double *As = Ts, *Bs = Ts + 64 * 68;
        const uint32_t as_s = (uint32_t)__cvta_generic_to_shared(As), bs_s = (uint32_t)__cvta_generic_to_shared(Bs);
        const int wr = (tw / 2) * 16, wc = (tw % 2) * 32, g = lane >> 2, q = lane & 3;
        for (int tile = c * 2 + team; tile < ntiles; tile += nc * 2) {
            int ti = 0, rem = tile;                       // lower tiles row-major: row ti has ti + 1
            while (rem > ti) { rem -= ti + 1; ++ti; }
            const int tj = rem;
            const int r0 = q0 + ti * 64, c0t = q0 + tj * 64;
            // stage A = VWd[r0 .. r0+63, 0:64), B = WVd[c0t .. c0t+63, 0:64) (16-B chunks, zero fill)
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int ch = tt + 256 * u, row = ch / 32, k2 = (ch % 32) * 2;
                const bool oka = r0 + row < n, okb = c0t + row < n;
                const double *sa = oka ? J.VWd + (size_t)(r0 + row) * 64 + k2 : J.VWd;
                const double *sb = okb ? J.WVd + (size_t)(c0t + row) * 64 + k2 : J.WVd;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(as_s + (uint32_t)(row * 68 + k2) * 8),
                             "l"(sa), "r"(oka ? 16u : 0u) : "memory");
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(bs_s + (uint32_t)(row * 68 + k2) * 8),
                             "l"(sb), "r"(okb ? 16u : 0u) : "memory");
            }
            asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
            asm volatile("bar.sync %0, 256;" ::"r"(team + 1) : "memory");
            double acc[2][4][2];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll 4
            for (int kk = 0; kk < 64; kk += 4) {
                double fa[2], fb[4];
#pragma unroll
                for (int a = 0; a < 2; ++a) fa[a] = As[(wr + a * 8 + g) * 68 + kk + q];
#pragma unroll
                for (int b = 0; b < 4; ++b) fb[b] = Bs[(wc + b * 8 + g) * 68 + kk + q];
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                     : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
                                     : "d"(fa[a]), "d"(fb[b]));
            }
            // C (fp32 working matrix) -= acc: element (r0 + wr + 8a + g, c0t + wc + 8b + 2q + e)
            float *Aw = const_cast<float *>(A);
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const int rr = r0 + wr + a * 8 + g;
                if (rr >= n) continue;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int cc2 = c0t + wc + b * 8 + 2 * q;
                    float *cp = Aw + (size_t)rr * ldw + cc2;
                    if (cc2 + 1 < n) {
                        float2 cv = *reinterpret_cast<float2 *>(cp);
                        cv.x = (float)((double)cv.x - acc[a][b][0]);
                        cv.y = (float)((double)cv.y - acc[a][b][1]);
                        *reinterpret_cast<float2 *>(cp) = cv;
                    } else if (cc2 < n) {
                        cp[0] = (float)((double)cp[0] - acc[a][b][0]);
                    }
                }
            }
            asm volatile("bar.sync %0, 256;" ::"r"(team + 1) : "memory");   // smem reused by the next tile
        }
    }
}

// ---------------------------------------------------------- D&C: tear --
// Leaves: boundaries b_i = floor(i n / 2^L).  Each internal boundary s splits T into
// diag(T1, T2) + |rho| u u^T, u = [e_last; sign(rho) e_first] (rho = e[s-1]), so both
// adjacent diagonal entries lose |rho| (Cuppen; LAPACK dlaed0).
__global__ void dc_tear(const TrdJob *jobs) {
    const TrdJob &J = jobs[blockIdx.y];
    const int n = J.n, nleaf = 1 << J.levels;
    auto is_boundary = [&](int i) {          // i == floor(b n / nleaf) for some 1 <= b < nleaf
        if (i <= 0 || i >= n) return false;
        const long long b = ((long long)i * nleaf + n - 1) / n;
        return b >= 1 && b < nleaf && (long long)b * n / nleaf == i;
    };
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double v = J.d[i];
        if (is_boundary(i)) v -= fabs(J.e[i - 1]);
        if (is_boundary(i + 1)) v -= fabs(J.e[i]);
        J.D[i] = v;
    }
}

// ------------------------------------------------------- D&C: leaves --
struct LeafDesc {
    int job, a, size;
};

// Implicit QL with Wilkinson-type shifts (EISPACK tql2) on one leaf; every lane runs the scalar
// recurrence redundantly (identical arithmetic) and owns one row of the eigenvector matrix.
// The QL sweeps index d, e and the eigenvector row z with run-time bounds; in registers they would
// live in local (stack) memory, so every lane keeps its own copies in shared memory as [i][lane]
// (conflict-free; lanes share nothing: each runs the same recurrence on its own d, e).
constexpr int kLeafWarps = 2;                 // 3 x 8 KB per warp of static shared memory (48 KB cap)
struct LeafCol {                                      // x[i] -> buf[i][lane]
    double (*p)[32];
    int lane;
    __device__ double &operator[](int i) const { return p[i][lane]; }
};
__global__ void __launch_bounds__(kLeafWarps * 32) dc_leaf(const TrdJob *jobs, const LeafDesc *leaves, int nleaves) {
    __shared__ double sd[kLeafWarps][kLeaf][32], se[kLeafWarps][kLeaf][32], sz[kLeafWarps][kLeaf][32];
    const int li = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (li >= nleaves) return;
    const LeafDesc Ld = leaves[li];
    const TrdJob &J = jobs[Ld.job];
    const int lane = threadIdx.x % 32, ns = Ld.size, a = Ld.a, w = threadIdx.x / 32;
    const LeafCol d{sd[w], lane}, e{se[w], lane}, z{sz[w], lane};
    for (int i = 0; i < kLeaf; ++i) {
        d[i] = i < ns ? J.D[a + i] : 0.0;
        e[i] = (i + 1 < ns) ? J.e[a + i] : 0.0;       // e[i] = T[i+1][i]
        z[i] = (i == lane) ? 1.0 : 0.0;               // row `lane` of the eigenvector matrix
    }
    double f = 0.0, tst1 = 0.0;
    int iters = 0;
    for (int l = 0; l < ns; ++l) {
        tst1 = fmax(tst1, fabs(d[l]) + fabs(e[l]));
        int m = l;
        while (m < ns - 1 && fabs(e[m]) > kEps * tst1) ++m;
        if (m > l) {
            do {
                if (++iters > 60 * kLeaf) break;
                double g = d[l];
                double p = (d[l + 1] - g) / (2.0 * e[l]);
                double r = hypot(p, 1.0);
                if (p < 0) r = -r;
                d[l] = e[l] / (p + r);
                d[l + 1] = e[l] * (p + r);
                const double dl1 = d[l + 1];
                double h = g - d[l];
                for (int i = l + 2; i < ns; ++i) d[i] -= h;
                f += h;
                p = d[m];
                double c = 1.0, c2 = 1.0, c3 = 1.0, s = 0.0, s2 = 0.0;
                const double el1 = e[l + 1];
                for (int i = m - 1; i >= l; --i) {
                    c3 = c2;
                    c2 = c;
                    s2 = s;
                    g = c * e[i];
                    h = c * p;
                    r = hypot(p, e[i]);
                    e[i + 1] = s * r;
                    s = e[i] / r;
                    c = p / r;
                    p = c * d[i] - s * g;
                    d[i + 1] = h + s * (c * g + s * d[i]);
                    const double zi1 = z[i + 1];
                    z[i + 1] = s * z[i] + c * zi1;
                    z[i] = c * z[i] - s * zi1;
                }
                p = -s * s2 * c3 * el1 * e[l] / dl1;
                e[l] = s * p;
                d[l] = c * p;
            } while (fabs(e[l]) > kEps * tst1);
        }
        d[l] += f;
        e[l] = 0.0;
    }
    // ascending order: rank of each eigenvalue (ties by index)
    for (int j = 0; j < ns; ++j) {
        int rk = 0;
        for (int q = 0; q < ns; ++q) rk += (d[q] < d[j]) || (d[q] == d[j] && q < j);
        if (lane == 0) J.D[a + rk] = d[j];
        if (lane < ns) J.Z0[(size_t)(a + lane) * J.ldw + a + rk] = z[j];
    }
    if (iters > 60 * kLeaf && lane == 0 && J.info) atomicAdd(J.info, 1);
}

// ------------------------------------------------------- D&C: merges --
struct MergeDesc {
    int job, a, n1, n2, m;      // m: merge index inside the job's level (state slot = a)
};

// Sort the two halves' eigenvalues into one ascending list, form z, and deflate (LAPACK dlaed2).
// Non-deflated entries go to [0, k) of (dval, zval, col) in ascending d; deflated ones fill
// [k, n) from the back.  Rotations (p, j, c, s) act on original columns: q_p <- c q_p + s q_j,
// q_j <- c q_j - s q_p.
__global__ void dc_deflate(const TrdJob *jobs, const MergeDesc *merges, int ping, int smem_n) {
    // With smem_n >= nm the sorted (d, z, col) lists live in shared memory for the serial deflation
    // scan (dynamic smem: 2 smem_n doubles + smem_n ints); otherwise in the global scratch arrays.
    extern __shared__ double dsm[];
    const MergeDesc M = merges[blockIdx.x];
    const TrdJob &J = jobs[M.job];
    const int a = M.a, n1 = M.n1, nm = M.n1 + M.n2, ldw = J.ldw;
    const double *Z = ping ? J.Z1 : J.Z0;
    const double rho = J.e[a + n1 - 1];
    const double sgn = rho < 0 ? -1.0 : 1.0;
    const bool sm = nm <= smem_n;
    double *dv = sm ? dsm : J.dval + a, *zv = sm ? dsm + smem_n : J.zval + a;
    int *col = sm ? reinterpret_cast<int *>(dsm + 2 * (size_t)smem_n) : J.col + a;
    const double rs2 = 0.70710678118654752440;
    double dmax = 0.0, zmax = 0.0;
    for (int c = threadIdx.x; c < nm; c += blockDim.x) {
        const double dc = J.D[a + c];
        double zc;
        int rank;
        if (c < n1) {
            zc = Z[(size_t)(a + n1 - 1) * ldw + a + c];
            int lo = 0, hi = M.n2;                   // # right entries < dc
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (J.D[a + n1 + mid] < dc) lo = mid + 1; else hi = mid;
            }
            rank = c + lo;
        } else {
            zc = sgn * Z[(size_t)(a + n1) * ldw + a + c];
            int lo = 0, hi = n1;                     // # left entries <= dc
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (J.D[a + mid] <= dc) lo = mid + 1; else hi = mid;
            }
            rank = (c - n1) + lo;
        }
        zc *= rs2;
        dv[rank] = dc;
        zv[rank] = zc;
        col[rank] = c;
        dmax = fmax(dmax, fabs(dc));
        zmax = fmax(zmax, fabs(zc));
    }
    // max-reductions
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
    }
    __shared__ double shd[32], shz[32];
    __shared__ int s_k, s_ndef, s_all, s_kt1, s_kt2;
    if (threadIdx.x % 32 == 0) {
        shd[threadIdx.x / 32] = dmax;
        shz[threadIdx.x / 32] = zmax;
    }
    __syncthreads();
    double *defv = J.rtau + a;
    int *defc = J.rorg + a;
    if (threadIdx.x == 0) {
        for (int w = 0; w < (int)(blockDim.x / 32); ++w) {
            dmax = fmax(dmax, shd[w]);
            zmax = fmax(zmax, shz[w]);
        }
        const double rho2 = 2.0 * fabs(rho);
        const double tol = 8.0 * kEps * fmax(dmax, zmax);
        int *rp = J.rot_p + a, *rj = J.rot_j + a;
        double *rc = J.rot_c + a, *rsn = J.rot_s + a;
        int k = 0, nrot = 0, ndef = 0;
        int kt[4] = {0, 0, 0, 0};                    // non-deflated columns per type
        int *ctyp = J.ctyp + a;
        s_all = rho2 * zmax <= tol;
        if (!s_all) {
            // Deflated entries are accumulated in rtau/rorg scratch (value, col) and appended.
            // Column types (LAPACK dlaed2): 1 = nonzero only in the upper n1 rows, 3 = only in the
            // lower rows, 2 = mixed by a rotation; the eigenvector GEMM skips the zero blocks.
            int pj = -1;
            double dp = 0.0, zp = 0.0;
            int cp = 0, tp = 0;
            // serial scan (LAPACK dlaed2 order); the next entry is loaded before the current one is
            // processed, and the rotation test |t c s| <= tol with c = z_j / h, s = -z_p / h,
            // h^2 = z_j^2 + z_p^2, is evaluated as |t z_j z_p| <= tol h^2 (no sqrt or division unless
            // the pair is rotated; every z here exceeds tol / rho2, so h^2 does not underflow)
            double dn = nm > 0 ? dv[0] : 0.0, zn = nm > 0 ? zv[0] : 0.0;
            int cn = nm > 0 ? col[0] : 0;
            for (int j = 0; j < nm; ++j) {
                double dj = dn, zj = zn;
                const int cj = cn;
                if (j + 1 < nm) {
                    dn = dv[j + 1];
                    zn = zv[j + 1];
                    cn = col[j + 1];
                }
                if (rho2 * fabs(zj) <= tol) {
                    defv[ndef] = dj;
                    defc[ndef++] = cj;
                    continue;
                }
                const int tj = cj < n1 ? 1 : 3;
                if (pj < 0) {
                    pj = j; dp = dj; zp = zj; cp = cj; tp = tj;
                    continue;
                }
                const double t = dj - dp;
                const double hh = fma(zj, zj, zp * zp);
                if (fabs(t * zj * zp) <= tol * hh) {
                    const double tt = hypot(zj, zp);
                    const double cv = zj / tt, sv = -zp / tt;
                    // deflate p after rotating (p, j)
                    zj = tt;
                    rp[nrot] = cp; rj[nrot] = cj; rc[nrot] = cv; rsn[nrot] = sv; ++nrot;
                    const double t2 = dp * cv * cv + dj * sv * sv;
                    dj = dp * sv * sv + dj * cv * cv;
                    defv[ndef] = t2;
                    defc[ndef++] = cp;
                    tp = tp == tj ? tj : 2;          // q_j now mixes q_p in
                    pj = j; dp = dj; zp = zj; cp = cj;
                } else {
                    dv[k] = dp; zv[k] = zp; col[k] = cp; ctyp[k] = tp; ++kt[tp]; ++k;
                    pj = j; dp = dj; zp = zj; cp = cj; tp = tj;
                }
            }
            if (pj >= 0) {
                dv[k] = dp; zv[k] = zp; col[k] = cp; ctyp[k] = tp; ++kt[tp]; ++k;
            }
        }
        s_kt1 = kt[1];
        s_kt2 = kt[2];
        s_k = k;
        s_ndef = ndef;
        J.mstate[4 * a + 0] = k;
        J.mstate[4 * a + 1] = nrot;
        J.mstate[4 * a + 2] = k;                     // upper rows: N = k, K = [0, k1 + k2)
        J.mstate[4 * a + 3] = kt[1] + kt[2];
        J.mstate[4 * a + 4] = 0;
        J.mstate[4 * a + 5] = k;                     // lower rows: N = k, K = [k1, k)
        J.mstate[4 * a + 6] = k;
        J.mstate[4 * a + 7] = kt[1];
        J.mscal[2 * a + 0] = rho2;
        J.mscal[2 * a + 1] = tol;
    }
    __syncthreads();
    // everything deflated: keep the sorted order; otherwise append the deflated list after k
    const int k = s_k, ndef = s_ndef;
    if (!s_all) {
        for (int q = threadIdx.x; q < ndef; q += blockDim.x) {
            dv[k + q] = defv[q];
            col[k + q] = defc[q];
            zv[k + q] = 0.0;
        }
        __syncthreads();
    }
    int *posof = J.posof + a;
    double *gdv = J.dval + a, *gzv = J.zval + a;
    int *gcol = J.col + a;
    // GEMM position of each non-deflated column: types grouped 1 | 2 | 3, stable (block-wide
    // ballot scan over chunks of blockDim entries; ctyp is overwritten in place by its reader)
    {
        __shared__ int wcnt[32][3], run[3];
        int *gpos = J.ctyp + a;
        const int lane = threadIdx.x % 32, w = threadIdx.x / 32, nw = blockDim.x / 32;
        const int base[4] = {0, 0, s_kt1, s_kt1 + s_kt2};
        if (threadIdx.x < 3) run[threadIdx.x] = 0;
        for (int c0 = 0; c0 < k; c0 += blockDim.x) {
            __syncthreads();
            const int p = c0 + threadIdx.x;
            const int ty = p < k ? gpos[p] : 0;
            const unsigned m1 = __ballot_sync(0xffffffffu, ty == 1), m2 = __ballot_sync(0xffffffffu, ty == 2),
                           m3 = __ballot_sync(0xffffffffu, ty == 3);
            if (lane == 0) {
                wcnt[w][0] = __popc(m1);
                wcnt[w][1] = __popc(m2);
                wcnt[w][2] = __popc(m3);
            }
            __syncthreads();
            int g = 0;
            if (ty > 0) {
                const unsigned mt = ty == 1 ? m1 : ty == 2 ? m2 : m3;
                g = base[ty] + run[ty - 1] + __popc(mt & ((1u << lane) - 1u));
                for (int q = 0; q < w; ++q) g += wcnt[q][ty - 1];
            }
            __syncthreads();
            if (threadIdx.x < 3) {
                int add = 0;
                for (int q = 0; q < nw; ++q) add += wcnt[q][threadIdx.x];
                run[threadIdx.x] += add;
            }
            if (ty > 0) gpos[p] = g;
        }
        __syncthreads();
    }
    const int *gpos = J.ctyp + a;
    for (int j = threadIdx.x; j < nm; j += blockDim.x) {
        const int cj = col[j];
        posof[cj] = j < k ? gpos[j] : j;
        if (sm) {
            gdv[j] = dv[j];
            gzv[j] = zv[j];
            gcol[j] = cj;
        }
    }
}

// Qnd[a + r][posof[c]] = (block-diagonal child eigenvectors)[r][c]  (one warp per row).
__global__ void dc_permute(const TrdJob *jobs, const MergeDesc *merges, int ping) {
    const MergeDesc M = merges[blockIdx.y];
    const TrdJob &J = jobs[M.job];
    const int a = M.a, n1 = M.n1, nm = M.n1 + M.n2, ldw = J.ldw;
    const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (r >= nm) return;
    const double *Z = ping ? J.Z1 : J.Z0;
    const int *posof = J.posof + a;
    double *dst = J.Qnd + (size_t)(a + r) * ldw;
    const double *src = Z + (size_t)(a + r) * ldw + a;
    for (int c = lane; c < nm; c += 32) {
        const bool same = (c < n1) == (r < n1);
        dst[posof[c]] = same ? src[c] : 0.0;
    }
}

// Apply the merge's Givens rotations to every row of Qnd (one thread per row, in order).
__global__ void dc_rotate(const TrdJob *jobs, const MergeDesc *merges) {
    const MergeDesc M = merges[blockIdx.y];
    const TrdJob &J = jobs[M.job];
    const int a = M.a, nm = M.n1 + M.n2;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int nrot = J.mstate[4 * a + 1];
    if (r >= nm || nrot == 0) return;
    double *row = J.Qnd + (size_t)(a + r) * J.ldw;
    const int *posof = J.posof + a;
    for (int q = 0; q < nrot; ++q) {
        const int pp = posof[J.rot_p[a + q]], pj = posof[J.rot_j[a + q]];
        const double c = J.rot_c[a + q], s = J.rot_s[a + q];
        const double x = row[pp], y = row[pj];
        row[pp] = c * x + s * y;
        row[pj] = c * y - s * x;
    }
}

// Secular equation 1/rho + sum_i z_i^2 / (d_i - lambda) = 0, root j in (d_j, d_{j+1})
// (last root in (d_k, d_k + rho ||z||^2)), one warp per root.  lambda_j = d_{org} + tau with the
// origin at the nearer pole so that d_i - lambda_j = (d_i - d_org) - tau keeps full relative
// accuracy.  Iteration: two-pole rational model of psi (poles <= j) and phi (poles > j) fitted to
// value and slope at tau (fixed-weight / "middle way" family), safeguarded by the bracket.
__global__ void dc_secular(const TrdJob *jobs, const MergeDesc *merges) {
    const MergeDesc M = merges[blockIdx.y];
    const TrdJob &J = jobs[M.job];
    const int a = M.a;
    const int k = J.mstate[4 * a + 0];
    const int j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (j >= k) return;
    const double *dv = J.dval + a, *zv = J.zval + a;
    const double rho = J.mscal[2 * a + 0];
    const double rinv = 1.0 / rho;
    const bool last = (j == k - 1);
    int org;
    double lo, hi;
    if (last) {
        double zz = 0.0;
        for (int i = lane; i < k; i += 32) zz += zv[i] * zv[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) zz += __shfl_xor_sync(0xffffffffu, zz, o);
        org = j;
        lo = 0.0;
        hi = rho * zz;
    } else {
        const double del = dv[j + 1] - dv[j];
        const double mid = 0.5 * del;
        double f = 0.0;
        for (int i = lane; i < k; i += 32) f += zv[i] * zv[i] / ((dv[i] - dv[j]) - mid);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
        f += rinv;
        if (f >= 0.0) { org = j; lo = 0.0; hi = mid; }
        else { org = j + 1; lo = -mid; hi = 0.0; }
    }
    if (k == 1) {                                    // lambda = d_0 + rho z_0^2 exactly
        if (lane == 0) {
            J.rtau[a] = hi;
            J.rorg[a] = 0;
        }
        return;
    }
    const double dorg = dv[org];
    const int L = j, R = j + 1;                      // poles bounding the root (R absent if last)
    const double dL = dv[L] - dorg, dR = last ? 0.0 : dv[R] - dorg;
    double tau = 0.5 * (lo + hi);
    for (int it = 0; it < 100; ++it) {
        double psi = 0.0, dpsi = 0.0, phi = 0.0, dphi = 0.0;
        for (int i = lane; i < k; i += 32) {
            const double del = (dv[i] - dorg) - tau;
            const double tq = zv[i] / del;
            const double term = zv[i] * tq, dterm = tq * tq;
            if (i <= L) { psi += term; dpsi += dterm; }
            else { phi += term; dphi += dterm; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            psi += __shfl_xor_sync(0xffffffffu, psi, o);
            dpsi += __shfl_xor_sync(0xffffffffu, dpsi, o);
            phi += __shfl_xor_sync(0xffffffffu, phi, o);
            dphi += __shfl_xor_sync(0xffffffffu, dphi, o);
        }
        const double w = rinv + psi + phi;
        if (w > 0.0) hi = tau; else lo = tau;
        const double err = 8.0 * (phi - psi) + rinv + fabs(tau) * (dpsi + dphi);
        if (fabs(w) <= kEps * err) break;
        if (hi - lo <= 2.0 * kEps * fmax(fabs(lo), fabs(hi))) break;
        // model: c + q/(dL - x) + s/(dR - x) = 0
        const double aL = dL - tau;
        const double qL = dpsi * aL * aL;
        double cc = rinv + (psi - qL / aL);
        double tn;
        if (last) {
            cc += phi;                               // phi carries no pole term
            tn = (cc != 0.0) ? dL + qL / cc : 0.5 * (lo + hi);
            // c + q/(dL - x) = 0  ->  x = dL + q/c
        } else {
            const double aR = dR - tau;
            const double sR = dphi * aR * aR;
            cc += phi - sR / aR;
            // c (dL - x)(dR - x) + q (dR - x) + s (dL - x) = 0, quadratic in y = x - dL... solve in x:
            // c x^2 - (c (dL + dR) + q + s) x + (c dL dR + q dR + s dL) = 0
            const double B = cc * (dL + dR) + qL + sR;
            const double C = cc * dL * dR + qL * dR + sR * dL;
            double x1, x2;
            if (cc == 0.0) {
                x1 = x2 = (B != 0.0) ? C / B : 0.5 * (lo + hi);
            } else {
                const double disc = fmax(B * B - 4.0 * cc * C, 0.0);
                const double sq = sqrt(disc);
                const double qq = B >= 0 ? 0.5 * (B + sq) : 0.5 * (B - sq);
                x1 = qq / cc;
                x2 = (qq != 0.0) ? C / qq : x1;
            }
            const bool in1 = x1 > lo && x1 < hi, in2 = x2 > lo && x2 < hi;
            tn = in1 ? (in2 ? (fabs(x1 - tau) < fabs(x2 - tau) ? x1 : x2) : x1) : (in2 ? x2 : 0.5 * (lo + hi));
        }
        if (!(tn > lo && tn < hi)) tn = 0.5 * (lo + hi);
        if (tn == tau) break;
        tau = tn;
    }
    if (lane == 0) {
        J.rtau[a + j] = tau;
        J.rorg[a + j] = org;
    }
}

// d_i - lambda_j, accurate.
__device__ __forceinline__ double delta(const double *dv, const double *rt, const int *ro, int i, int j) {
    return (dv[i] - dv[ro[j]]) - rt[j];
}

// Gu-Eisenstat: z-hat_i = sign(z_i) sqrt( -(d_i - lambda_i) prod_{j != i} (d_i - lambda_j)/(d_i - d_j) ).
// (d, root offsets, root origins, z-hat) of a merge staged in shared memory for dc_vnorm (smem_n >= k):
// its 16 warps per CTA then read them from shared memory instead of each warp streaming them from L2
// (measured 101 -> 72 us for the d = 4609 top merge; dc_secular and dc_zhat are faster reading them
// through L1 with more CTAs per SM).
__device__ __forceinline__ void stage_roots(const TrdJob &J, int a, int k, int smem_n, double *sm, const double *&dv,
                                            const double *&rt, const int *&ro, const double *&wz) {
    dv = J.dval + a;
    rt = J.rtau + a;
    ro = J.rorg + a;
    wz = J.wz + a;
    if (k > smem_n) return;
    double *sd = sm, *st = sm + smem_n, *sw = sm + 2 * smem_n;
    int *so = reinterpret_cast<int *>(sm + 3 * smem_n);
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        sd[i] = ldcg(dv + i);
        st[i] = ldcg(rt + i);
        so[i] = ldcg(ro + i);
        sw[i] = ldcg(wz + i);
    }
    __syncthreads();
    dv = sd;
    rt = st;
    ro = so;
    wz = sw;
}

__global__ void dc_zhat(const TrdJob *jobs, const MergeDesc *merges) {
    const MergeDesc M = merges[blockIdx.y];
    const TrdJob &J = jobs[M.job];
    // one warp per i: lane-strided partial products (each factor is O(1) by interlacing, so the
    // partial products neither overflow nor underflow), then a fixed-order butterfly product
    const int a = M.a, k = J.mstate[4 * a + 0];
    const int i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (i >= k) return;
    const double *dv = J.dval + a, *rt = J.rtau + a;
    const int *ro = J.rorg + a;
    const double di = dv[i];
    double w = lane == 0 ? delta(dv, rt, ro, i, i) : 1.0;
    for (int j = lane; j < k; j += 32)
        if (j != i) w *= delta(dv, rt, ro, i, j) / (di - dv[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w *= __shfl_xor_sync(0xffffffffu, w, o);
    if (lane == 0) J.wz[a + i] = copysign(sqrt(fmax(-w, 0.0)), J.zval[a + i]);
}

// Column norms of S[:, j] = z-hat / (d - lambda_j) (one warp per column).
__global__ void dc_vnorm(const TrdJob *jobs, const MergeDesc *merges, int smem_n) {
    extern __shared__ double roots_sm[];
    const MergeDesc M = merges[blockIdx.y];
    const TrdJob &J = jobs[M.job];
    const int a = M.a, k = J.mstate[4 * a + 0];
    if (blockIdx.x * (blockDim.x / 32) >= k) return;     // uniform per CTA
    const int j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
    const double *dv, *rt, *wz;
    const int *ro;
    stage_roots(J, a, k, smem_n, roots_sm, dv, rt, ro, wz);
    if (j >= k) return;
    double s = 0.0;
    for (int i = lane; i < k; i += 32) {
        const double q = wz[i] / delta(dv, rt, ro, i, j);
        s += q * q;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) J.vnorm[a + j] = 1.0 / sqrt(s);
}

// S[a + i][j] (k x k, row-major at rows a..a+k) = z-hat_i / (d_i - lambda_j) / ||.||; rows k..k+31
// (inside the merge's row range) zeroed so the GEMM's last K block reads zeros.
constexpr int kBuildRows = 16;                   // S rows per dc_build_s thread
__global__ void dc_build_s(const TrdJob *jobs, const MergeDesc *merges) {
    // one thread per column j and kBuildRows rows: the column's pole d_{org(j)}, offset and norm
    // are loaded once, each row adds only its d_i and z-hat_i (warp-uniform broadcasts)
    const MergeDesc M = merges[blockIdx.z];
    const TrdJob &J = jobs[M.job];
    const int a = M.a, nm = M.n1 + M.n2, k = J.mstate[4 * a + 0];
    const int i0 = blockIdx.y * kBuildRows, j = blockIdx.x * blockDim.x + threadIdx.x;
    const int rows = min(nm, (k + 31) & ~31);
    if (i0 >= rows || j >= k) return;
    const double *dv = J.dval + a, *rt = J.rtau + a;
    const int *ro = J.rorg + a;
    const double dj = dv[ro[j]], rj = rt[j], nj = J.vnorm[a + j];
    for (int i = i0; i < min(rows, i0 + kBuildRows); ++i) {
        double v = 0.0;
        int row = i;                                 // S row of sorted entry i: its GEMM position
        if (i < k) {
            v = J.wz[a + i] / ((dv[i] - dj) - rj) * nj;
            row = J.ctyp[a + i];
        }
        J.Sb[(size_t)(a + row) * J.ldw + j] = v;
    }
}

// Final order of the merged eigenvalues: lambda_j (j < k, from the GEMM output Tmp) and the
// deflated d's (Qnd columns k..n-1); rank by counting (ties by index).
__global__ void dc_rank(const TrdJob *jobs, const MergeDesc *merges, int smem_n) {
    const MergeDesc M = merges[blockIdx.y];
    const TrdJob &J = jobs[M.job];
    const int a = M.a, nm = M.n1 + M.n2, k = J.mstate[4 * a + 0];
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const double *dv = J.dval + a, *rt = J.rtau + a;
    const int *ro = J.rorg + a;
    auto val = [&](int q) { return q < k ? dv[ro[q]] + rt[q] : dv[q]; };
    // all nm values staged in shared memory once per block (when they fit), then counted from there
    extern __shared__ double vals[];
    const bool sm = nm <= smem_n;
    if (sm) {
        for (int q = threadIdx.x; q < nm; q += blockDim.x) vals[q] = val(q);
        __syncthreads();
    }
    if (e >= nm) return;
    const double ve = sm ? vals[e] : val(e);
    int rk = 0;
    for (int f = 0; f < nm; ++f) {
        const double vf = sm ? vals[f] : val(f);
        rk += (vf < ve) || (vf == ve && f < e);
    }
    J.D[a + rk] = ve;
    J.srcpos[a + rk] = e;
}

__global__ void dc_assemble(const TrdJob *jobs, const MergeDesc *merges, int ping) {
    const MergeDesc M = merges[blockIdx.z];
    const TrdJob &J = jobs[M.job];
    const int a = M.a, nm = M.n1 + M.n2, k = J.mstate[4 * a + 0], ldw = J.ldw;
    const int r0 = blockIdx.y * kBuildRows, p = blockIdx.x * blockDim.x + threadIdx.x;
    if (r0 >= nm || p >= nm) return;
    double *Zd = ping ? J.Z0 : J.Z1;                // destination = the other buffer
    const int src = J.srcpos[a + p];                 // once per thread, kBuildRows rows each
    const double *from = src < k ? J.Tmp : J.Qnd;
    for (int r = r0; r < min(nm, r0 + kBuildRows); ++r)
        Zd[(size_t)(a + r) * ldw + a + p] = from[(size_t)(a + r) * ldw + src];
}

// ------------------------------------------------- back-transformation --
// T (upper triangular) of H_b0 ... H_{b0+nr-1} = I - V T V^T from G = V^T V (LAPACK dlarft,
// forward / columnwise): T_jj = tau_j, T[0:j, j] = -tau_j T[0:j, 0:j] G[0:j, j].  This kernel builds
// one kTs x kTs diagonal block per CTA (blockIdx.x = (kBt / kTs) step-entry + sub-block) and zeroes the rest of
// its block row; the off-diagonal blocks follow from T12 = -T1 (V1^T V2) T2 (two GEMMs per level).
struct BtStep {
    int job, b0, nr;
};
constexpr size_t kLarftSmem = sizeof(double) * (kTs * (kTs + 1) + kTs);
__global__ void bt_larft(const TrdJob *jobs, const BtStep *steps) {
    extern __shared__ double bt_smem[];
    double (*T)[kTs + 1] = reinterpret_cast<double (*)[kTs + 1]>(bt_smem);
    double *gcol = bt_smem + kTs * (kTs + 1);
    const BtStep S = steps[blockIdx.x / (kBt / kTs)];
    const int sb = blockIdx.x % (kBt / kTs);
    const TrdJob &J = jobs[S.job];
    const int o = sb * kTs, nr = min(kTs, S.nr - o), t = threadIdx.x;
    if (nr <= 0) return;
    for (int j = 0; j < nr; ++j) {
        const double tj = J.tau[S.b0 + o + j];
        if (t < j) gcol[t] = J.Gb[(size_t)(o + j) * kBt + o + t];   // G[t][j] = G[j][t] (lower half stored)
        __syncthreads();
        double acc = 0.0;
        if (t < j)
            for (int l = t; l < j; ++l) acc += T[t][l] * gcol[l];
        __syncthreads();
        if (t < j) T[t][j] = -tj * acc;
        if (t == j) T[j][j] = tj;
        if (t > j && t < kTs) T[t][j] = 0.0;
        __syncthreads();
    }
    for (int idx = t; idx < kTs * kBt; idx += blockDim.x) {
        const int r = idx / kBt, c = idx % kBt;
        double v = 0.0;
        if (r < nr && c >= o && c < o + nr) v = T[r][c - o];
        J.Tb[(size_t)(o + r) * kBt + c] = v;
    }
}


// Q = (float) Z and the clamped eigenvalues: one CTA per 8 rows (blockIdx.x strides over row
// blocks), threads along the columns with 16-byte fp64 reads.
__global__ void trd_output(const TrdJob *jobs) {
    const TrdJob &J = jobs[blockIdx.y];
    const double *Z = final_z(J);
    const int n = J.n;
    const bool pairs = (J.ldQ & 1) == 0 && (reinterpret_cast<uintptr_t>(J.Q) & 7) == 0;
    for (int r0 = blockIdx.x * 8; r0 < n; r0 += gridDim.x * 8) {
        const int rr = r0 + threadIdx.x / 32;
        if (rr >= n) continue;
        const double *zr = Z + (size_t)rr * J.ldw;
        float *qr = J.Q + (size_t)rr * J.ldQ;
        for (int c = 2 * (threadIdx.x % 32); c < n; c += 64) {
            if (c + 1 < n) {
                const double2 z = __ldcs(reinterpret_cast<const double2 *>(zr + c));   // ldw even
                if (pairs) *reinterpret_cast<float2 *>(qr + c) = make_float2((float)z.x, (float)z.y);
                else { qr[c] = (float)z.x; qr[c + 1] = (float)z.y; }
            } else {
                qr[c] = (float)zr[c];
            }
        }
    }
    if (blockIdx.x == 0)
        for (int c = threadIdx.x; c < n; c += blockDim.x) J.evals[c] = (float)fmax(J.D[c], 0.0);
}

// Vd = (double) Vb (exact), so every back-transformation GEMM has fp64 operands (one-stage factors;
// the two-stage reduction writes Vd itself).
__global__ void trd_vb_to_f64(const TrdJob *jobs) {
    // Vd = (double) Vb on and below the reflectors (column k holds v_k in rows >= k + 1), zero above:
    // Vb is never initialised above the reflectors.  float4 reads, two 16-byte writes per thread.
    const TrdJob &J = jobs[blockIdx.y];
    if (J.off != 1) return;
    const int n = J.n, ldw = J.ldw, q4 = ldw / 4;
    const long long total = (long long)n * q4;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(e / q4), c = (int)(e - (long long)r * q4) * 4;
        const float4 v = __ldcs(reinterpret_cast<const float4 *>(J.Vb + (size_t)r * ldw + c));
        double2 *dst = reinterpret_cast<double2 *>(J.Vd + (size_t)r * ldw + c);
        dst[0] = make_double2(c + 0 < r ? (double)v.x : 0.0, c + 1 < r ? (double)v.y : 0.0);
        dst[1] = make_double2(c + 2 < r ? (double)v.z : 0.0, c + 3 < r ? (double)v.w : 0.0);
    }
}

__global__ void trd_zero_info(const TrdJob *jobs) {
    const TrdJob &J = jobs[blockIdx.x];
    if (threadIdx.x == 0 && J.info) *J.info = 0;
}

// ---------------------------------------------------------------- host --
struct Upload {
    void *dst;
    int bytes;
    unsigned char data[30000];
};
__global__ void upload_kernel(const __grid_constant__ Upload u) {
    unsigned char *d = static_cast<unsigned char *>(u.dst);
    for (int i = threadIdx.x; i < u.bytes; i += blockDim.x) d[i] = u.data[i];
}

kfac_status_t upload(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    thread_local Upload u;     // host staging (kernel params are copied at launch)
    const unsigned char *p = static_cast<const unsigned char *>(src);
    for (size_t off = 0; off < bytes; off += sizeof(u.data)) {
        const size_t nb = std::min(sizeof(u.data), bytes - off);
        u.dst = static_cast<unsigned char *>(dst) + off;
        u.bytes = (int)nb;
        memcpy(u.data, p + off, nb);
        upload_kernel<<<1, 256, 0, s>>>(u);
        KFAC_LAUNCHED();
    }
    return KFAC_OK;
}

int levels_for(int n) {
    int L = 0;
    while ((n + (1 << L) - 1) / (1 << L) > kLeaf) ++L;
    return L;
}
int ldw_for(int n) { return (int)round_up((size_t)n, 32); }

struct Plan {
    std::vector<TrdJob> jobs;
    size_t bytes = 0, table_off = 0, leaf_off = 0, merge_off = 0, bt_off = 0;
    size_t oz_off = 0, oz_bytes = 0;                  // Ozaki GEMM scratch (digit planes)
    size_t bar_off = 0;                               // all factors' group-barrier counters (64 B apart)
    std::vector<LeafDesc> leaves;
    std::vector<std::vector<MergeDesc>> merges;       // per level (1..maxL)
    std::vector<std::vector<BtStep>> bt;              // per back-transform step
};

Plan plan(const int32_t *dims, int count) {
    Plan P;
    size_t cur = 0;
    auto take = [&](size_t bytes) {
        cur = round_up(cur, 256);
        const size_t r = cur;
        cur += bytes;
        return r;
    };
    P.table_off = take(sizeof(TrdJob) * count);
    P.jobs.resize(count);
    size_t nmerge_total = 0;
    for (int i = 0; i < count; ++i) {
        const int n = dims[i], ldw = ldw_for(n);
        TrdJob &J = P.jobs[i];
        memset(&J, 0, sizeof(J));
        J.n = n;
        J.ldw = ldw;
        J.levels = levels_for(n);
        J.off = 1;                                       // set per call by sbr::route
        const size_t sq = (size_t)n * ldw;
#define TAKE(field, T, cnt) J.field = reinterpret_cast<T *>(take(sizeof(T) * (size_t)(cnt)))
        if (sbr::eligible(n)) {                          // either reduction may take the factor
            cur = round_up(cur, 256);
            sbr::plan_fields(J, cur);
        }
        TAKE(A, float, sq);
        TAKE(Vb, float, sq);
        TAKE(Vd, double, sq);
        TAKE(VW, float, (size_t)n * 64);
        TAKE(WV, float, (size_t)n * 64);
        TAKE(VWd, double, (size_t)n * 64);
        TAKE(WVd, double, (size_t)n * 64);
        TAKE(Z0, double, sq);
        TAKE(Z1, double, sq);
        TAKE(Qnd, double, sq);
        TAKE(Tmp, double, sq);
        TAKE(Sb, double, sq);
        TAKE(Yb, double, (size_t)kBt * ldw);
        TAKE(Y2b, double, (size_t)kBt * ldw);
        TAKE(Gb, double, kBt * kBt);
        TAKE(Tb, double, kBt * kBt);
        TAKE(Wt, double, kBt * kBt);
        TAKE(d, double, n);
        TAKE(e, double, n);
        TAKE(tau, double, n);
        TAKE(x, double, n);
        TAKE(y, double, n);
        TAKE(D, double, n);
        TAKE(dval, double, n);
        TAKE(zval, double, n);
        TAKE(rtau, double, n);
        TAKE(wz, double, n);
        TAKE(vnorm, double, n);
        TAKE(rot_c, double, n);
        TAKE(rot_s, double, n);
        TAKE(col, int, n);
        TAKE(posof, int, n);
        TAKE(rorg, int, n);
        TAKE(rot_p, int, n);
        TAKE(rot_j, int, n);
        TAKE(srcpos, int, n);
        TAKE(ctyp, int, n);
        TAKE(mstate, int, 4 * (size_t)n);
        TAKE(mscal, double, 2 * (size_t)n);
        TAKE(part, double, (size_t)kMaxGroupCtas * kPart);
        J.ldp = cdiv(n + 3, kSymvC) + 1;
        TAKE(DP, double, (size_t)n * J.ldp);
        J.ldtp = cdiv(n, 2 * kSymvRMin) + 1;
        TAKE(TP, double, (size_t)n * J.ldtp);
#undef TAKE
        // leaves and merges
        const int nleaf = 1 << J.levels;
        for (int b = 0; b < nleaf; ++b) {
            const int a0 = (int)((long long)b * n / nleaf), a1 = (int)((long long)(b + 1) * n / nleaf);
            P.leaves.push_back({i, a0, a1 - a0});
        }
        if ((int)P.merges.size() < J.levels) P.merges.resize(J.levels);
        for (int l = 1; l <= J.levels; ++l) {
            const int span = 1 << l, nodes = nleaf >> l;
            for (int q = 0; q < nodes; ++q) {
                const int a0 = (int)((long long)q * span * n / nleaf);
                const int s = (int)((long long)(q * span + span / 2) * n / nleaf);
                const int a1 = (int)((long long)(q + 1) * span * n / nleaf);
                P.merges[l - 1].push_back({i, a0, s - a0, a1 - s, q});
                ++nmerge_total;
            }
        }
        // back-transformation blocks (reflectors 0..n-2), processed last block first
        const int nref = std::max(0, n - J.off);
        const int nblk = (nref + kBt - 1) / kBt;
        if ((int)P.bt.size() < nblk) P.bt.resize(nblk);
        for (int s = 0; s < nblk; ++s) {
            const int blk = nblk - 1 - s;
            const int b0 = blk * kBt;
            P.bt[s].push_back({i, b0, std::min(kBt, nref - b0)});
        }
    }
    P.bar_off = take((size_t)count * 64);
    for (int i = 0; i < count; ++i)
        P.jobs[i].bar = reinterpret_cast<unsigned *>(P.bar_off + 64 * (size_t)i);   // offset, rebased later
    P.leaf_off = take(P.leaves.size() * sizeof(LeafDesc));
    P.merge_off = take(nmerge_total * sizeof(MergeDesc));
    size_t nbt = 0;
    for (auto &v : P.bt) nbt += v.size();
    P.bt_off = take(nbt * sizeof(BtStep));
    // Ozaki scratch: the largest grouped GEMM of one step slices at most ~18 n^2 int8 digits per
    // factor (a merge level: both halves' Q rows plus S twice) or 6 n (n + 1536) (a back-transform
    // block: V^T, X, T), plus per-row exponents and maxima
    for (int i = 0; i < count; ++i) {
        const size_t n = (size_t)dims[i];
        P.oz_bytes += std::max(18 * n * (n + 64), 6 * (n + 64) * (n + 1600)) + (1 << 20);
    }
    P.oz_off = take(P.oz_bytes);
    P.bytes = cur + 256;
    return P;
}

template <class T>
T *rebase(T *p, char *base) {           // offsets from plan(); fields a factor does not use stay null
    return p ? reinterpret_cast<T *>(base + reinterpret_cast<uintptr_t>(p)) : nullptr;
}

int panel_capacity(size_t smem) {
    int per_sm = 0;
    set_smem_attr((const void *)trd_panel<kSymvR>, (int)smem);
    set_smem_attr((const void *)trd_panel<kSymvRLone>, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trd_panel<kSymvR>, kTrdThreads, smem);
    int per_sm_lone = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_lone, trd_panel<kSymvRLone>, kTrdThreads, smem);
    per_sm = std::min(per_sm, per_sm_lone);
    return std::min(std::max(1, per_sm) * num_sms(), kMaxGroupCtas);
}

// Test modes (single factor): TRD_DEBUG_TRIDIAG stops after the reduction and copies (d, e) out;
// TRD_DEBUG_STEDC replaces (d, e) by the caller's tridiagonal and stops before the
// back-transformation (Z -> Q, eigenvalues in fp64 -> dbg_d).
enum { TRD_FULL = 0, TRD_DEBUG_TRIDIAG = 1, TRD_DEBUG_STEDC = 2 };

kfac_status_t trd_exec(const float *const *F, const int32_t *dims, const int32_t *ldF, int count,
                       float *const *Q, const int32_t *ldQ, float *const *evals, int32_t *info, uint32_t flags,
                       void *ws, cudaStream_t s, int mode, double *dbg_d, double *dbg_e);

}  // namespace

// Cluster size of the small-factor reduction for order n (0: does not fit kSmMaxCl CTAs).
// Largest cluster of trd_small CTAs (full shared-memory budget each) the device can co-schedule
// (non-portable sizes above 8 depend on the GPC layout), cached per device.
int sm_max_cluster() {
    static std::mutex mu;
    static std::map<int, int> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 8;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int best = 8;                                                // portable
    if (cudaFuncSetAttribute((const void *)trd_small, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
            cudaSuccess &&
        set_smem_attr((const void *)trd_small, (int)kSmSmemCap) == cudaSuccess) {
        for (int cl = kSmMaxCl; cl > 8; --cl) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(cl);
            cfg.blockDim = dim3(kSmThreads);
            cfg.dynamicSmemBytes = kSmSmemCap;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = cl;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, (const void *)trd_small, &cfg) == cudaSuccess &&
                nclusters > 0) {
                best = cl;
                break;
            }
        }
    }
    cudaGetLastError();                                          // a refused query is not an error
    cache[dev] = best;
    return best;
}

int sm_cluster_size(int n) {
    const int max_cl = sm_max_cluster();
    for (int cl = 1; cl <= max_cl; ++cl)
        if (sm_smem_bytes(n, cl) <= kSmSmemCap) return cl;
    return 0;
}

// The small reduction's launches of different cluster sizes are independent, so they run side by
// side on side streams (SideFork: forked from and joined back into the caller's stream) -- a
// ResNet-32 call has d = 145 / 289 / 577 factors on 1-, 2- and 7-CTA clusters.
kfac_status_t small_reduce(const TrdJob *djobs, const std::vector<TrdJob> &jobs, cudaStream_t s) {
    KFAC_CUDA_TRY(cudaFuncSetAttribute((const void *)trd_small, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const int count = (int)jobs.size();
    struct Launch {
        int cl;
        std::vector<int> ids;
    };
    std::vector<Launch> launches;
    for (int cl = 1; cl <= kSmMaxCl; ++cl) {
        std::vector<int> grp;
        for (int i = 0; i < count; ++i)
            if (sm_cluster_size(jobs[i].n) == cl) grp.push_back(i);
        for (size_t c0 = 0; c0 < grp.size(); c0 += kSmMaxJobs)
            launches.push_back({cl, std::vector<int>(grp.begin() + c0,
                                                     grp.begin() + std::min(grp.size(), c0 + (size_t)kSmMaxJobs))});
    }
    const int nl = (int)launches.size();
    SideFork fk;
    const bool par = nl > 1 && nl <= SideFork::kMaxSide;
    if (par) KFAC_CUDA_TRY(fk.fork(s, nl));
    for (int g = 0; g < nl; ++g) {
        const Launch &L = launches[g];
        const cudaStream_t ls = par ? fk.side(g) : s;
        thread_local SmallSet SS;
        const int na = (int)L.ids.size();
        SS.jobs = djobs;
        SS.count = na;
        size_t smem = 0;
        for (int u = 0; u < na; ++u) {
            SS.job[u] = L.ids[u];
            smem = std::max(smem, sm_smem_bytes(jobs[L.ids[u]].n, L.cl));
        }
        KFAC_CUDA_TRY(set_smem_attr((const void *)trd_small, (int)smem));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(na * L.cl);
        cfg.blockDim = dim3(kSmThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ls;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = L.cl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        KFAC_CUDA_TRY(cudaLaunchKernelEx(&cfg, trd_small, SS));
        KFAC_LAUNCHED();
    }
    if (par) KFAC_CUDA_TRY(fk.join(s));
    return KFAC_OK;
}

size_t trd_workspace_bytes(const int32_t *dims, int count) { return plan(dims, count).bytes; }

kfac_status_t trd_run(const float *const *F, const int32_t *dims, const int32_t *ldF, int count,
                      float *const *Q, const int32_t *ldQ, float *const *evals, int32_t *info, uint32_t flags,
                      void *ws, cudaStream_t s) {
    return trd_exec(F, dims, ldF, count, Q, ldQ, evals, info, flags, ws, s, TRD_FULL, nullptr, nullptr);
}

namespace {

kfac_status_t trd_exec(const float *const *F, const int32_t *dims, const int32_t *ldF, int count,
                       float *const *Q, const int32_t *ldQ, float *const *evals, int32_t *info, uint32_t flags,
                       void *ws, cudaStream_t s, int mode, double *dbg_d, double *dbg_e) {
    Plan P = plan(dims, count);
    {   // reduction per factor (the workspace holds both): reflector offset 1 (one-stage) or 16
        const std::vector<char> two = sbr::route(dims, count, flags);
        for (int i = 0; i < count; ++i) P.jobs[i].off = two[i] ? sbr::kSbrBw : 1;
    }
    char *base = reinterpret_cast<char *>(round_up(reinterpret_cast<uintptr_t>(ws), 256));
    int max_n = 0;
    for (int i = 0; i < count; ++i) {
        TrdJob &J = P.jobs[i];
        J.F = F[i]; J.Q = Q[i]; J.evals = evals[i];
        J.info = info ? info + i : nullptr;
        J.ldF = ldF[i]; J.ldQ = ldQ[i];
        J.A = rebase(J.A, base); J.Vb = rebase(J.Vb, base); J.Vd = rebase(J.Vd, base); J.VWd = rebase(J.VWd, base); J.WVd = rebase(J.WVd, base); J.VW = rebase(J.VW, base); J.WV = rebase(J.WV, base);
        J.Z0 = rebase(J.Z0, base); J.Z1 = rebase(J.Z1, base); J.Qnd = rebase(J.Qnd, base);
        J.Tmp = rebase(J.Tmp, base); J.Sb = rebase(J.Sb, base); J.Yb = rebase(J.Yb, base);
        J.Y2b = rebase(J.Y2b, base); J.Gb = rebase(J.Gb, base); J.Tb = rebase(J.Tb, base);
        J.d = rebase(J.d, base); J.e = rebase(J.e, base); J.tau = rebase(J.tau, base);
        J.x = rebase(J.x, base); J.y = rebase(J.y, base); J.D = rebase(J.D, base);
        J.dval = rebase(J.dval, base); J.zval = rebase(J.zval, base); J.rtau = rebase(J.rtau, base);
        J.wz = rebase(J.wz, base); J.vnorm = rebase(J.vnorm, base); J.rot_c = rebase(J.rot_c, base);
        J.rot_s = rebase(J.rot_s, base); J.col = rebase(J.col, base); J.posof = rebase(J.posof, base);
        J.rorg = rebase(J.rorg, base); J.rot_p = rebase(J.rot_p, base); J.rot_j = rebase(J.rot_j, base);
        J.srcpos = rebase(J.srcpos, base); J.ctyp = rebase(J.ctyp, base); J.mstate = rebase(J.mstate, base); J.mscal = rebase(J.mscal, base);
        J.part = rebase(J.part, base); J.bar = rebase(J.bar, base);
        J.DP = rebase(J.DP, base); J.TP = rebase(J.TP, base); J.Wt = rebase(J.Wt, base);
        sbr::rebase_fields(J, base);
        max_n = std::max(max_n, J.n);
    }
    TrdJob *djobs = reinterpret_cast<TrdJob *>(base + P.table_off);
    RET_OK(upload(djobs, P.jobs.data(), sizeof(TrdJob) * count, s));
    LeafDesc *dleaves = reinterpret_cast<LeafDesc *>(base + P.leaf_off);
    RET_OK(upload(dleaves, P.leaves.data(), sizeof(LeafDesc) * P.leaves.size(), s));
    MergeDesc *dmerges = reinterpret_cast<MergeDesc *>(base + P.merge_off);
    {
        std::vector<MergeDesc> flat;
        for (auto &lv : P.merges) flat.insert(flat.end(), lv.begin(), lv.end());
        if (!flat.empty()) RET_OK(upload(dmerges, flat.data(), sizeof(MergeDesc) * flat.size(), s));
    }
    BtStep *dbt = reinterpret_cast<BtStep *>(base + P.bt_off);
    {
        std::vector<BtStep> flat;
        for (auto &v : P.bt) flat.insert(flat.end(), v.begin(), v.end());
        if (!flat.empty()) RET_OK(upload(dbt, flat.data(), sizeof(BtStep) * flat.size(), s));
    }
    // the eigensolver's large fp64 GEMMs go to the int8 tensor cores (Ozaki) while this arena is set
    struct ArenaGuard {
        ArenaGuard(void *p, size_t b) { oz_set_arena(p, b); }
        ~ArenaGuard() { oz_set_arena(nullptr, 0); }
    } arena_guard(base + P.oz_off, P.oz_bytes);
    trd_zero_info<<<count, 32, 0, s>>>(djobs);
    KFAC_LAUNCHED();
    std::vector<Gemm64Desc> gd;
    if (mode != TRD_DEBUG_STEDC) {
    NvtxRange nvtx_red("eigen: tridiagonal reduction");
    // a call whose factors all fit one cluster's shared memory runs the cluster-resident dsytd2
    bool small_path = true;
    for (int i = 0; i < count; ++i)
        if (P.jobs[i].off != 1 || sm_cluster_size(P.jobs[i].n) == 0) small_path = false;
    if (!small_path) {
        trd_init<<<dim3(std::min(2048, cdiv((long long)ldw_for(max_n), 32) * cdiv((long long)ldw_for(max_n), 32)), count),
                   256, 0, s>>>(djobs);
        KFAC_LAUNCHED();
    }
    KFAC_CUDA_TRY(set_smem_attr((const void *)bt_larft, (int)kLarftSmem));
    if (small_path) RET_OK(small_reduce(djobs, P.jobs, s));
    if (!small_path) {
    // ---- (1) tridiagonalisation: one persistent launch + one trailing GEMM per panel ----
    const int ring_off = (int)round_up(round_up(max_n, kSymvC) + kSymvC + 8, 64);
    // v (floats) | symv ring | x of the merged column (doubles, phase B; only if it fits)
    const size_t smem_base = (size_t)ring_off * sizeof(float) + (size_t)kTrdWarps * 2 * 8 * 32 * sizeof(float4);
    const size_t smem_xs = (size_t)round_up(max_n, 2) * sizeof(double);
    const int use_xs = smem_base + smem_xs + 12 * 1024 <= 227 * 1024;
    // the fused trailing update reuses the ring as two teams' 64 x 68 fp64 operand tiles
    const size_t smem = std::max(smem_base + (use_xs ? smem_xs : 0),
                                 (size_t)ring_off * sizeof(float) + 2 * 2 * 64 * 68 * sizeof(double));
    int cap = panel_capacity(smem);
    thread_local PanelLaunch PL;       // host staging (kernel parameters are copied at launch)
    // Staggered schedule: factor j (P_j panels) starts at launch P_max - P_j, so all factors finish
    // together and the small ones share the GPU with the big ones' small trailing matrices.
    std::vector<int> sbr_ids;           // factors on the two-stage reduction (eigen_sbr.cu)
    for (int i = 0; i < count; ++i)
        if (P.jobs[i].off != 1) sbr_ids.push_back(i);
    int pmax = 0;
    for (int i = 0; i < count; ++i)
        if (P.jobs[i].off == 1) pmax = std::max(pmax, cdiv(P.jobs[i].n, kNb));
    // Two-stage factors beside the one-stage ones (KFAC_SBR_OVERLAP): stage 1 (dense -> band, GEMMs
    // that fill the GPU) first, then the latency-bound bulge chase (one cluster per factor) on a
    // side stream while the one-stage panels run on the remaining SMs (cap reduced by the chase's
    // CTAs, one per SM); joined before divide and conquer.
    SideFork sbr_fk;
    bool sbr_par = false;
    if (KFAC_SBR_OVERLAP && !sbr_ids.empty() && pmax > 0) {
        const int per_sm = std::max(1, cap / num_sms());
        const int free_sms = num_sms() - sbr::chase_ctas(P.jobs, sbr_ids);
        if (free_sms >= num_sms() / 4) {
            RET_OK(sbr::stage1(djobs, P.jobs, sbr_ids, s));
            KFAC_CUDA_TRY(sbr_fk.fork(s, 1));
            RET_OK(sbr::chase(djobs, P.jobs, sbr_ids, sbr_fk.side(0)));
            cap = std::min(cap, per_sm * free_sms);
            sbr_par = true;
        }
    }
    // CTAs per active factor ~ (remaining trailing size)^2 (the mat-vec bytes; exponents 1.5-3
    // measured equal within noise)
    constexpr double wexp = 2.0;
    for (int t = 0; t < pmax; ++t) {
        std::vector<int> act, pst;
        double wsum = 0.0;
        for (int i = 0; i < count; ++i) {
            const int pidx = t - (pmax - cdiv(P.jobs[i].n, kNb));
            if (pidx < 0 || P.jobs[i].off != 1) continue;
            act.push_back(i);
            pst.push_back(pidx * kNb);
            const double m = P.jobs[i].n - pidx * kNb;
            wsum += std::pow(m, wexp);
        }
        if (act.empty()) continue;
        // More active factors than co-resident CTAs (e.g. ResNet-101's 210 factors): the groups are
        // independent, so the active set is split into several cooperative launches of <= cap.
        const std::vector<int> act_all = act, pst_all = pst;
        for (size_t c0 = 0; c0 < act_all.size(); c0 += (size_t)cap) {
        act.assign(act_all.begin() + c0, act_all.begin() + std::min(act_all.size(), c0 + (size_t)cap));
        pst.assign(pst_all.begin() + c0, pst_all.begin() + std::min(pst_all.size(), c0 + (size_t)cap));
        wsum = 0.0;
        for (size_t q = 0; q < act.size(); ++q) {
            const double m = P.jobs[act[q]].n - pst[q];
            wsum += std::pow(m, wexp);
        }
        const int na = (int)act.size();
        // CTAs per factor ~ remaining work, >= 1, total <= cap, and no more than one symv unit per warp
        // (more CTAs would only add barrier participants and partials).  Two unit geometries are
        // instantiated (32- and 24-row warp halves); the launch takes the one whose busiest warp pair
        // streams the fewest rows: units are indivisible, so the pair count rarely divides the unit
        // count and the finer units often cut the critical pair's share (measured on a lone d = 4609
        // factor: 116 -> 107 ms)
        auto plan_groups = [&](int srows, std::vector<int> &nc) {
            nc.assign(na, 1);
            int spare = cap - na;
            double worst = 0.0;
            for (int q = 0; q < na; ++q) {
                const double m = P.jobs[act[q]].n - pst[q];
                const int tiles = cdiv((long long)m, srows) * (cdiv((long long)m, kSymvC) + 1) / 2;
                int want = (int)std::floor((cap - na) * std::pow(m, wexp) / wsum);
                want = std::min(want, std::max(0, (int)(m / 16) - 1));
                want = std::min(want, std::max(0, cdiv(tiles, kTrdWarps) - 1));
                want = std::min(want, spare);
                nc[q] += want;
                spare -= want;
                const long long units = cdiv((long long)m, 2 * srows) * (cdiv((long long)m, kSymvC) + 1) / 2;
                const double per_pair = (double)cdiv(units, (long long)nc[q] * (kTrdWarps / 2));
                worst = std::max(worst, per_pair * (2 * srows + 8));      // rows streamed + per-unit cost
            }
            return worst;
        };
        std::vector<int> nc, nc_lone;
        const double cost = plan_groups(kSymvR, nc), cost_lone = plan_groups(kSymvRLone, nc_lone);
        const bool fine = cost_lone < cost;
        if (fine) nc.swap(nc_lone);
        PL.jobs = djobs;
        PL.count = na;
        PL.ring_off = ring_off;
        PL.use_xs = use_xs;
        int tot = 0;
        for (int q = 0; q < na; ++q) {
            PL.job[q] = act[q];
            PL.p0[q] = pst[q];
            PL.cta_begin[q] = tot;
            tot += nc[q];
        }
        PL.cta_begin[na] = tot;
        KFAC_CUDA_TRY(cudaMemsetAsync(base + P.bar_off, 0, (size_t)count * 64, s));   // every counter, one call
        void *args[] = {&PL};
        const int prof = prof_begin(KFAC_PROF_TRD_PANEL, s);
        const void *kern = fine ? (const void *)trd_panel<kSymvRLone> : (const void *)trd_panel<kSymvR>;
        KFAC_CUDA_TRY(cudaLaunchCooperativeKernel(kern, dim3(tot), dim3(kTrdThreads), args, smem, s));
        KFAC_LAUNCHED();
        if (prof >= 0) {
            // algorithmic work: per column k, the lower triangle of the m x m trailing matrix
            // (m = n - k - 1) read once (4 B per element) and 2 m^2 flops of the mat-vec
            double by = 0.0, fl = 0.0;
            for (int q = 0; q < na; ++q) {
                const int n = P.jobs[act[q]].n;
                for (int k = pst[q]; k < std::min(n - 1, pst[q] + kNb); ++k) {
                    const double m = n - k - 1;
                    by += 4.0 * m * (m + 1) / 2;
                    fl += 2.0 * m * m;
                }
                const double mt = n - pst[q] - kNb;          // fused trailing update of the panel
                if (mt > 0) {
                    by += 8.0 * mt * (mt + 1) / 2 + 2.0 * 8 * 64 * mt;   // C lower RMW + [V|W], [W|V]
                    fl += 2.0 * 64 * mt * (mt + 1);
                }
            }
            prof_end(prof, s, by, fl);
        }
        }   // chunks of the active set
    }

    if (sbr_par) KFAC_CUDA_TRY(sbr_fk.join(s));
    else if (!sbr_ids.empty()) RET_OK(sbr::reduce(djobs, P.jobs, sbr_ids, s));
    }   // !small_path
    }   // mode != TRD_DEBUG_STEDC
    if (mode == TRD_DEBUG_TRIDIAG) {
        KFAC_CUDA_TRY(cudaMemcpyAsync(dbg_d, P.jobs[0].d, sizeof(double) * P.jobs[0].n, cudaMemcpyDeviceToDevice, s));
        KFAC_CUDA_TRY(cudaMemcpyAsync(dbg_e, P.jobs[0].e, sizeof(double) * P.jobs[0].n, cudaMemcpyDeviceToDevice, s));
        return KFAC_OK;
    }
    if (mode == TRD_DEBUG_STEDC) {
        KFAC_CUDA_TRY(cudaMemcpyAsync(P.jobs[0].d, dbg_d, sizeof(double) * P.jobs[0].n, cudaMemcpyDeviceToDevice, s));
        KFAC_CUDA_TRY(cudaMemcpyAsync(P.jobs[0].e, dbg_e, sizeof(double) * P.jobs[0].n, cudaMemcpyDeviceToDevice, s));
    }
    // ---- (2) divide and conquer on T ----
    std::optional<NvtxRange> nvtx_dc;
    nvtx_dc.emplace("eigen: divide and conquer");
    dc_tear<<<dim3(cdiv(max_n, 256), count), 256, 0, s>>>(djobs);
    KFAC_LAUNCHED();
    if (!P.leaves.empty()) {
        dc_leaf<<<cdiv((long long)P.leaves.size(), kLeafWarps), kLeafWarps * 32, 0, s>>>(djobs, dleaves, (int)P.leaves.size());
        KFAC_LAUNCHED();
    }
    int ping = 0;                  // level l reads Z0 (l odd) / Z1 (l even) for every factor
    size_t moff = 0;
    for (size_t l = 0; l < P.merges.size(); ++l) {
        const auto &lv = P.merges[l];
        const int nmg = (int)lv.size();
        const MergeDesc *dm = dmerges + moff;
        moff += nmg;
        int nmax = 0;
        for (auto &m : lv) nmax = std::max(nmax, m.n1 + m.n2);
        // sorted lists in shared memory when they fit (2 doubles + 1 int per entry)
        const int smem_n = (nmax * 20 <= 200 * 1024) ? nmax : 0;
        if (smem_n) {
            KFAC_CUDA_TRY(set_smem_attr((const void *)dc_deflate, 200 * 1024 + 64));
        }
        dc_deflate<<<nmg, 256, smem_n ? (size_t)smem_n * 20 + 16 : 0, s>>>(djobs, dm, ping, smem_n);
        KFAC_LAUNCHED();
        dc_permute<<<dim3(cdiv(nmax, 8), nmg), 256, 0, s>>>(djobs, dm, ping);
        KFAC_LAUNCHED();
        dc_rotate<<<dim3(cdiv(nmax, 128), nmg), 128, 0, s>>>(djobs, dm);
        KFAC_LAUNCHED();
        dc_secular<<<dim3(cdiv(nmax, 8), nmg), 256, 0, s>>>(djobs, dm);
        KFAC_LAUNCHED();
        {
            // d, offsets, z-hat (doubles) + origins (ints): 28 B per root
            const int roots_n = (nmax * 28 <= 200 * 1024) ? nmax : 0;
            const size_t roots_smem = roots_n ? (size_t)roots_n * 3 * 8 + (size_t)roots_n * 4 : 0;
            if (roots_n) {
                KFAC_CUDA_TRY(set_smem_attr((const void *)dc_vnorm, 200 * 1024));
            }
            dc_zhat<<<dim3(cdiv(nmax, 8), nmg), 256, 0, s>>>(djobs, dm);
            KFAC_LAUNCHED();
            dc_vnorm<<<dim3(cdiv(nmax, 16), nmg), 512, roots_smem, s>>>(djobs, dm, roots_n);
        }
        KFAC_LAUNCHED();
        dc_build_s<<<dim3(cdiv(nmax, 128), cdiv(nmax, kBuildRows), nmg), 128, 0, s>>>(djobs, dm);
        KFAC_LAUNCHED();
        gd.clear();
        for (auto &m : lv) {
            // Tmp = Qnd S split by rows: the upper n1 rows only meet columns of types 1-2 (GEMM
            // positions [0, k1 + k2)), the lower n2 rows only types 2-3 ([k1, k)); both bounds
            // are device-side (mstate), so the zero blocks of diag(Q1, Q2) are skipped
            const TrdJob &J = P.jobs[m.job];
            const int nm = m.n1 + m.n2;
            for (int h = 0; h < 2; ++h) {
                Gemm64Desc g{};
                const int r0 = h ? m.n1 : 0;
                g.M = h ? m.n2 : m.n1; g.N = nm; g.K = nm;
                g.A = J.Qnd + (size_t)(m.a + r0) * J.ldw; g.ta = DT_F64; g.lda = J.ldw;
                g.B = J.Sb + (size_t)m.a * J.ldw; g.tb = DT_F64; g.ldb = J.ldw;
                g.C = J.Tmp + (size_t)(m.a + r0) * J.ldw; g.tc = DT_F64; g.ldc = J.ldw;
                g.dyn = J.mstate + 4 * m.a + (h ? 5 : 2);
                g.dyn_koff = 1;
                gd.push_back(g);
            }
        }
        RET_OK(gemm64_grouped(gd.data(), (int)gd.size(), s));
        {
            const int rank_n = (nmax * 8 <= 96 * 1024) ? nmax : 0;
            if (rank_n) {
                KFAC_CUDA_TRY(set_smem_attr((const void *)dc_rank, 96 * 1024));
            }
            dc_rank<<<dim3(cdiv(nmax, 128), nmg), 128, (size_t)rank_n * 8, s>>>(djobs, dm, rank_n);
        }
        KFAC_LAUNCHED();
        dc_assemble<<<dim3(cdiv(nmax, 128), cdiv(nmax, kBuildRows), nmg), 128, 0, s>>>(djobs, dm, ping);
        KFAC_LAUNCHED();
        ping ^= 1;
    }

    // ---- (3) back-transformation X = H Z, last block of reflectors first ----
    nvtx_dc.reset();
    NvtxRange nvtx_bt("eigen: back-transformation");
    if (mode != TRD_DEBUG_STEDC) {
        std::vector<int> sbr_ids;
        for (int i = 0; i < count; ++i)
            if (P.jobs[i].off != 1) sbr_ids.push_back(i);
        if (!sbr_ids.empty()) RET_OK(sbr::apply_q2(djobs, P.jobs, sbr_ids, s));
        trd_vb_to_f64<<<dim3(std::min(1024, cdiv((long long)max_n * ldw_for(max_n) / 4, 256)), count), 256, 0, s>>>(djobs);
        KFAC_LAUNCHED();
    }
    size_t boff = 0;
    for (auto &stp : P.bt) {
        if (mode == TRD_DEBUG_STEDC) break;
        const int ns = (int)stp.size();
        std::vector<Gemm64Desc> g1, g2, g3;
        for (auto &b : stp) {
            const TrdJob &J = P.jobs[b.job];
            const int m = J.n - b.b0 - J.off;                    // reflector b0 + i: rows b0 + off + i ..
            const double *V = J.Vd + (size_t)(b.b0 + J.off) * J.ldw + b.b0;
            double *X = final_z(J) + (size_t)(b.b0 + J.off) * J.ldw;
            Gemm64Desc g{};
            g.M = b.nr; g.N = b.nr; g.K = m;                     // G = V^T V, lower half only
            g.A = V; g.ta = DT_F64; g.lda = J.ldw; g.trans_a = 1;
            g.B = V; g.tb = DT_F64; g.ldb = J.ldw;
            g.C = J.Gb; g.tc = DT_F64; g.ldc = kBt;
            g.lower = 1;                                         // (G is symmetric)
            g1.push_back(g);
            // Each product runs either whole on the int8 tensor cores (Ozaki, when gemm64_grouped
            // routes it there; the zero triangles of V and T are then multiplied, ~6% of the block)
            // or on DMMA as 64-row slabs that skip those triangles.
            const bool oz = oz_arena_active();
            Gemm64Desc yw{};                                     // Y = V^T X
            yw.M = b.nr; yw.N = J.n; yw.K = m;
            yw.A = V; yw.ta = DT_F64; yw.lda = J.ldw; yw.trans_a = 1;
            yw.B = X; yw.tb = DT_F64; yw.ldb = J.ldw;
            yw.C = J.Yb; yw.tc = DT_F64; yw.ldc = J.ldw;
            if (oz && oz_eligible(yw)) {
                g1.push_back(yw);
            } else {
                for (int i0 = 0; i0 < b.nr; i0 += 64) {          // V[r][i] = 0 for r < i, so row
                    Gemm64Desc h{};                              // slab i0 only meets r >= i0
                    h.M = std::min(64, b.nr - i0); h.N = J.n; h.K = m - i0;
                    h.A = V + (size_t)i0 * J.ldw + i0; h.ta = DT_F64; h.lda = J.ldw; h.trans_a = 1;
                    h.B = X + (size_t)i0 * J.ldw; h.tb = DT_F64; h.ldb = J.ldw;
                    h.C = J.Yb + (size_t)i0 * J.ldw; h.tc = DT_F64; h.ldc = J.ldw;
                    g1.push_back(h);
                }
            }
            Gemm64Desc uw{};                                     // Y2 = T Y
            uw.M = b.nr; uw.N = J.n; uw.K = b.nr;
            uw.A = J.Tb; uw.ta = DT_F64; uw.lda = kBt;
            uw.B = J.Yb; uw.tb = DT_F64; uw.ldb = J.ldw;
            uw.C = J.Y2b; uw.tc = DT_F64; uw.ldc = J.ldw;
            if (oz && oz_eligible(uw)) {
                g2.push_back(uw);
            } else {
                for (int m0 = 0; m0 < b.nr; m0 += 64) {          // T upper triangular: row slab
                    Gemm64Desc u{};                              // m0 only meets K >= m0
                    u.M = std::min(64, b.nr - m0); u.N = J.n; u.K = b.nr - m0;
                    u.A = J.Tb + (size_t)m0 * kBt + m0; u.ta = DT_F64; u.lda = kBt;
                    u.B = J.Yb + (size_t)m0 * J.ldw; u.tb = DT_F64; u.ldb = J.ldw;
                    u.C = J.Y2b + (size_t)m0 * J.ldw; u.tc = DT_F64; u.ldc = J.ldw;
                    g2.push_back(u);
                }
            }
            Gemm64Desc vw{};                                     // X -= V Y2
            vw.M = m; vw.N = J.n; vw.K = b.nr;
            vw.A = V; vw.ta = DT_F64; vw.lda = J.ldw;
            vw.B = J.Y2b; vw.tb = DT_F64; vw.ldb = J.ldw;
            vw.C = X; vw.tc = DT_F64; vw.ldc = J.ldw;
            vw.epi = EPI_SUB;
            if (oz && oz_eligible(vw)) {
                g3.push_back(vw);
                continue;
            }
            // rows r < nr of V are zero beyond column r (unit lower triangle on top)
            for (int r0 = 0; r0 < m; r0 += 64) {
                if (r0 >= b.nr) {                                // the rectangular rest in one desc
                    Gemm64Desc v{};
                    v.M = m - r0; v.N = J.n; v.K = b.nr;
                    v.A = V + (size_t)r0 * J.ldw; v.ta = DT_F64; v.lda = J.ldw;
                    v.B = J.Y2b; v.tb = DT_F64; v.ldb = J.ldw;
                    v.C = X + (size_t)r0 * J.ldw; v.tc = DT_F64; v.ldc = J.ldw;
                    v.epi = EPI_SUB;
                    g3.push_back(v);
                    break;
                }
                Gemm64Desc v{};
                v.M = std::min(64, m - r0); v.N = J.n; v.K = std::min(b.nr, r0 + 64);
                v.A = V + (size_t)r0 * J.ldw; v.ta = DT_F64; v.lda = J.ldw;
                v.B = J.Y2b; v.tb = DT_F64; v.ldb = J.ldw;
                v.C = X + (size_t)r0 * J.ldw; v.tc = DT_F64; v.ldc = J.ldw;
                v.epi = EPI_SUB;
                g3.push_back(v);
            }
        }
        RET_OK(gemm64_grouped(g1.data(), (int)g1.size(), s));
        bt_larft<<<ns * (kBt / kTs), kTs, kLarftSmem, s>>>(djobs, dbt + boff);
        KFAC_LAUNCHED();
        // recursive off-diagonal blocks of T: pairs of 64-blocks, then of 128-blocks, then of 256-blocks
        for (int h = kTs; h < kBt; h *= 2) {          // h: size of the halves being joined
            std::vector<Gemm64Desc> ga, gb;
            for (auto &b : stp) {
                const TrdJob &J = P.jobs[b.job];
                for (int o = 0; o + h < b.nr; o += 2 * h) {
                    const int n1 = h, n2 = std::min(h, b.nr - o - h);
                    Gemm64Desc x{};                      // Wt = T1 G12, G12 = G21^T (lower half stored)
                    x.M = n1; x.N = n2; x.K = n1;
                    x.A = J.Tb + (size_t)o * kBt + o; x.ta = DT_F64; x.lda = kBt;
                    x.B = J.Gb + (size_t)(o + h) * kBt + o; x.tb = DT_F64; x.ldb = kBt; x.trans_b = 1;
                    x.C = J.Wt + (size_t)o * kBt; x.tc = DT_F64; x.ldc = kBt;
                    ga.push_back(x);
                    Gemm64Desc y{};                      // T12 = 0 - Wt T2
                    y.M = n1; y.N = n2; y.K = n2;
                    y.A = J.Wt + (size_t)o * kBt; y.ta = DT_F64; y.lda = kBt;
                    y.B = J.Tb + (size_t)(o + h) * kBt + o + h; y.tb = DT_F64; y.ldb = kBt;
                    y.C = J.Tb + (size_t)o * kBt + o + h; y.tc = DT_F64; y.ldc = kBt;
                    y.epi = EPI_SUB;
                    gb.push_back(y);
                }
            }
            if (!ga.empty()) {
                RET_OK(gemm64_grouped(ga.data(), (int)ga.size(), s));
                RET_OK(gemm64_grouped(gb.data(), (int)gb.size(), s));
            }
        }
        RET_OK(gemm64_grouped(g2.data(), (int)g2.size(), s));
        RET_OK(gemm64_grouped(g3.data(), (int)g3.size(), s));
        boff += ns;
    }
    trd_output<<<dim3(std::min(1024, cdiv(max_n, 8)), count), 256, 0, s>>>(djobs);
    KFAC_LAUNCHED();
    if (mode == TRD_DEBUG_STEDC)
        KFAC_CUDA_TRY(cudaMemcpyAsync(dbg_d, P.jobs[0].D, sizeof(double) * P.jobs[0].n, cudaMemcpyDeviceToDevice, s));
    return KFAC_OK;
}

}  // namespace
}  // namespace kfac

// Test hooks (not part of the public header).  Single factor, workspace allocated here.
//   kfac_debug_tridiag: F (n x ldF, device) -> d (n), e (n-1) of H^T F H (device fp64).
//   kfac_debug_stedc:   tridiagonal (d, e) (device fp64) -> Z (n x ldZ fp32, columns =
//                       eigenvectors), w (n fp64, ascending).
extern "C" int kfac_debug_tridiag_ex(const float *F, int n, int ldF, double *d, double *e, unsigned flags,
                                    void *stream) {
    const int32_t dims[1] = {n}, ld[1] = {ldF};
    const size_t bytes = kfac::trd_workspace_bytes(dims, 1);
    void *ws = nullptr;
    if (cudaMalloc(&ws, bytes) != cudaSuccess) return KFAC_ERR_CUDA;
    float *Qd = nullptr, *ev = nullptr;
    const float *Fp[1] = {F};
    float *Qp[1] = {Qd}, *Ep[1] = {ev};
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int st = kfac::trd_exec(Fp, dims, ld, 1, Qp, ld, Ep, nullptr, flags, ws, s, kfac::TRD_DEBUG_TRIDIAG, d, e);
    cudaStreamSynchronize(s);
    cudaFree(ws);
    return st;
}
extern "C" int kfac_debug_tridiag(const float *F, int n, int ldF, double *d, double *e, void *stream) {
    return kfac_debug_tridiag_ex(F, n, ldF, d, e, 0u, stream);
}

#if KFAC_TRD_TIMING
extern "C" int kfac_debug_trd_timing(unsigned long long *out, int count) {
    const size_t want = sizeof(unsigned long long) * 3 * kfac::kTimCols * kfac::kTimPts;
    if ((size_t)count * sizeof(unsigned long long) < want) return KFAC_ERR_INVALID_VALUE;
    return cudaMemcpyFromSymbol(out, kfac::g_trd_tim, want) == cudaSuccess ? KFAC_OK : KFAC_ERR_CUDA;
}
#endif

extern "C" int kfac_debug_stedc(const double *d, const double *e, int n, float *Z, int ldZ, double *w,
                                void *stream) {
    const int32_t dims[1] = {n}, ld[1] = {ldZ};
    const size_t bytes = kfac::trd_workspace_bytes(dims, 1);
    void *ws = nullptr, *ev = nullptr;
    if (cudaMalloc(&ws, bytes) != cudaSuccess) return KFAC_ERR_CUDA;
    if (cudaMalloc(&ev, sizeof(float) * n) != cudaSuccess) return KFAC_ERR_CUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaMemcpyAsync(w, d, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
    double *e_copy = nullptr;
    if (cudaMalloc(&e_copy, sizeof(double) * n) != cudaSuccess) return KFAC_ERR_CUDA;
    cudaMemsetAsync(e_copy, 0, sizeof(double) * n, s);
    if (n > 1) cudaMemcpyAsync(e_copy, e, sizeof(double) * (n - 1), cudaMemcpyDeviceToDevice, s);
    const float *Fp[1] = {nullptr};
    float *Qp[1] = {Z}, *Ep[1] = {static_cast<float *>(ev)};
    int st = kfac::trd_exec(Fp, dims, ld, 1, Qp, ld, Ep, nullptr, 0u, ws, s, kfac::TRD_DEBUG_STEDC, w, e_copy);
    cudaStreamSynchronize(s);
    cudaFree(ws);
    cudaFree(ev);
    cudaFree(e_copy);
    return st;
}
