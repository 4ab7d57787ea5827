// gemm_ozaki.cu -- fp64-accurate GEMM on the int8 tensor cores (Ozaki scheme) for the eigensolver's
// large products (divide-and-conquer eigenvector updates Q_nd S, back-transformation V^T X, T Y,
// X - V Y2).
//
// Why: the eigensolver must keep eigenvector errors far below fp32 rounding (the preconditioner
// divides by v_G v_A^T + damping, amplifying them by up to ~Lambda/damping), so
// its GEMMs run in fp64.  The fp64 tensor pipe (DMMA) peaks at ~40 TFLOP/s on B200; the int8 pipe
// (tcgen05 kind::i8, int32 accumulation, 4.5 POPS dense) is exact, so an fp64 product can be
// assembled from a few exact int8 products (Ozaki, Ogita, Oishi, Rump 2012):
//
//   every row r of op(A) is scaled by 2^-e_r (e_r: the exponent of the row's largest |entry| + 1)
//   and split into s = 5 signed digits of 7 bits:  a = 2^e_r sum_i d_i 2^(-7 i) + r_s,
//   |d_i| <= 64, |r_s| <= 2^(e_r - 7 s - 1); op(B)'s columns likewise (exponents f_c, digits d'_j);
//   C[r][c] = 2^(e_r + f_c) sum_{L=2}^{s+1} 2^(-7 L) S_L[r][c],   S_L = sum_{i+j=L} D_i D'_j,
//
// where every S_L is an exact int32 GEMM (|S_L| <= s K 64^2 < 2^31 for K < 100000).  Digit pairs with
// i + j > s + 1 are dropped: with s = 5 the error is below ~K 2^-35 max|a_r| max|b_c| (34 bits; the
// fp32 rounding of the eigenvectors this feeds is 2^-24).  15 int8 products per fp64 product.
// Measured (profiles/r02_n_ozaki_digits.md): s = 6 -> 5 keeps every GPU parity test green with the same
// eigen residuals (largest factor reconstruction 5.5e-8 / 5.6e-8) and saves 2.2 ms per ResNet-50
// update; s = 4 (27 bits) fails the full-size eigen tests (reconstruction 1.2e-6).
//
// Kernels: ozk_rowmax (max |x| per operand row over the valid K range, atomicMax on the bit
// pattern), ozk_slice (exponent + digits, int8 planes [s][R][Kp], K-major), ozk_gemm:
//   128 x 64 output tile per CTA, K staged 64 bytes at a time (SWIZZLE_64B, 3 stages of 60 KB:
//   all s A digit planes and s B digit planes of the k-block, one 3-D TMA box each);
//   warp 0 TMA producer, warp 1 MMA issuer (per k-step, digit plane i of A times the stacked B
//   planes 0..s-1-i in one MMA that starts at TMEM column 64 i, so product (i, j) accumulates into
//   level i + j's 64 columns; 6 MMAs of N <= 256 for s = 5), warps 4-7 the epilogue (TMEM -> fp64 sum of the
//   levels -> 2^(e_r + f_c) -> store / C -= through shared memory in coalesced rows).
#include "internal.cuh"
#include "tc_ptx.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

namespace kfac {

namespace {

#ifndef KFAC_OZ_DIGITS
#define KFAC_OZ_DIGITS 5
#endif
constexpr int kOzS = KFAC_OZ_DIGITS;                  // digits per element
constexpr int kOzPairs = kOzS * (kOzS + 1) / 2;       // 21
constexpr int OBM = 128, OBN = 64, OBK = 64;          // tile M x N, k-block bytes
constexpr int kOzStages = kOzS <= 4 ? 4 : 3;              // stages of the k-block ring (fit 227 KB)
constexpr int kOzATile = OBM * OBK;                   // 8 KB per digit plane
constexpr int kOzBTile = OBN * OBK;                   // 4 KB
constexpr int kOzStageBytes = kOzS * (kOzATile + kOzBTile);   // 60 KB (s = 5)
constexpr int kOzSmem = kOzStages * kOzStageBytes + 1024 + 256;
constexpr int kOzThreads = 256;
constexpr int kOzTmemCols = 512;                      // 6 levels x 64 columns used
constexpr int kOzMaxDescs = 64;
constexpr int kOzMaxOps = 128;
constexpr int kOzEpiStride = OBN + 1;                 // fp64 staging row stride
// smallest K routed here: below it the two slicing passes and the per-tile prologue/epilogue cost
// more than DMMA saves (scripts/micro_ozaki.py)
constexpr int kOzMinK = 512;

static_assert(kOzSmem <= 227 * 1024, "ozaki smem");
static_assert(kOzS * OBN <= kOzTmemCols, "ozaki tmem");

// One operand to slice: op(X) is R x K, op(X)[r][k] = X[r*ld + k] (trans 0) or X[k*ld + r] (trans 1).
struct OzOperand {
    const void *X;
    int8_t *planes;                 // [kOzS][R][Kp]
    int *expo;                      // [R]
    unsigned long long *rmax;       // [R] bit pattern of max |x| (zeroed before the launch)
    const int *dyn;                 // optional device {N_eff, K_eff, K start}
    int dyn_koff, is_b;             // is_b: rows are op(B)'s columns (clipped by dyn[0])
    int dt, ld, trans, R, K, Kp;
    int tile_begin, tiles_k;        // 32-row x 256-k tiles (rowmax) / 32 x 128 (slice)
};

struct OzOpBatch {
    int count;
    OzOperand op[kOzMaxOps];
};

struct OzDesc {
    CUtensorMap ta;                 // 3-D: {Kp, M, s} int8, SWIZZLE_64B, box {64, 128, 6}
    CUtensorMap tb;                 // 3-D: {Kp, N, s} int8, box {64, 64, 6}
    const int *ea, *eb;
    void *C;
    const int *dyn;
    int dyn_koff, tc, ldc, M, N, K, epi, lower, tile_begin, tiles_n;
};

struct __align__(64) OzBatch {
    OzDesc d[kOzMaxDescs];
    int count;
};

__device__ __forceinline__ int op_range(const OzOperand &o, int &k0, int &k1, int &r1) {
    k0 = 0;
    k1 = o.K;
    r1 = o.R;
    if (o.dyn) {
        k1 = min(k1, o.dyn[1]);
        if (o.dyn_koff) k0 = max(0, o.dyn[2]);
        if (o.is_b) r1 = min(r1, o.dyn[0]);
    }
    return 0;
}

__device__ __forceinline__ double ld_op(const OzOperand &o, int r, int k) {
    const size_t i = o.trans ? (size_t)k * o.ld + r : (size_t)r * o.ld + k;
    return o.dt == DT_F64 ? __ldg(static_cast<const double *>(o.X) + i) : (double)__ldg(static_cast<const float *>(o.X) + i);
}

__device__ __forceinline__ int find_op(const OzOpBatch &b, int blk) {
    int lo = 0, hi = b.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (b.op[mid].tile_begin <= blk) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// 16-byte load of op(X) elements (i, i+1) (fp64: one double2; fp32: one float2 widened).
__device__ __forceinline__ double2 ld_pair(const OzOperand &o, size_t i) {
    if (o.dt == DT_F64) return __ldg(reinterpret_cast<const double2 *>(static_cast<const double *>(o.X) + i));
    const float2 f = __ldg(reinterpret_cast<const float2 *>(static_cast<const float *>(o.X) + i));
    return make_double2((double)f.x, (double)f.y);
}
// pairs along the contiguous index are aligned: even leading dimension and 16-byte (fp64) / 8-byte
// (fp32) aligned base
__device__ __forceinline__ bool pair_ok(const OzOperand &o) {
    return (o.ld & 1) == 0 && (reinterpret_cast<uintptr_t>(o.X) & (o.dt == DT_F64 ? 15 : 7)) == 0;
}

// max |op(X)[r][k]| over the valid range, per row; 32 rows x 256 k per CTA of 32 x 8 threads.  All of
// a thread's loads are issued before any is used (pairs along the contiguous index when aligned).
__global__ void __launch_bounds__(256) ozk_rowmax(const __grid_constant__ OzOpBatch b) {
    __shared__ double red[8][33];
    const OzOperand &o = b.op[find_op(b, blockIdx.x)];
    const int t = blockIdx.x - o.tile_begin;
    const int r0 = (t / o.tiles_k) * 32, kt0 = (t % o.tiles_k) * 256;
    int k0, k1, r1;
    op_range(o, k0, k1, r1);
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
    const bool vec = pair_ok(o);
    double m = 0.0;
    if (!o.trans) {
        // X[r][k]: lanes along k (coalesced); warp ty covers rows ty, ty + 8, ...; reduce per row
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = r0 + ty + 8 * j;
            double mr = 0.0;
            if (r < r1) {
                double x[8];
                if (vec) {                                   // lane: k pairs kt0 + 2 tx + 64 i
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int k = kt0 + 2 * tx + 64 * i;
                        const double2 p = (k + 1 < k1 && k >= k0) ? ld_pair(o, (size_t)r * o.ld + k) : make_double2(0.0, 0.0);
                        x[2 * i] = p.x;
                        x[2 * i + 1] = p.y;
                        if (!(k + 1 < k1 && k >= k0)) {      // ragged edge: element loads
                            x[2 * i] = (k >= k0 && k < k1) ? ld_op(o, r, k) : 0.0;
                            x[2 * i + 1] = (k + 1 >= k0 && k + 1 < k1) ? ld_op(o, r, k + 1) : 0.0;
                        }
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int k = kt0 + tx + 32 * i;
                        x[i] = (k >= k0 && k < k1) ? ld_op(o, r, k) : 0.0;
                    }
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) mr = fmax(mr, fabs(x[i]));
            }
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) mr = fmax(mr, __shfl_xor_sync(0xffffffffu, mr, s));
            if (tx == 0 && r < r1 && mr > 0.0)
                atomicMax(o.rmax + r, (unsigned long long)__double_as_longlong(mr));
        }
        return;
    }
    // X[k][r]: lanes along r (coalesced); thread (ty, tx) covers k = ty, ty + 8, ... of row r0 + tx
    const int r = r0 + tx;
    if (r < r1) {
#pragma unroll
        for (int i0 = 0; i0 < 32; i0 += 8) {
            double x[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int k = kt0 + ty + 8 * (i0 + i);
                x[i] = (k >= k0 && k < k1) ? ld_op(o, r, k) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) m = fmax(m, fabs(x[i]));
        }
    }
    red[ty][tx] = m;
    __syncthreads();
    if (ty == 0) {
        for (int j = 1; j < 8; ++j) m = fmax(m, red[j][tx]);
        if (r < r1 && m > 0.0) atomicMax(o.rmax + r, (unsigned long long)__double_as_longlong(m));
    }
}

// Exponent and the kOzS int8 digits of every element; 32 rows x 128 k per CTA (staged through shared
// memory so both the fp64 read and the int8 write are coalesced for either storage order).
__global__ void __launch_bounds__(256) ozk_slice(const __grid_constant__ OzOpBatch b) {
    __shared__ double tile[32][129];
    __shared__ int ex[32];
    const OzOperand &o = b.op[find_op(b, blockIdx.x)];
    const int t = blockIdx.x - o.tile_begin;
    const int r0 = (t / o.tiles_k) * 32, kt0 = (t % o.tiles_k) * 128;
    int k0, k1, r1;
    op_range(o, k0, k1, r1);
    const int tid = threadIdx.x;
    if (tid < 32) {
        const int r = r0 + tid;
        int e = 0;
        if (r < o.R) {
            const double m = __longlong_as_double((long long)o.rmax[r]);
            if (m > 0.0) {
                int p;
                frexp(m, &p);          // m < 2^p
                e = p + 1;             // |x| 2^-e < 1/2: the first digit is at most 64
            }
            if (kt0 == 0) o.expo[r] = e;
        }
        ex[tid] = e;
    }
    // stage the 32 x 128 tile: every thread issues its 8 pair loads (16 bytes each, along the
    // contiguous index) before storing any; element loads at ragged edges / unaligned operands
    {
        const bool vec = pair_ok(o);
        double2 x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i2 = tid + 256 * u;                // pair index in the tile
            int rr, kk;
            if (!o.trans) { rr = i2 / 64; kk = 2 * (i2 % 64); }
            else          { kk = i2 / 16; rr = 2 * (i2 % 16); }
            const int r = r0 + rr, k = kt0 + kk;
            const bool full = !o.trans ? (r < r1 && k >= k0 && k + 1 < k1) : (r + 1 < r1 && k >= k0 && k < k1);
            if (vec && full) {
                x[u] = ld_pair(o, !o.trans ? (size_t)r * o.ld + k : (size_t)k * o.ld + r);
            } else if (!o.trans) {
                x[u].x = (r < r1 && k >= k0 && k < k1) ? ld_op(o, r, k) : 0.0;
                x[u].y = (r < r1 && k + 1 >= k0 && k + 1 < k1) ? ld_op(o, r, k + 1) : 0.0;
            } else {
                x[u].x = (r < r1 && k >= k0 && k < k1) ? ld_op(o, r, k) : 0.0;
                x[u].y = (r + 1 < r1 && k >= k0 && k < k1) ? ld_op(o, r + 1, k) : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i2 = tid + 256 * u;
            if (!o.trans) {
                const int rr = i2 / 64, kk = 2 * (i2 % 64);
                tile[rr][kk] = x[u].x;
                tile[rr][kk + 1] = x[u].y;
            } else {
                const int kk = i2 / 16, rr = 2 * (i2 % 16);
                tile[rr][kk] = x[u].x;
                tile[rr + 1][kk] = x[u].y;
            }
        }
    }
    __syncthreads();
    // thread: one row, 16 consecutive k -> one 16-byte store per digit plane
    const int rr = tid / 8, kseg = (tid % 8) * 16, r = r0 + rr;
    if (r >= o.R || kt0 + kseg >= o.Kp) return;
    const int e = ex[rr];
    // 2^(7 - e) as a double built from its exponent bits (exact scaling): one multiply per element
    // instead of ldexp; rows whose maximum is denormal (7 - e outside the normal range) keep ldexp
    const int be = 1023 + 7 - e;
    const bool fast = be >= 1 && be <= 2046;
    const double scale = fast ? __longlong_as_double((long long)be << 52) : 0.0;
    uint32_t w[kOzS][4];
#pragma unroll
    for (int s = 0; s < kOzS; ++s)
#pragma unroll
        for (int q = 0; q < 4; ++q) w[s][q] = 0u;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        double v = fast ? tile[rr][kseg + u] * scale : ldexp(tile[rr][kseg + u], 7 - e);
#pragma unroll
        for (int s = 0; s < kOzS; ++s) {
            const double d = rint(v);
            v = (v - d) * 128.0;
            w[s][u / 4] |= ((uint32_t)(uint8_t)(int8_t)(int)d) << (8 * (u % 4));
        }
    }
    const size_t plane = (size_t)o.R * o.Kp;
#pragma unroll
    for (int s = 0; s < kOzS; ++s)
        *reinterpret_cast<uint4 *>(o.planes + s * plane + (size_t)r * o.Kp + kt0 + kseg) =
            make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
}

__device__ __forceinline__ int find_desc_oz(const OzBatch &b, int tile) {
    int lo = 0, hi = b.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (b.d[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ uint64_t oz_desc(uint32_t addr) {
    return smem_desc(addr, 16, 512, 4);         // K-major, SWIZZLE_64B: 8-row atoms of 64-byte rows
}

__global__ void __launch_bounds__(kOzThreads, 1) ozk_gemm(const __grid_constant__ OzBatch batch) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t a0 = smem_u32(smem_raw);
    uint8_t *base = smem_raw + (((a0 + 1023u) & ~1023u) - a0);
    uint64_t *bars = reinterpret_cast<uint64_t *>(base + kOzStages * kOzStageBytes);
    const uint32_t full = smem_u32(bars), empty = smem_u32(bars + kOzStages), tfull = smem_u32(bars + 2 * kOzStages);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * kOzStages + 1);

    const int di = find_desc_oz(batch, blockIdx.x);
    const OzDesc &d = batch.d[di];
    const int local = blockIdx.x - d.tile_begin;
    const int m0 = (local / d.tiles_n) * OBM, n0 = (local % d.tiles_n) * OBN;
    int Ne = d.N, ke = d.K, ks0 = 0;
    if (d.dyn) {
        Ne = min(Ne, d.dyn[0]);
        ke = min(ke, d.dyn[1]);
        if (d.dyn_koff) ks0 = max(0, d.dyn[2]);
    }
    if (n0 >= Ne) return;
    if (d.lower && n0 >= m0 + OBM) return;
    const int kb0 = ks0 / OBK, kb1 = (ke + OBK - 1) / OBK;
    const int nk = max(0, kb1 - kb0);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kOzStages; ++i) {
            mbar_init(full + 8 * i, 1);
            mbar_init(empty + 8 * i, 1);
        }
        mbar_init(tfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        if (lane == 0) {
            prefetch_map(&d.ta);
            prefetch_map(&d.tb);
        }
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kOzTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            for (int q = 0; q < nk; ++q) {
                const int s = q % kOzStages;
                if (q >= kOzStages) mbar_wait(empty + 8 * s, ((q / kOzStages) - 1) & 1);
                const uint32_t st = smem_u32(base + s * kOzStageBytes);
                mbar_expect_tx(full + 8 * s, kOzStageBytes);
                const int kc = (kb0 + q) * OBK;
                tma_load_3d(st, &d.ta, full + 8 * s, kc, m0, 0);
                tma_load_3d(st + kOzS * kOzATile, &d.tb, full + 8 * s, kc, n0, 0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // A digit plane i times the stacked B planes 0 .. s-1-i in ONE instruction: product
            // (i, j) lands in TMEM columns 64 (i + j) -- level i + j -- because the MMA starts at
            // column 64 i and the B planes are consecutive 64-row blocks in shared memory; N is split
            // at 256 (the instruction's maximum).  6 MMAs per k-step instead of 15 (s = 5), so each reads
            // the A tile once per plane and B in up to 256-row blocks (half the smem operand traffic).
            const uint32_t idesc0 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OBM >> 4) << 24);
            for (int q = 0; q < nk; ++q) {
                const int s = q % kOzStages;
                mbar_wait(full + 8 * s, (q / kOzStages) & 1);
                tc_fence_after();
                const uint32_t sa = smem_u32(base + s * kOzStageBytes), sb = sa + kOzS * kOzATile;
#pragma unroll
                for (int ks = 0; ks < OBK / 32; ++ks) {
#pragma unroll
                    for (int i = 0; i < kOzS; ++i) {
#pragma unroll
                        for (int j0 = 0; j0 + i < kOzS; j0 += 4) {
                            const int nb = min(4, kOzS - i - j0);          // B planes in this MMA
                            const uint32_t idesc = idesc0 | ((uint32_t)((nb * OBN) >> 3) << 17);
                            mma_i8(tmem + (uint32_t)((i + j0) * OBN), oz_desc(sa + i * kOzATile + ks * 32),
                                   oz_desc(sb + j0 * kOzBTile + ks * 32), idesc, (q > 0 || ks > 0 || i > 0) ? 1u : 0u);
                        }
                    }
                }
                mma_commit(empty + 8 * s);
            }
            if (nk > 0) mma_commit(tfull);
        }
    } else if (warp >= 4) {
        const int wq = warp - 4, row = wq * 32 + lane, m = m0 + row;
        double acc[OBN];
#pragma unroll
        for (int j = 0; j < OBN; ++j) acc[j] = 0.0;
        if (nk > 0) {
            mbar_wait(tfull, 0);
            tc_fence_after();
#pragma unroll
            for (int L = 0; L < kOzS; ++L) {
                const double w = ldexp(1.0, -7 * (L + 2));
#pragma unroll
                for (int c = 0; c < OBN / 32; ++c) {
                    uint32_t r[32];
                    tmem_ld32(tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(L * OBN + c * 32), r);
#pragma unroll
                    for (int j = 0; j < 32; ++j) acc[c * 32 + j] = fma((double)(int)r[j], w, acc[c * 32 + j]);
                }
            }
        }
        // stage the scaled tile (every MMA and TMA has completed: the stages are free); the scale
        // 2^(e_r + f_c) is an exact power of two built from its exponent bits when it is normal
        double *stg = reinterpret_cast<double *>(base);
        const int er = m < d.M ? d.ea[m] : 0;
#pragma unroll
        for (int j = 0; j < OBN; ++j) {
            const int n = n0 + j;
            const int sc = er + (n < Ne ? __ldg(d.eb + n) : 0);
            const double p2 = (sc >= -1022 && sc <= 1023) ? __longlong_as_double((long long)(sc + 1023) << 52)
                                                           : ldexp(1.0, sc);
            stg[row * kOzEpiStride + j] = n < Ne ? acc[j] * p2 : 0.0;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        // coalesced rows: warp wq writes its 32 rows, lanes over 2 columns each; for C -= the 64 C
        // values of the lane are all loaded before any is used (independent loads in flight)
        const int nrows = min(32, d.M - (m0 + wq * 32));
        const bool sub = d.epi == EPI_SUB;
        if (d.tc == DT_F64) {
            double *C = static_cast<double *>(d.C);
            double cin[64];
#pragma unroll
            for (int rr = 0; rr < 32; ++rr)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int n = n0 + lane + 32 * h;
                    cin[2 * rr + h] = (sub && rr < nrows && n < Ne) ? __ldcg(C + (size_t)(m0 + wq * 32 + rr) * d.ldc + n) : 0.0;
                }
#pragma unroll
            for (int rr = 0; rr < 32; ++rr)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int n = n0 + lane + 32 * h;
                    if (rr >= nrows || n >= Ne) continue;
                    const double v = stg[(wq * 32 + rr) * kOzEpiStride + lane + 32 * h];
                    C[(size_t)(m0 + wq * 32 + rr) * d.ldc + n] = sub ? cin[2 * rr + h] - v : v;
                }
        } else {
            float *C = static_cast<float *>(d.C);
            float cin[64];
#pragma unroll
            for (int rr = 0; rr < 32; ++rr)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int n = n0 + lane + 32 * h;
                    cin[2 * rr + h] = (sub && rr < nrows && n < Ne) ? __ldcg(C + (size_t)(m0 + wq * 32 + rr) * d.ldc + n) : 0.f;
                }
#pragma unroll
            for (int rr = 0; rr < 32; ++rr)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int n = n0 + lane + 32 * h;
                    if (rr >= nrows || n >= Ne) continue;
                    const double v = stg[(wq * 32 + rr) * kOzEpiStride + lane + 32 * h];
                    C[(size_t)(m0 + wq * 32 + rr) * d.ldc + n] = sub ? (float)((double)cin[2 * rr + h] - v) : (float)v;
                }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kOzTmemCols));
    }
}

PFN_cuTensorMapEncodeTiled_v12000 oz_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 3-D int8 map over the digit planes [kOzS][R][Kp]: box {64 bytes of k, rows, all kOzS planes}.
bool oz_map(CUtensorMap *map, const int8_t *planes, int R, int Kp, int box_rows) {
    auto fn = oz_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)R, (cuuint64_t)kOzS};
    cuuint64_t strides[2] = {(cuuint64_t)Kp, (cuuint64_t)Kp * R};
    cuuint32_t box[3] = {(cuuint32_t)OBK, (cuuint32_t)box_rows, (cuuint32_t)kOzS};
    cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t *>(planes), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline int oz_kp(int K) { return (int)round_up((size_t)K, 16); }

size_t oz_operand_bytes(int R, int K) {
    return round_up((size_t)kOzS * R * oz_kp(K), 256) + round_up(sizeof(int) * R, 256) +
           round_up(sizeof(unsigned long long) * R, 256);
}

thread_local char *g_oz_base = nullptr;
thread_local size_t g_oz_bytes = 0;

}  // namespace

size_t oz_scratch_bytes(const Gemm64Desc &g) { return oz_operand_bytes(g.M, g.K) + oz_operand_bytes(g.N, g.K); }

bool oz_eligible(const Gemm64Desc &g) {
    return g.ta == DT_F64 && g.tb == DT_F64 && g.M >= OBM && g.N >= OBN && g.K >= kOzMinK && g.K < 80000 &&
           oz_encode_fn() != nullptr;
}

void oz_set_arena(void *base, size_t bytes) {
    g_oz_base = static_cast<char *>(base);
    g_oz_bytes = base ? bytes : 0;
}
bool oz_arena_active() { return g_oz_base != nullptr; }

kfac_status_t oz_gemm_grouped(const Gemm64Desc *descs, int count, cudaStream_t s) {
    KFAC_CUDA_TRY(set_smem_attr((const void *)ozk_gemm, kOzSmem));
    for (int base = 0; base < count;) {
        // as many descriptors as fit the arena (and the kernel-parameter batches)
        size_t used = 0;
        int end = base;
        while (end < count && end - base < std::min(kOzMaxDescs, kOzMaxOps / 2)) {
            const size_t need = oz_scratch_bytes(descs[end]);
            if (used + need > g_oz_bytes) break;
            used += need;
            ++end;
        }
        if (end == base) {
            set_error("oz_gemm_grouped: Ozaki scratch arena too small");
            return KFAC_ERR_WORKSPACE;
        }
        thread_local OzOpBatch ob;
        thread_local OzBatch gb;
        memset(&ob, 0, sizeof(ob));
        memset(&gb, 0, sizeof(gb));
        char *p = g_oz_base;
        char *rmax_lo = nullptr, *rmax_hi = nullptr;
        int rm_tiles = 0, sl_tiles = 0;
        std::vector<int> rm_begin, sl_begin;
        for (int i = base; i < end; ++i) {
            const Gemm64Desc &g = descs[i];
            for (int w = 0; w < 2; ++w) {
                OzOperand &o = ob.op[ob.count++];
                o.X = w ? g.B : g.A;
                o.dt = w ? g.tb : g.ta;
                o.ld = w ? g.ldb : g.lda;
                // op(A)[r][k]: trans_a = 0 -> A[r*lda + k]; op(B)^T[c][k] = op(B)[k][c]:
                // trans_b = 0 -> B[k*ldb + c] (transposed access), trans_b = 1 -> B[c*ldb + k]
                o.trans = w ? (g.trans_b ? 0 : 1) : (g.trans_a ? 1 : 0);
                o.R = w ? g.N : g.M;
                o.K = g.K;
                o.Kp = oz_kp(g.K);
                o.is_b = w;
                o.dyn = g.dyn;
                o.dyn_koff = g.dyn_koff;
                o.planes = reinterpret_cast<int8_t *>(p);
                p += round_up((size_t)kOzS * o.R * o.Kp, 256);
                o.expo = reinterpret_cast<int *>(p);
                p += round_up(sizeof(int) * o.R, 256);
                o.rmax = reinterpret_cast<unsigned long long *>(p);
                if (!rmax_lo) rmax_lo = p;
                p += round_up(sizeof(unsigned long long) * o.R, 256);
                rmax_hi = p;
            }
        }
        // rmax regions are interleaved with the planes: zero each one (small memsets)
        for (int q = 0; q < ob.count; ++q)
            KFAC_CUDA_TRY(cudaMemsetAsync(ob.op[q].rmax, 0, sizeof(unsigned long long) * ob.op[q].R, s));
        (void)rmax_lo;
        (void)rmax_hi;
        for (int q = 0; q < ob.count; ++q) {
            OzOperand &o = ob.op[q];
            o.tiles_k = cdiv(o.K, 256);
            o.tile_begin = rm_tiles;
            rm_tiles += cdiv(o.R, 32) * o.tiles_k;
        }
        ozk_rowmax<<<rm_tiles, 256, 0, s>>>(ob);
        KFAC_LAUNCHED();
        for (int q = 0; q < ob.count; ++q) {
            OzOperand &o = ob.op[q];
            o.tiles_k = cdiv(o.Kp, 128);
            o.tile_begin = sl_tiles;
            sl_tiles += cdiv(o.R, 32) * o.tiles_k;
        }
        ozk_slice<<<sl_tiles, 256, 0, s>>>(ob);
        KFAC_LAUNCHED();
        int tiles = 0;
        for (int i = base; i < end; ++i) {
            const Gemm64Desc &g = descs[i];
            const OzOperand &oa = ob.op[2 * (i - base)], &obb = ob.op[2 * (i - base) + 1];
            OzDesc &z = gb.d[gb.count++];
            if (!oz_map(&z.ta, oa.planes, oa.R, oa.Kp, OBM) || !oz_map(&z.tb, obb.planes, obb.R, obb.Kp, OBN)) {
                set_error("cuTensorMapEncodeTiled failed (ozaki)");
                return KFAC_ERR_CUDA;
            }
            z.ea = oa.expo;
            z.eb = obb.expo;
            z.C = g.C;
            z.dyn = g.dyn;
            z.dyn_koff = g.dyn_koff;
            z.tc = g.tc;
            z.ldc = g.ldc;
            z.M = g.M;
            z.N = g.N;
            z.K = g.K;
            z.epi = g.epi;
            z.lower = g.lower;
            z.tiles_n = cdiv(g.N, OBN);
            z.tile_begin = tiles;
            tiles += cdiv(g.M, OBM) * z.tiles_n;
        }
        const int prof = prof_begin(KFAC_PROF_GEMM64, s);
        ozk_gemm<<<tiles, kOzThreads, kOzSmem, s>>>(gb);
        KFAC_LAUNCHED();
        if (prof >= 0) {
            double by = 0.0, fl = 0.0;
            for (int i = base; i < end; ++i) {
                const Gemm64Desc &g = descs[i];
                const double mn = g.lower ? 0.5 * g.M * (g.N + 1.0) : (double)g.M * g.N;
                fl += 2.0 * mn * g.K;
                by += 8.0 * ((double)g.M * g.K + (double)g.N * g.K) + mn * 8 * (g.epi == EPI_SUB ? 2 : 1);
            }
            prof_end(prof, s, by, fl);
        }
        base = end;
    }
    return KFAC_OK;
}

}  // namespace kfac

// Test hooks: one Ozaki GEMM (fp64 operands; epi 0 store / 3 C -= ...).  kfac_debug_ozaki allocates
// the scratch and synchronises; kfac_debug_ozaki_ws takes caller scratch (size: kfac_debug_ozaki_bytes)
// and only enqueues (timing).
extern "C" int kfac_debug_ozaki_digits(void) { return kfac::kOzS; }

extern "C" size_t kfac_debug_ozaki_bytes(int M, int N, int K) {
    kfac::Gemm64Desc d{};
    d.M = M; d.N = N; d.K = K;
    return kfac::oz_scratch_bytes(d) + 1024;
}

extern "C" int kfac_debug_ozaki_ws(const double *A, int lda, int trans_a, const double *B, int ldb, int trans_b,
                                   void *C, int tc, int ldc, int M, int N, int K, int epi, void *ws, size_t bytes,
                                   void *stream) {
    kfac::Gemm64Desc d{};
    d.A = A; d.ta = kfac::DT_F64; d.lda = lda; d.trans_a = trans_a;
    d.B = B; d.tb = kfac::DT_F64; d.ldb = ldb; d.trans_b = trans_b;
    d.C = C; d.tc = tc; d.ldc = ldc;
    d.M = M; d.N = N; d.K = K; d.epi = epi;
    kfac::oz_set_arena(ws, bytes);
    int st = kfac::oz_gemm_grouped(&d, 1, reinterpret_cast<cudaStream_t>(stream));
    kfac::oz_set_arena(nullptr, 0);
    return st;
}

extern "C" int kfac_debug_ozaki(const double *A, int lda, int trans_a, const double *B, int ldb, int trans_b,
                                void *C, int tc, int ldc, int M, int N, int K, int epi, void *stream) {
    const size_t bytes = kfac_debug_ozaki_bytes(M, N, K);
    void *ws = nullptr;
    if (cudaMalloc(&ws, bytes) != cudaSuccess) return KFAC_ERR_CUDA;
    int st = kfac_debug_ozaki_ws(A, lda, trans_a, B, ldb, trans_b, C, tc, ldc, M, N, K, epi, ws, bytes, stream);
    cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
    cudaFree(ws);
    return st;
}
