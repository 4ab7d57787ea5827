// gemm_tc.cu -- tcgen05 tensor-core grouped GEMM, kind::tf32 with a 3xTF32 split (fp32-faithful).
//
//   C = op(A) op(B) (+ Eq. 14 epilogue), 128x128 output tile per CTA, K staged 32 at a time.
//
// Warp roles (256 threads):
//   warp 0      TMA producer: one elected lane loads the raw fp32 A/B tiles of a k-block with
//               cp.async.bulk.tensor (128-byte swizzle) into the "hi" slots of a stage;
//   warps 4..7  split warpgroup: hi = x rounded to TF32, lo = (x - hi) rounded to TF32 (x - hi
//               is exact in fp32), both exactly representable so the hardware's own TF32
//               conversion is a no-op; hi overwrites the raw tile, lo goes to the "lo" slots,
//               then fence.proxy.async so the tensor core sees the generic-proxy writes;
//               after the main loop the same warps are the epilogue (tcgen05.ld -> registers ->
//               divide by v_G v_A^T + damping -> global);
//   warp 1      MMA issuer: one thread issues, per k-step of 8, the three products
//               A_lo B_hi + A_hi B_lo + A_hi B_hi into the TMEM accumulator (128 lanes x 128
//               columns fp32) and commits the smem slot back to the producer;
//   warp 2      TMEM allocator.
// Operand tiles may be K-major (k contiguous) or MN-major (m/n contiguous); the UMMA
// instruction descriptor's major bits select the layout, so no operand is ever transposed.
#include "internal.cuh"
#include "tc_ptx.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <vector>

namespace kfac {
namespace {

constexpr int BM = 128, BN = 128, BK = 32;
constexpr int kRaw = 4;                                 // raw (hi) stages: operand tiles in flight
constexpr int kLo = 2;                                  // lo stages: written by the split, read by the MMA
constexpr int kTileBytes = BM * BK * 4;                 // 16 KB per operand tile
constexpr int kStageBytes = 2 * kTileBytes;             // A, B
constexpr int kBarBytes = 512;
constexpr int kSmemBytes = (kRaw + kLo) * kStageBytes + 1024 /*align*/ + kBarBytes;
constexpr int kMaxTc = 24;                              // problems per launch (tensor maps in params)
constexpr int kMaxSyrk = 64;
constexpr int NT = 320;                                 // 10 warps
constexpr int kTmemCols = 256;                          // two 128-column accumulators

// warp roles
constexpr int W_SPLIT0 = 0;     // warps 0-3: (SYRK producer) + hi/lo split
constexpr int W_DRAIN0 = 4;     // warps 4-7: TMEM drain into fp32 registers + epilogue
constexpr int W_TMA = 8;        // warp 8: TMA producer (GEMM) + TMEM allocator
constexpr int W_MMA = 9;        // warp 9: MMA issuer

struct TcDesc {
    CUtensorMap ta;       // 128 B, 64-byte aligned
    CUtensorMap tb;
    float *C;
    const float *vr;
    const float *vc;
    const int *dyn;       // optional device {N_eff, K_eff}
    int M, N, K, ldc;
    int a_mn, b_mn, epi, lower;
    int tile_begin, tiles_n;
};

struct SyrkBatch {
    int count;
    int drain;
    FactorJob j[kMaxSyrk];
};

__device__ const float kBiasChunk[4] = {1.f, 0.f, 0.f, 0.f};   // the homogeneous column (R7)

// ------------------------------------------------------- shared pieces --
struct Smem {
    uint8_t *base;       // kRaw raw stages, then kLo lo stages (each A tile + B tile)
    uint32_t raw_full, ready, raw_empty, lo_empty, tfull, tempty;   // barrier arrays (8 B stride)
    uint32_t *tmem_slot;
    int2 *rowtab;        // SYRK producer: per warp 8 (origin offset, packed ih0/iw0) row descriptors
    __device__ __forceinline__ uint8_t *raw(int s) const { return base + s * kStageBytes; }
    __device__ __forceinline__ uint8_t *lo(int l) const { return base + (kRaw + l) * kStageBytes; }
};

// Round an fp32 value to the nearest TF32 (10-bit mantissa), ties away from zero; exact in fp32.
__device__ __forceinline__ float tf32_rn(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int kstep, int mn_major) {
    // k-step of 8 tf32: K-major advances 32 B inside the 128-B swizzle row (SBO 1024 = 8-row
    // atoms); MN-major (BASE32B) advances 8 k-rows = 1024 B (SBO 512 = 4-row k-groups,
    // LBO 4096 = 32-element mn groups).
    if (!mn_major) return smem_desc(base + kstep * 32, 16, 1024, 2);
    return smem_desc(base + kstep * 1024, 4096, 512, 1);
}

// Drain warps: every segment's 128x128 partial product is added into fp32 registers with IEEE
// rounding (the tensor-core accumulator truncates, so an accumulation stays in TMEM for only
// 12 * drain MMAs).  Thread (quarter wq, lane) owns row 32*wq + lane.
__device__ __forceinline__ void drain_loop(const Smem &S, uint32_t tmem, int nk, int wq, float (&acc)[BN],
                                           int drain) {
#pragma unroll
    for (int j = 0; j < BN; ++j) acc[j] = 0.f;
    const int nseg = (nk + drain - 1) / drain;
    for (int sg = 0; sg < nseg; ++sg) {
        const int b = sg & 1;
        mbar_wait(S.tfull + 8 * b, (sg >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(tmem + b * BN + ((uint32_t)(wq * 32) << 16) + c * 32, r);
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[c * 32 + j] += __uint_as_float(r[j]);
        }
        tc_fence_before();
        mbar_arrive(S.tempty + 8 * b);
    }
}

// ------------------------------------------------------------ GEMM kernel --
//   K-major: one box {32 (k), 128 (mn)}, 128B swizzle -> 128 rows x 128 B
//   MN-major: four boxes {32 (mn), 32 (k)}, 128B swizzle with 32-B atoms -> 32 k-rows x 128 B each
__device__ __forceinline__ void load_tile(uint32_t dst, const CUtensorMap *map, uint32_t bar, int mn0, int k0, int mn_major) {
    if (!mn_major) {
        tma_load_2d(dst, map, bar, k0, mn0);
    } else {
#pragma unroll
        for (int g = 0; g < 4; ++g) tma_load_2d(dst + g * 4096, map, bar, mn0 + 32 * g, k0);
    }
}

// --------------------------------------------------- planes GEMM kernel --
// Operands arrive pre-split as TF32 planes (hi, lo), so there is no split pass: per k-block the
// TMA warp loads four 16 KB tiles [A_hi | B_hi | A_lo | B_lo] into one of kPS stages, the MMA
// thread issues the three products straight from them, the drain warps accumulate the TMEM
// segments in fp32 registers and the epilogue leaves through shared memory in coalesced 512-byte
// rows (optionally as hi/lo planes again, for the next GEMM of the chain).
constexpr int kPS = 3;                                  // stages of 64 KB
constexpr int kPlaneStage = 4 * kTileBytes;
constexpr int kEpiStride = 132;                         // staging row stride (floats), 16-B aligned

struct __align__(64) TcPlanesBatch {
    TcDesc d[kMaxTc];
    CUtensorMap ta_lo[kMaxTc];
    CUtensorMap tb_lo[kMaxTc];
    float *c_lo[kMaxTc];
    int count;
    float damping;
    int drain;
};

__device__ __forceinline__ int find_desc_p(const TcPlanesBatch &b, int tile) {
    int lo = 0, hi = b.count - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (b.d[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(NT, 1) gemm_tc_planes_kernel(const __grid_constant__ TcPlanesBatch batch) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t a0 = smem_u32(smem_raw);
    uint8_t *base = smem_raw + (((a0 + 1023u) & ~1023u) - a0);
    uint64_t *bars = reinterpret_cast<uint64_t *>(base + kPS * kPlaneStage);
    const uint32_t full = smem_u32(bars), empty = smem_u32(bars + kPS);
    Smem S;                                             // drain_loop's view: TMEM barriers only
    S.base = base;
    S.tfull = smem_u32(bars + 2 * kPS);
    S.tempty = smem_u32(bars + 2 * kPS + 2);
    S.tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * kPS + 4);

    const int di = find_desc_p(batch, blockIdx.x);
    const TcDesc &d = batch.d[di];
    const int local = blockIdx.x - d.tile_begin;
    const int m0 = (local / d.tiles_n) * BM, n0 = (local % d.tiles_n) * BN;
    const int Ne = d.dyn ? min(d.N, d.dyn[0]) : d.N, Ke = d.dyn ? min(d.K, d.dyn[1]) : d.K;
    const int nk = (Ke + BK - 1) / BK;
    if (n0 >= Ne || nk <= 0) return;
    if (d.lower && n0 >= m0 + BM) return;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kPS; ++i) {
            mbar_init(full + 8 * i, 1);
            mbar_init(empty + 8 * i, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(S.tfull + 8 * b, 1);
            mbar_init(S.tempty + 8 * b, 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == W_TMA) {
        if (lane == 0) {
            prefetch_map(&d.ta); prefetch_map(&d.tb);
            prefetch_map(&batch.ta_lo[di]); prefetch_map(&batch.tb_lo[di]);
        }
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(S.tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *S.tmem_slot;

    if (warp == W_TMA) {
        if (lane == 0) {
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % kPS;
                if (kb >= kPS) mbar_wait(empty + 8 * s, ((kb / kPS) - 1) & 1);
                const uint32_t st = smem_u32(base + s * kPlaneStage);
                mbar_expect_tx(full + 8 * s, kPlaneStage);
                load_tile(st, &d.ta, full + 8 * s, m0, kb * BK, d.a_mn);
                load_tile(st + kTileBytes, &d.tb, full + 8 * s, n0, kb * BK, d.b_mn);
                load_tile(st + 2 * kTileBytes, &batch.ta_lo[di], full + 8 * s, m0, kb * BK, d.a_mn);
                load_tile(st + 3 * kTileBytes, &batch.tb_lo[di], full + 8 * s, n0, kb * BK, d.b_mn);
            }
        }
    } else if (warp == W_MMA) {
        if (lane == 0) {
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)d.a_mn << 15) |
                                   ((uint32_t)d.b_mn << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
            const int drain = batch.drain;
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % kPS;
                const int seg = kb / drain, pos = kb - seg * drain, b = seg & 1, u = seg >> 1;
                mbar_wait(full + 8 * s, (kb / kPS) & 1);
                if (pos == 0 && u >= 1) mbar_wait(S.tempty + 8 * b, (u - 1) & 1);
                tc_fence_after();
                const uint32_t st = smem_u32(base + s * kPlaneStage);
                const uint32_t a_hi = st, b_hi = st + kTileBytes, a_lo = st + 2 * kTileBytes, b_lo = st + 3 * kTileBytes;
                const uint32_t dt = tmem + b * BN;
#pragma unroll
                for (int ks = 0; ks < BK / 8; ++ks) {
                    mma_tf32(dt, operand_desc(a_lo, ks, d.a_mn), operand_desc(b_hi, ks, d.b_mn), idesc,
                             (ks > 0 || pos > 0) ? 1u : 0u);
                    mma_tf32(dt, operand_desc(a_hi, ks, d.a_mn), operand_desc(b_lo, ks, d.b_mn), idesc, 1u);
                    mma_tf32(dt, operand_desc(a_hi, ks, d.a_mn), operand_desc(b_hi, ks, d.b_mn), idesc, 1u);
                }
                mma_commit(empty + 8 * s);
                if (pos == drain - 1 || kb == nk - 1) mma_commit(S.tfull + 8 * b);
            }
        }
    } else if (warp >= W_DRAIN0 && warp < W_TMA) {
        const int wq = warp - W_DRAIN0;
        float acc[BN];
        drain_loop(S, tmem, nk, wq, acc, batch.drain);
        // every MMA has completed (the last tfull), so the stages are free: stage this warp's
        // 32 x 128 block row-major, then leave in coalesced rows (lane -> 4 consecutive columns)
        float *stg = reinterpret_cast<float *>(base) + wq * 32 * kEpiStride;
#pragma unroll
        for (int j = 0; j < BN / 4; ++j)
            *reinterpret_cast<float4 *>(stg + lane * kEpiStride + 4 * j) =
                make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
        __syncwarp();
        const int n = n0 + 4 * lane;
        float vc[4] = {0.f, 0.f, 0.f, 0.f};
        if (epi_uses_vectors(d.epi))
#pragma unroll
            for (int e = 0; e < 4; ++e) vc[e] = n + e < Ne ? d.vc[n + e] : 0.f;
        float *clo = batch.c_lo[di];
        const bool vec = n + 3 < Ne;
        for (int r = 0; r < 32; ++r) {
            const int m = m0 + wq * 32 + r;
            if (m >= d.M) break;
            const float4 a4 = *reinterpret_cast<const float4 *>(stg + r * kEpiStride + 4 * lane);
            float v[4] = {a4.x, a4.y, a4.z, a4.w};
            const float vr = epi_uses_vectors(d.epi) ? d.vr[m] : 0.f;
            float *crow = d.C + (size_t)m * d.ldc;
            float cin[4] = {0.f, 0.f, 0.f, 0.f};
            if (d.epi == EPI_SUB) {
                if (vec) {
                    const float4 c4 = *reinterpret_cast<const float4 *>(crow + n);
                    cin[0] = c4.x; cin[1] = c4.y; cin[2] = c4.z; cin[3] = c4.w;
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) if (n + e < Ne) cin[e] = crow[n + e];
                }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (d.epi == EPI_DIV_EIGEN) v[e] = v[e] / fmaxf(fmaf(vr, vc[e], batch.damping), 1e-12f);
                else if (d.epi == EPI_DIV_FACTORED) v[e] = v[e] / fmaxf((vr + batch.damping) * (vc[e] + batch.damping), 1e-12f);
                else if (d.epi == EPI_SUB) v[e] = cin[e] - v[e];
            }
            if (clo) {                                    // result as TF32 planes (next GEMM's operand)
                float h[4], l[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    h[e] = tf32_rn(v[e]);
                    l[e] = tf32_rn(v[e] - h[e]);
                }
                float *lrow = clo + (size_t)m * d.ldc;
                if (vec) {
                    *reinterpret_cast<float4 *>(crow + n) = make_float4(h[0], h[1], h[2], h[3]);
                    *reinterpret_cast<float4 *>(lrow + n) = make_float4(l[0], l[1], l[2], l[3]);
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (n + e < Ne) { crow[n + e] = h[e]; lrow[n + e] = l[e]; }
                }
            } else if (vec) {
                *reinterpret_cast<float4 *>(crow + n) = make_float4(v[0], v[1], v[2], v[3]);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) if (n + e < Ne) crow[n + e] = v[e];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == W_TMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

// x -> (rn_tf32(x), rn_tf32(x - hi)), one float4 unit per thread and iteration, grid-stride over
// the units of all jobs (job j: rows x ld_dst/4 units; columns >= cols are written as zeros).
struct SplitBatch {
    int count;
    SplitJob j[64];
    long long unit_begin[65];
};

__global__ void __launch_bounds__(256) split_planes_kernel(const __grid_constant__ SplitBatch b) {
    const long long total = b.unit_begin[b.count];
    for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < total;
         u += (long long)gridDim.x * blockDim.x) {
        int lo = 0, hi = b.count - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (b.unit_begin[mid] <= u) lo = mid; else hi = mid - 1;
        }
        const SplitJob &J = b.j[lo];
        const long long v = u - b.unit_begin[lo];
        const int w4 = J.ld_dst / 4;
        const long long r = v / w4;
        const int c = (int)(v - r * w4) * 4;
        float x[4], h[4], l[4];
        if (J.ld_src >= J.ld_dst) {
            const float4 x4 = __ldg(reinterpret_cast<const float4 *>(J.src + r * J.ld_src + c));
            x[0] = x4.x; x[1] = x4.y; x[2] = x4.z; x[3] = x4.w;
        } else {                                   // rows padded with zero columns (ld_dst > cols)
#pragma unroll
            for (int e = 0; e < 4; ++e) x[e] = c + e < J.cols ? __ldg(J.src + r * J.ld_src + c + e) : 0.f;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float xe = c + e < J.cols ? x[e] : 0.f;
            h[e] = tf32_rn(xe);
            l[e] = tf32_rn(xe - h[e]);
        }
        *reinterpret_cast<float4 *>(J.hi + r * J.ld_dst + c) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4 *>(J.lo + r * J.ld_dst + c) = make_float4(l[0], l[1], l[2], l[3]);
    }
}
// ------------------------------------------------------------ SYRK kernel --
__device__ __forceinline__ int find_job(const SyrkBatch &b, int item) {
    int lo = 0, hi = b.count - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (b.j[mid].item_begin <= item) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ void upper_tile(int tau, int t1d, int &ti, int &tj) {
    int i = 0;
    while (tau >= t1d - i) { tau -= t1d - i; ++i; }
    ti = i;
    tj = i + tau;
}

// Byte offset of the 16-B chunk (k, m..m+3) in an MN-major SWIZZLE_128B_BASE32B operand tile
// (128 m x 32 k): 32-m groups of 4 KB, k-rows of 128 B, 32-B chunks XOR (k % 4).
__device__ __forceinline__ uint32_t mn_off(int k, int m) {
    return (uint32_t)((m >> 5) * 4096 + k * 128 + ((((m & 31) >> 3) ^ (k & 3)) << 5) + ((m & 7) << 2));
}

// Gather descriptor of a 4-column chunk of X = [im2col | 1] (or of the gradient rows).
struct ChunkInfo {
    int off, kh, kw, kind;    // kind 0: load, 1: bias chunk {1,0,0,0}, 2: zero
};

__device__ __forceinline__ ChunkInfo chunk_info(const FactorJob &J, int c) {
    ChunkInfo ci{0, 0, 0, 2};
    if (c >= J.d) return ci;
    if (!J.is_a) { ci.kind = 0; ci.off = c; return ci; }
    if (c >= J.patch_cols) { ci.kind = 1; return ci; }
    const int kwc = J.k_w * J.c_in;
    ci.kh = c / kwc;
    const int rem = c - ci.kh * kwc;
    ci.kw = rem / J.c_in;
    ci.off = (ci.kh * J.w_in + ci.kw) * J.c_in + (rem - ci.kw * J.c_in);
    ci.kind = 0;
    return ci;
}

// Geometry of one SYRK job, copied out of the (dynamically indexed) kernel parameters once.
struct SyrkGeom {
    const float *src;
    int is_a, c_in, h_in, w_in, h_out, w_out, stride_h, stride_w, pad_h, pad_w;
    const float *src_lo;
};

// ------------------------------------------------- planes SYRK, wide producer --
// Same pipeline as syrk_tc_planes_kernel with twice the gather throughput: 8 producer warps (warp
// w fills k-rows w + 8j, j < 4) and 8 drain warps (two per TMEM lane quadrant, 64 columns each,
// so an accumulator row needs 64 registers), 18 warps in all.
constexpr int NT2 = 576;
#ifndef KFAC_SYRK_SPLIT_MAJOR
#define KFAC_SYRK_SPLIT_MAJOR 1
#endif
constexpr int W2_DRAIN0 = 8, W2_ALLOC = 16, W2_MMA = 17;

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}

template <bool IS_A>
__device__ __forceinline__ void syrk_issue_planes8(const SyrkGeom &G, uint32_t st, int2 *tabw, long long r0,
                                                   long long r_end, const ChunkInfo (&ci)[2], int cc, int warp,
                                                   int lane, bool diag) {
    if (!IS_A) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = warp + 8 * j;
            const long long r = r0 + k;
            const bool rv = r < r_end;
            const float *rowh = G.src + (size_t)r * G.c_in, *rowl = G.src_lo + (size_t)r * G.c_in;
#pragma unroll
            for (int op = 0; op < 2; ++op) {
                if (op == 1 && diag) break;
                const uint32_t dhi = st + op * kTileBytes + mn_off(k, 4 * cc);
                if (ci[op].kind == 1) {
                    cp_async16(dhi, kBiasChunk, rv ? 16u : 0u);
                    cp_async16(dhi + 2 * kTileBytes, kBiasChunk, 0u);
                    continue;
                }
                const bool ok = rv && ci[op].kind == 0;
                cp_async16(dhi, ok ? rowh + ci[op].off : G.src, ok ? 16u : 0u);
                cp_async16(dhi + 2 * kTileBytes, ok ? rowl + ci[op].off : G.src_lo, ok ? 16u : 0u);
            }
        }
        return;
    }
    int org = 0, ihw = 0;
    {
        const long long r = r0 + warp + 8 * (lane & 3);
        const bool rv = r < r_end;
        const int hw = G.h_out * G.w_out;
        const int ri = rv ? (int)r : 0;
        const int img = ri / hw;
        const int p = ri - img * hw;
        const int oh = p / G.w_out, ow = p - (p / G.w_out) * G.w_out;
        const int ih0 = oh * G.stride_h - G.pad_h, iw0 = ow * G.stride_w - G.pad_w;
        org = ((img * G.h_in + ih0) * G.w_in + iw0) * G.c_in;
        ihw = rv ? (int)(((unsigned)ih0 << 16) | ((unsigned)iw0 & 0xffffu)) : (int)0x80000000;
    }
    __syncwarp();
    if (lane < 4) tabw[lane] = make_int2(org, ihw);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int k = warp + 8 * j;
        const int2 rd = tabw[j];
        const int o = rd.x, hv = rd.y;
        const bool rv = hv != (int)0x80000000;
        const int ih0 = hv >> 16, iw0 = (int)(short)(hv & 0xffff);
#pragma unroll
        for (int op = 0; op < 2; ++op) {
            if (op == 1 && diag) break;
            const uint32_t dhi = st + op * kTileBytes + mn_off(k, 4 * cc);
            const uint32_t dlo = dhi + 2 * kTileBytes;
            const ChunkInfo &c = ci[op];
            if (c.kind == 1) {
                cp_async16(dhi, kBiasChunk, rv ? 16u : 0u);
                cp_async16(dlo, kBiasChunk, 0u);
                continue;
            }
            const bool ok = rv && c.kind == 0 && (unsigned)(ih0 + c.kh) < (unsigned)G.h_in &&
                            (unsigned)(iw0 + c.kw) < (unsigned)G.w_in;
            cp_async16(dhi, ok ? G.src + (o + c.off) : G.src, ok ? 16u : 0u);
            cp_async16(dlo, ok ? G.src_lo + (o + c.off) : G.src_lo, ok ? 16u : 0u);
        }
    }
}

__global__ void __launch_bounds__(NT2, 1) syrk_tc_planes8_kernel(const __grid_constant__ SyrkBatch batch) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t a0 = smem_u32(smem_raw);
    uint8_t *base = smem_raw + (((a0 + 1023u) & ~1023u) - a0);
    uint64_t *bars = reinterpret_cast<uint64_t *>(base + kPS * kPlaneStage);
    const uint32_t full = smem_u32(bars), empty = smem_u32(bars + kPS);
    const uint32_t tfull = smem_u32(bars + 2 * kPS), tempty = smem_u32(bars + 2 * kPS + 2);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * kPS + 4);
    int2 *rowtab = reinterpret_cast<int2 *>(bars + 32);

    const int item = blockIdx.x;
    const FactorJob &J = batch.j[find_job(batch, item)];
    const int local = item - J.item_begin;
#if KFAC_SYRK_SPLIT_MAJOR
    // row-chunk-major: the CTAs resident together share row chunks, so the column blocks every
    // tile of a chunk re-reads (and the im2col halo) come from L2, not HBM
    const int tau = local % J.tiles, split = local / J.tiles;
#else
    const int tau = local / J.splits, split = local % J.splits;
#endif
    int ti, tj;
    upper_tile(tau, J.t1d, ti, tj);
    const bool diag = ti == tj;
    const long long r_begin = (long long)split * J.chunk;
    const long long r_end = min(J.n, r_begin + J.chunk);
    const int nk = (int)((r_end - r_begin + BK - 1) / BK);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kPS; ++i) {
            mbar_init(full + 8 * i, 256);
            mbar_init(empty + 8 * i, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull + 8 * b, 1);
            mbar_init(tempty + 8 * b, 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == W2_ALLOC) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int drain = batch.drain;

    if (warp == W2_MMA) {
        if (lane == 0) {
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
                                   ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % kPS;
                const int seg = kb / drain, pos = kb - seg * drain, b = seg & 1, u = seg >> 1;
                mbar_wait(full + 8 * s, (kb / kPS) & 1);
                if (pos == 0 && u >= 1) mbar_wait(tempty + 8 * b, (u - 1) & 1);
                tc_fence_after();
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const uint32_t st = smem_u32(base + s * kPlaneStage);
                const uint32_t a_hi = st, a_lo = st + 2 * kTileBytes;
                const uint32_t b_hi = diag ? a_hi : st + kTileBytes, b_lo = diag ? a_lo : st + 3 * kTileBytes;
                const uint32_t dt = tmem + b * BN;
#pragma unroll
                for (int ks = 0; ks < BK / 8; ++ks) {
                    mma_tf32(dt, operand_desc(a_lo, ks, 1), operand_desc(b_hi, ks, 1), idesc, (ks > 0 || pos > 0) ? 1u : 0u);
                    mma_tf32(dt, operand_desc(a_hi, ks, 1), operand_desc(b_lo, ks, 1), idesc, 1u);
                    mma_tf32(dt, operand_desc(a_hi, ks, 1), operand_desc(b_hi, ks, 1), idesc, 1u);
                }
                mma_commit(empty + 8 * s);
                if (pos == drain - 1 || kb == nk - 1) mma_commit(tfull + 8 * b);
            }
        }
    } else if (warp < W2_DRAIN0) {
        const int cc = lane;
        ChunkInfo ci[2] = {chunk_info(J, ti * BM + 4 * cc), chunk_info(J, tj * BM + 4 * cc)};
        SyrkGeom G{J.src, J.is_a, J.c_in, J.h_in, J.w_in, J.h_out, J.w_out,
                   J.stride_h, J.stride_w, J.pad_h, J.pad_w, J.src_lo};
        const bool plain = !G.is_a || (J.k_w == 1 && J.h_in == J.h_out && J.w_in == J.w_out && J.pad_h == 0 &&
                                       J.pad_w == 0 && J.stride_h == 1 && J.stride_w == 1);
        int2 *tabw = rowtab + warp * 4;
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % kPS;
            if (kb >= kPS) mbar_wait(empty + 8 * s, ((kb / kPS) - 1) & 1);
            const uint32_t st = smem_u32(base + s * kPlaneStage);
            if (plain)
                syrk_issue_planes8<false>(G, st, tabw, r_begin + (long long)kb * BK, r_end, ci, cc, warp, lane, diag);
            else
                syrk_issue_planes8<true>(G, st, tabw, r_begin + (long long)kb * BK, r_end, ci, cc, warp, lane, diag);
            cp_async_arrive(full + 8 * s);
        }
    } else if (warp < W2_ALLOC) {
        // drain warp: TMEM lane quadrant (warp % 4), column half h
        const int wq = warp % 4, h = (warp - W2_DRAIN0) / 4;
        float acc[64];
#pragma unroll
        for (int j = 0; j < 64; ++j) acc[j] = 0.f;
        const int nseg = (nk + drain - 1) / drain;
        for (int sg = 0; sg < nseg; ++sg) {
            const int b = sg & 1;
            mbar_wait(tfull + 8 * b, (sg >> 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t r[16];
                tmem_ld16(tmem + b * BN + ((uint32_t)(wq * 32) << 16) + h * 64 + c * 16, r);
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[c * 16 + j] += __uint_as_float(r[j]);
            }
            tc_fence_before();
            mbar_arrive(tempty + 8 * b);
        }
        float4 *dst = reinterpret_cast<float4 *>(J.partial + ((size_t)split * J.tiles + tau) * (BM * BN) +
                                                 (size_t)(wq * 32 + lane) * BN + h * 64);
#pragma unroll
        for (int j = 0; j < 16; ++j) dst[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == W2_ALLOC) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

// ------------------------------------------------------------- host side --
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// 2-D fp32 row-major tensor of `rows` x `cols` (cols contiguous) with leading dimension ld.
bool make_map(CUtensorMap *map, const float *ptr, int rows, int cols, int ld, int box_cols, int box_rows,
              CUtensorMapSwizzle swz) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// k-blocks per TMEM accumulation segment: the tensor core's fp32 accumulation
// truncates, so a segment stays in TMEM for 2 k-blocks (24 MMAs) before the IEEE drain.
constexpr int kDrainGemm = 2;
constexpr int kDrainSyrk = 2;

}  // namespace

bool gemm_tc_supported(const GemmDesc &d) {
    if (d.M < 64 || d.N < 64 || d.K < 32) return false;         // small problems: SIMT
    if ((d.lda & 3) || (d.ldb & 3) || (d.ldc & 3)) return false;
    if (!aligned16(d.A) || !aligned16(d.B)) return false;
    return encode_fn() != nullptr;
}

kfac_status_t gemm_tc_planes_grouped(const GemmDesc *descs, int count, float damping, cudaStream_t s) {
    KFAC_CUDA_TRY(set_smem_attr((const void *)gemm_tc_planes_kernel, kSmemBytes));
    static_assert(kPS * kPlaneStage + 1024 + 2 * kPS * 8 + 64 <= kSmemBytes, "planes smem");
    for (int base = 0; base < count; base += kMaxTc) {
        thread_local TcPlanesBatch b;    // host staging (kernel parameters are copied at launch)
        memset(&b, 0, sizeof(b));
        b.damping = damping;
        b.drain = kDrainGemm;
        int tiles = 0;
        for (int i = base; i < count && b.count < kMaxTc; ++i) {
            const GemmDesc &g = descs[i];
            const int q = b.count;
            TcDesc &t = b.d[q];
            t.a_mn = g.trans_a ? 1 : 0;
            t.b_mn = g.trans_b ? 0 : 1;
            const CUtensorMapSwizzle kmaj = CU_TENSOR_MAP_SWIZZLE_128B, mnmaj = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
            auto mapA = [&](CUtensorMap *m, const float *p) {
                return t.a_mn ? make_map(m, p, g.K, g.M, g.lda, 32, 32, mnmaj) : make_map(m, p, g.M, g.K, g.lda, 32, 128, kmaj);
            };
            auto mapB = [&](CUtensorMap *m, const float *p) {
                return t.b_mn ? make_map(m, p, g.K, g.N, g.ldb, 32, 32, mnmaj) : make_map(m, p, g.N, g.K, g.ldb, 32, 128, kmaj);
            };
            if (!(mapA(&t.ta, g.A) && mapB(&t.tb, g.B) && mapA(&b.ta_lo[q], g.A_lo) && mapB(&b.tb_lo[q], g.B_lo))) {
                set_error("cuTensorMapEncodeTiled failed (planes)");
                return KFAC_ERR_CUDA;
            }
            t.C = g.C; t.vr = g.vr; t.vc = g.vc; t.dyn = g.dyn; t.lower = g.lower;
            t.M = g.M; t.N = g.N; t.K = g.K; t.ldc = g.ldc; t.epi = g.epi;
            b.c_lo[q] = g.C_lo;
            t.tiles_n = cdiv(g.N, BN);
            t.tile_begin = tiles;
            tiles += cdiv(g.M, BM) * t.tiles_n;
            ++b.count;
        }
        if (!b.count) continue;
        const int prof = prof_begin(KFAC_PROF_GEMM_TC, s);
        gemm_tc_planes_kernel<<<tiles, NT, kSmemBytes, s>>>(b);
        KFAC_LAUNCHED();
        if (prof >= 0) {
            double by = 0.0, fl = 0.0;
            for (int i = 0; i < b.count; ++i) {
                const TcDesc &g = b.d[i];
                fl += 2.0 * g.M * g.N * g.K;
                by += 4.0 * ((double)g.M * g.K + (double)g.K * g.N + (double)g.M * g.N);
            }
            prof_end(prof, s, by, fl);
        }
    }
    return KFAC_OK;
}

kfac_status_t split_planes(const SplitJob *jobs, int count, cudaStream_t s) {
    for (int base = 0; base < count; base += 64) {
        SplitBatch b;
        b.count = 0;
        long long units = 0;
        for (int i = base; i < count && b.count < 64; ++i) {
            const SplitJob &J = jobs[i];
            // destination rows 16-byte aligned; source rows too unless they are padded (ld_src < ld_dst:
            // zero columns appended, scalar loads)
            const bool padded = J.ld_src < J.ld_dst;
            KFAC_CHECK_ARG(J.ld_dst % 4 == 0 && J.cols <= J.ld_dst && J.cols <= J.ld_src && aligned16(J.hi) &&
                               aligned16(J.lo) && (padded || (J.ld_src % 4 == 0 && aligned16(J.src))),
                           KFAC_ERR_ALIGNMENT, "split_planes: rows must be 16-byte aligned");
            b.j[b.count] = J;
            b.unit_begin[b.count] = units;
            units += (long long)J.rows * (J.ld_dst / 4);
            ++b.count;
        }
        b.unit_begin[b.count] = units;
        if (units == 0) continue;
        const int grid = (int)std::min<long long>((units + 255) / 256, 148 * 16);
        split_planes_kernel<<<grid, 256, 0, s>>>(b);
        KFAC_LAUNCHED();
    }
    return KFAC_OK;
}

bool syrk_tc_supported(const FactorJob &j) {
    if (j.d < 64 || j.n < 32) return false;               // small factors: SIMT tile
    if (j.c_in % 4 != 0) return false;                    // 16-byte gathers
    if (j.is_a && j.bias_col && j.patch_cols % 4 != 0) return false;
    // 32-bit element offsets in the gather
    const long long elems = j.is_a ? (long long)(j.n / ((long long)j.h_out * j.w_out)) * j.h_in * j.w_in * j.c_in
                                   : j.n * j.c_in;
    if (elems >= (1ll << 31) - 4096) return false;
    return aligned16(j.src);
}

kfac_status_t syrk_tc_partial(const FactorJob *jobs, int count, cudaStream_t s) {
    KFAC_CUDA_TRY(set_smem_attr((const void *)syrk_tc_planes8_kernel, kSmemBytes));
    for (int base = 0; base < count; base += kMaxSyrk) {
        SyrkBatch b;
        b.count = 0;
        b.drain = kDrainSyrk;
        int items = 0;
        for (int i = base; i < count && b.count < kMaxSyrk; ++i) {
            FactorJob j = jobs[i];
            j.item_begin = items;
            items += j.tiles * j.splits;
            b.j[b.count++] = j;
        }
        const int prof = prof_begin(KFAC_PROF_SYRK_TC, s);
        syrk_tc_planes8_kernel<<<items, NT2, kSmemBytes, s>>>(b);
        KFAC_LAUNCHED();
        if (prof >= 0) {
            // algorithmic work of the factors in this launch: n d (d + 1) flops (upper triangle incl.
            // diagonal); bytes: the input tensor read once + the fp32 partial tiles
            double by = 0.0, fl = 0.0;
            for (int i = 0; i < b.count; ++i) {
                const FactorJob &j = b.j[i];
                fl += (double)j.n * j.d * (j.d + 1.0);
                const double in = j.is_a ? (double)(j.n / ((long long)j.h_out * j.w_out)) * j.h_in * j.w_in * j.c_in
                                         : (double)j.n * j.c_in;
                by += 4.0 * in + 4.0 * (double)j.splits * j.tiles * BM * BN;
            }
            prof_end(prof, s, by, fl);
        }
    }
    return KFAC_OK;
}

}  // namespace kfac

// Test hook (not part of the public header): run one GEMM through a chosen engine.
// engine 0 = SIMT, 1 = tcgen05 (in-kernel split), 2 = tcgen05 on pre-split planes; | 4 selects
// the C -= AB epilogue.  Returns a kfac_status_t.
extern "C" int kfac_debug_gemm(int engine, const float *A, int lda, int trans_a, const float *B, int ldb,
                               int trans_b, float *C, int ldc, int M, int N, int K, void *stream, float *debug) {
    kfac::GemmDesc d{};
    d.A = A; d.lda = lda; d.trans_a = trans_a; d.B = B; d.ldb = ldb; d.trans_b = trans_b;
    d.C = C; d.ldc = ldc; d.M = M; d.N = N; d.K = K;
    if (engine & 4) d.epi = kfac::EPI_SUB;      // C -= op(A) op(B)
    engine &= 3;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (engine == 1) return KFAC_ERR_UNSUPPORTED;     // the in-kernel-split engine was retired
    if (engine == 2) {
        // pre-split planes engine: A, B split into TF32 planes here; with `debug` non-null the
        // result is emitted as planes too (hi -> C, lo -> debug, same leading dimension)
        if (!kfac::gemm_tc_supported(d)) return KFAC_ERR_UNSUPPORTED;
        const int ar = trans_a ? K : M, ac = trans_a ? M : K, br = trans_b ? N : K, bc = trans_b ? K : N;
        float *ap = nullptr, *bp = nullptr;
        if (cudaMalloc(&ap, sizeof(float) * 2 * (size_t)ar * lda) != cudaSuccess) return KFAC_ERR_CUDA;
        if (cudaMalloc(&bp, sizeof(float) * 2 * (size_t)br * ldb) != cudaSuccess) return KFAC_ERR_CUDA;
        kfac::SplitJob sj[2] = {{A, ap, ap + (size_t)ar * lda, ar, ac, lda, lda},
                                {B, bp, bp + (size_t)br * ldb, br, bc, ldb, ldb}};
        int st = kfac::split_planes(sj, 2, s);
        kfac::GemmDesc p = d;
        p.A = ap; p.A_lo = ap + (size_t)ar * lda;
        p.B = bp; p.B_lo = bp + (size_t)br * ldb;
        p.C_lo = debug;
        if (st == KFAC_OK) st = kfac::gemm_tc_planes_grouped(&p, 1, 0.f, s);
        cudaStreamSynchronize(s);
        cudaFree(ap);
        cudaFree(bp);
        return st;
    }
    return kfac::gemm_simt_grouped(&d, 1, 0.f, s);
}
