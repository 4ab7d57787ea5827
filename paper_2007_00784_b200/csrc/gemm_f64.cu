// gemm_f64.cu -- grouped SIMT GEMM with fp64 accumulation for the eigensolver's internal
// products (trailing rank-2k update, divide-and-conquer eigenvector updates, back-transformation).
//
// Why not the tensor cores there: the preconditioner divides by v_G v_A^T + damping, so an
// eigenvector error e along a direction of eigenvalue L is amplified by ~L/damping (5e5 for the
// ResNet-50 fc A factor); the eigenvectors must be accurate to the fp32 rounding level, while a
// 3xTF32 product carries ~2^-22 relative error per term and accumulates across ~10 chained GEMMs.
// fp64 products of fp32/fp64 operands with fp64 accumulation leave one rounding per output.
//
// 128x128 tile per CTA, 256 threads, 8x8 outputs per thread, K staged 8 at a time through shared
// memory as fp64 (operands converted once when staged), register prefetch of the next slab.
#include "internal.cuh"

#include <vector>

namespace kfac {
namespace {

constexpr int BM = 128, BN = 128, BK = 8, NT = 256;

struct Batch64 {
    int count;
    Gemm64Desc d[kGemm64MaxDescs];
};

__device__ __forceinline__ int find_desc(const Batch64 &b, int tile) {
    int lo = 0, hi = b.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (b.d[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ double ld_any(const void *p, size_t i, int dt) {
    return dt == DT_F64 ? __ldg(static_cast<const double *>(p) + i) : (double)__ldg(static_cast<const float *>(p) + i);
}

// Epilogue shared by both kernels.  Thread (ty, tx) owns rows 2 ty + {0,1} + 32 i' and columns
// 2 tx + {0,1} + 32 j'; acc[i][j] with i = 2 i' + {0,1}, j = 2 j' + {0,1}.
__device__ __forceinline__ void epilogue(const Gemm64Desc &d, int m0, int n0, int Me, int Ne, int ty, int tx,
                                         const double (&acc)[8][8]) {
    // Epilogue.  Thread columns come in adjacent pairs (2 tx + {0,1} + 32 jj), so C is accessed as
    // 8- or 16-byte pairs; for C -= AB the 16 pairs of four rows are all loaded before any is
    // used or stored (independent loads in flight instead of one dependent round trip each).
    const bool pair_ok = ((d.ldc & 1) == 0) &&
                         ((reinterpret_cast<uintptr_t>(d.C) & (d.tc == DT_F64 ? 15 : 7)) == 0);
    const bool sub = d.epi == EPI_SUB;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        double cv[4][4][2];
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
            const int i = 4 * h + ii;
            const int m = m0 + 2 * ty + (i & 1) + 32 * (i >> 1);
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int n = n0 + 2 * tx + 32 * jj;
                cv[ii][jj][0] = cv[ii][jj][1] = 0.0;
                if (!sub || m >= Me || n >= Ne) continue;
                const size_t o = (size_t)m * d.ldc + n;
                if (d.tc == DT_F64) {
                    const double *C = static_cast<const double *>(d.C);
                    if (pair_ok && n + 1 < Ne) {
                        const double2 v = __ldcg(reinterpret_cast<const double2 *>(C + o));
                        cv[ii][jj][0] = v.x; cv[ii][jj][1] = v.y;
                    } else {
                        cv[ii][jj][0] = __ldcg(C + o);
                        if (n + 1 < Ne) cv[ii][jj][1] = __ldcg(C + o + 1);
                    }
                } else {
                    const float *C = static_cast<const float *>(d.C);
                    if (pair_ok && n + 1 < Ne) {
                        const float2 v = __ldcg(reinterpret_cast<const float2 *>(C + o));
                        cv[ii][jj][0] = v.x; cv[ii][jj][1] = v.y;
                    } else {
                        cv[ii][jj][0] = __ldcg(C + o);
                        if (n + 1 < Ne) cv[ii][jj][1] = __ldcg(C + o + 1);
                    }
                }
            }
        }
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
            const int i = 4 * h + ii;
            const int m = m0 + 2 * ty + (i & 1) + 32 * (i >> 1);
            if (m >= Me) continue;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int n = n0 + 2 * tx + 32 * jj;
                if (n >= Ne) continue;
                const double r0 = sub ? cv[ii][jj][0] - acc[i][2 * jj] : acc[i][2 * jj];
                const double r1 = sub ? cv[ii][jj][1] - acc[i][2 * jj + 1] : acc[i][2 * jj + 1];
                const size_t o = (size_t)m * d.ldc + n;
                if (d.tc == DT_F64) {
                    double *C = static_cast<double *>(d.C);
                    if (pair_ok && n + 1 < Ne) {
                        *reinterpret_cast<double2 *>(C + o) = make_double2(r0, r1);
                    } else {
                        C[o] = r0;
                        if (n + 1 < Ne) C[o + 1] = r1;
                    }
                } else {
                    float *C = static_cast<float *>(d.C);
                    if (pair_ok && n + 1 < Ne) {
                        *reinterpret_cast<float2 *>(C + o) = make_float2((float)r0, (float)r1);
                    } else {
                        C[o] = (float)r0;
                        if (n + 1 < Ne) C[o + 1] = (float)r1;
                    }
                }
            }
        }
    }
}

__global__ void __launch_bounds__(NT, 1) gemm64_kernel(const __grid_constant__ Batch64 batch) {
    __shared__ __align__(16) double As[2][BK][BM + 2];
    __shared__ __align__(16) double Bs[2][BK][BN + 2];
    const int tile = blockIdx.x;
    const Gemm64Desc &d = batch.d[find_desc(batch, tile)];
    const int local = tile - d.tile_begin;
    const int tiles_n = (d.N + BN - 1) / BN;
    const int m0 = (local / tiles_n) * BM, n0 = (local % tiles_n) * BN;
    const int Me = d.M, Ne = d.dyn ? min(d.N, d.dyn[0]) : d.N, Ke = d.dyn ? min(d.K, d.dyn[1]) : d.K;
    if (n0 >= Ne) return;
    if (d.lower && n0 >= m0 + BM) return;            // block strictly above the diagonal
    const int t = threadIdx.x;

    // loader: 4 elements of each operand per thread per slab (128 x 8)
    int a_r, a_c, b_r, b_c;
    if (d.trans_a) { a_r = t / 32; a_c = (t % 32) * 4; }    // A[k][m..m+4)
    else           { a_r = t / 2;  a_c = (t % 2) * 4; }     // A[m][k..k+4)
    if (d.trans_b) { b_r = t / 2;  b_c = (t % 2) * 4; }     // B[n][k..k+4)
    else           { b_r = t / 32; b_c = (t % 32) * 4; }    // B[k][n..n+4)

    double ra[4], rb[4];
    // Each thread's 4 elements of an operand are contiguous in memory (k for a K-major operand,
    // m/n otherwise): one 16-byte (fp32) or two 16-byte (fp64) loads when the run is in bounds
    // and aligned, element loads at the edges.
    const bool a_vec = ((d.lda & 3) == 0) && ((reinterpret_cast<uintptr_t>(d.A) & 15) == 0);
    const bool b_vec = ((d.ldb & 3) == 0) && ((reinterpret_cast<uintptr_t>(d.B) & 15) == 0);
    auto load4 = [&](const void *p, size_t i0, int dt, double (&r)[4]) {
        if (dt == DT_F64) {
            const double2 x = __ldg(reinterpret_cast<const double2 *>(static_cast<const double *>(p) + i0));
            const double2 y = __ldg(reinterpret_cast<const double2 *>(static_cast<const double *>(p) + i0 + 2));
            r[0] = x.x; r[1] = x.y; r[2] = y.x; r[3] = y.y;
        } else {
            const float4 x = __ldg(reinterpret_cast<const float4 *>(static_cast<const float *>(p) + i0));
            r[0] = x.x; r[1] = x.y; r[2] = x.z; r[3] = x.w;
        }
    };
    auto load = [&](int k0) {
        {
            int m, k;
            if (d.trans_a) { k = k0 + a_r; m = m0 + a_c; }
            else           { m = m0 + a_r; k = k0 + a_c; }
            const bool full = d.trans_a ? (k < Ke && m + 3 < Me) : (m < Me && k + 3 < Ke);
            const bool fast_a = a_vec && full;
            const bool fast_b = b_vec && (d.trans_b ? (n0 + b_r < Ne && k0 + b_c + 3 < Ke)
                                                    : (k0 + b_r < Ke && n0 + b_c + 3 < Ne));
            if (fast_a && fast_b) {
                load4(d.A, d.trans_a ? (size_t)k * d.lda + m : (size_t)m * d.lda + k, d.ta, ra);
                load4(d.B, d.trans_b ? (size_t)(n0 + b_r) * d.ldb + k0 + b_c : (size_t)(k0 + b_r) * d.ldb + n0 + b_c,
                      d.tb, rb);
                return;
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int m, k;
            if (d.trans_a) { k = k0 + a_r; m = m0 + a_c + i; }
            else           { m = m0 + a_r; k = k0 + a_c + i; }
            ra[i] = (m < Me && k < Ke) ? ld_any(d.A, d.trans_a ? (size_t)k * d.lda + m : (size_t)m * d.lda + k, d.ta)
                                       : 0.0;
            int n, kb;
            if (d.trans_b) { n = n0 + b_r; kb = k0 + b_c + i; }
            else           { kb = k0 + b_r; n = n0 + b_c + i; }
            rb[i] = (n < Ne && kb < Ke) ? ld_any(d.B, d.trans_b ? (size_t)n * d.ldb + kb : (size_t)kb * d.ldb + n, d.tb)
                                        : 0.0;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (d.trans_a) As[buf][a_r][a_c + i] = ra[i];
            else           As[buf][a_c + i][a_r] = ra[i];
            if (d.trans_b) Bs[buf][b_c + i][b_r] = rb[i];
            else           Bs[buf][b_r][b_c + i] = rb[i];
        }
    };

    double acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;

    // thread (ty, tx) owns rows 2 ty + {0,1} + 32 i and columns 2 tx + {0,1} + 32 j (i, j < 4): the
    // 16-byte shared loads of a quarter-warp then cover 128 contiguous bytes (no bank conflicts)
    const int ty = t / 16, tx = t % 16;
    const int nk = (Ke + BK - 1) / BK;
    if (nk > 0) {
        load(0);
        store(0);
    }
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nk) load((kt + 1) * BK);
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            double a[8], b[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double2 av = *reinterpret_cast<const double2 *>(&As[buf][k][2 * ty + 32 * i]);
                const double2 bv = *reinterpret_cast<const double2 *>(&Bs[buf][k][2 * tx + 32 * i]);
                a[2 * i] = av.x; a[2 * i + 1] = av.y;
                b[2 * i] = bv.x; b[2 * i + 1] = bv.y;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        if (kt + 1 < nk) {
            store(buf ^ 1);
            __syncthreads();
        }
    }

    epilogue(d, m0, n0, Me, Ne, ty, tx, acc);
}

}  // namespace

kfac_status_t gemm64_grouped(const Gemm64Desc *descs, int count, cudaStream_t s) {
    for (int base = 0; base < count; base += kGemm64MaxDescs) {
        static Batch64 b;       // host staging; parameters are copied at launch
        b.count = 0;
        int tiles = 0;
        for (int i = base; i < count && b.count < kGemm64MaxDescs; ++i) {
            const Gemm64Desc &g = descs[i];
            if (g.M <= 0 || g.N <= 0) continue;
            b.d[b.count] = g;
            b.d[b.count].tile_begin = tiles;
            tiles += cdiv(g.M, BM) * cdiv(g.N, BN);
            ++b.count;
        }
        if (b.count == 0) continue;
        gemm64_kernel<<<tiles, NT, 0, s>>>(b);
        KFAC_LAUNCHED();
    }
    return KFAC_OK;
}

}  // namespace kfac

// Test hook: one fp64-accumulating GEMM; dtype codes 0 = fp32, 1 = fp64 for A, B, C;
// epi 0 = store, 3 = C -= op(A) op(B).
extern "C" int kfac_debug_gemm64(const void *A, int ta, int lda, int trans_a, const void *B, int tb, int ldb,
                                 int trans_b, void *C, int tc, int ldc, int M, int N, int K, int epi, void *stream) {
    kfac::Gemm64Desc d{};
    d.A = A; d.ta = ta; d.lda = lda; d.trans_a = trans_a;
    d.B = B; d.tb = tb; d.ldb = ldb; d.trans_b = trans_b;
    d.C = C; d.tc = tc; d.ldc = ldc;
    d.M = M; d.N = N; d.K = K; d.epi = epi;
    return kfac::gemm64_grouped(&d, 1, reinterpret_cast<cudaStream_t>(stream));
}
