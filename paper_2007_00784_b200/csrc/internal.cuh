// internal.cuh -- launchers shared between the libkfac translation units.
#pragma once

#include "common.cuh"

namespace kfac {

// ----------------------------------------------------------- grouped GEMM --
// C = op(A) op(B) (+ epilogue), fp32 in/out.  op(A) is M x K, op(B) is K x N.
//   trans_a = 0: A[m*lda + k]   trans_a = 1: A[k*lda + m]
//   trans_b = 0: B[k*ldb + n]   trans_b = 1: B[n*ldb + k]
enum GemmEpi : int {
    EPI_STORE = 0,
    EPI_DIV_EIGEN = 1,      // C /= max(vr[m]*vc[n] + damping, 1e-12)        (Eq. 14)
    EPI_DIV_FACTORED = 2,   // C /= max((vr[m]+damping)*(vc[n]+damping), 1e-12)
    EPI_SUB = 3,            // C = C_in - op(A) op(B)   (symmetric rank-2k update, back-transform)
};

__host__ __device__ inline bool epi_uses_vectors(int epi) { return epi == EPI_DIV_EIGEN || epi == EPI_DIV_FACTORED; }

struct GemmDesc {
    const float *A;
    const float *B;
    float *C;
    const float *vr;
    const float *vc;
    int M, N, K;
    int lda, ldb, ldc;
    int trans_a, trans_b, epi;
    int tile_begin;          // filled by the launcher
    const int *dyn;          // optional device {N_eff, K_eff}: the kernel clips N and K to them
    int lower;               // tensor-core engine: skip 128x128 tiles strictly above the diagonal
    // Pre-split operands (tensor-core "planes" engine, gemm_tc_planes_grouped): A/B are the TF32
    // hi planes and A_lo/B_lo the lo planes (x = hi + lo, both exact TF32 values); C_lo non-null
    // makes the epilogue write its result as planes too (C = hi, C_lo = lo).
    const float *A_lo, *B_lo;
    float *C_lo;
};

constexpr int kGemmMaxDescs = 64;

struct GemmBatch {
    int count;
    int tiles_total;
    float damping;
    GemmDesc d[kGemmMaxDescs];
};

// SIMT fp32 grouped GEMM (any shape/transposition); used for small/ragged
// problems and as the numerics baseline of the tensor-core path.
kfac_status_t gemm_simt_grouped(const GemmDesc *descs, int count, float damping, cudaStream_t s);

// Tensor-core (tcgen05, kind::tf32, 3xTF32) grouped GEMM.  Returns
// KFAC_ERR_UNSUPPORTED if a descriptor does not meet its layout rules.
kfac_status_t gemm_tc_grouped(const GemmDesc *descs, int count, float damping, cudaStream_t s);
bool gemm_tc_supported(const GemmDesc &d);

// Tensor-core engine on pre-split TF32 operand planes: TMA loads hi and lo tiles, no split pass.
kfac_status_t gemm_tc_planes_grouped(const GemmDesc *descs, int count, float damping, cudaStream_t s);
// x -> (hi, lo) TF32 planes of a rows x cols matrix (ld_src / ld_dst in floats, multiples of 4).
struct SplitJob {
    const float *src;
    float *hi, *lo;
    int rows, cols, ld_src, ld_dst;
};
kfac_status_t split_planes(const SplitJob *jobs, int count, cudaStream_t s);

// Dispatch each descriptor to the tensor-core or SIMT engine.
kfac_status_t gemm_grouped(const GemmDesc *descs, int count, float damping, cudaStream_t s);

// fp64-accumulating SIMT grouped GEMM (eigensolver internals, gemm_f64.cu):
// C (dtype tc) = op(A) op(B)  or  C -= op(A) op(B)  (epi EPI_SUB), operands fp32 or fp64.
enum DType : int { DT_F32 = 0, DT_F64 = 1 };
struct Gemm64Desc {
    const void *A;
    const void *B;
    void *C;
    const int *dyn;          // optional device {N_eff, K_eff} (+ K start with dyn_koff)
    int dyn_koff;            // dyn[2]: first K index with nonzero products (kernels may ignore it)
    int ta, tb, tc;          // DType of A, B, C
    int M, N, K;
    int lda, ldb, ldc;
    int trans_a, trans_b, epi;
    int lower;               // skip 128x128 tiles strictly above the diagonal
    int tile_begin;          // filled by the launcher
};
constexpr int kGemm64MaxDescs = 256;
kfac_status_t gemm64_grouped(const Gemm64Desc *descs, int count, cudaStream_t s);

// fp64-accurate GEMM on the int8 tensor cores (Ozaki scheme, gemm_ozaki.cu).  gemm64_grouped routes
// the eligible descriptors (fp64 operands, M >= 128, N >= 64, K >= 256) there while a scratch arena
// is set on the calling thread (oz_set_arena; the eigensolver carves it from its workspace).
bool oz_eligible(const Gemm64Desc &g);
size_t oz_scratch_bytes(const Gemm64Desc &g);
void oz_set_arena(void *base, size_t bytes);
bool oz_arena_active();
kfac_status_t oz_gemm_grouped(const Gemm64Desc *descs, int count, cudaStream_t s);

// ------------------------------------------------------------ factor SYRK --
// One Kronecker factor of one layer: F_batch = X^T X / n over the n rows of X, where X is
// [im2col(act) | 1] (A factor, Eq. 5) or the output gradients (G factor).  The upper 128x128
// tiles of X^T X are computed per row chunk into `partial` ([splits][tiles][128*128]) and
// reduced by syrk_reduce (fixed order, running average, both triangles).
struct FactorJob {
    const float *src;       // act (NHWC) for A, gout (n x c_in) for G
    const float *src_lo;    // tensor-core path: src is the TF32 hi plane, src_lo the lo plane
    float *F;
    float *packed;          // nullable: upper triangle, row-major, d(d+1)/2 floats
    float *partial;
    long long n;            // rows
    int ldF, d, is_a;
    int splits, chunk, t1d, tiles, item_begin, tile_begin;
    int c_in, h_in, w_in, h_out, w_out, k_w, stride_h, stride_w, pad_h, pad_w;  // G: c_in = row length
    int patch_cols, bias_col;
    // Row length not a multiple of 4 (e.g. ResNet conv1, C_in = 3): the tensor-core SYRK runs on a
    // copy padded with zero channels to c_in (multiple of 4) -- d, t1d, tiles, c_in and patch_cols
    // above describe that padded geometry -- and the fold maps the real factor's columns into it.
    int c_real;             // real row length / channel count (0: no padding)
    int d_out, t1d_out, tiles_out;   // geometry of the real factor F (== d, t1d, tiles unpadded)
};

// Tensor-core (tcgen05 3xTF32) partial SYRK for the jobs it supports (row length % 4 == 0).
bool syrk_tc_supported(const FactorJob &j);
kfac_status_t syrk_tc_partial(const FactorJob *jobs, int count, cudaStream_t s);

}  // namespace kfac
