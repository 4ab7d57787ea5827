// inverse.cu -- comparison variant of Stage 2: explicit damped inverse (Eq. 11):
//   (F + damping I)^{-1} = L^{-T} L^{-1},  F + damping I = L L^T  (R15),
// blocked right-looking Cholesky in FP64 (64x64 tiles), blocked triangular inversion and the
// product X = Y^T Y with Y = L^{-1}; every launch covers the same step of all factors of the
// batch.  FP64 because the explicit inverse amplifies rounding by cond(F + damping I)
// (SURVEY 8(c) numerics: fp32 inversion adds up to 4.8e-3 error on ResNet-50 layer4).
#include "internal.cuh"

#include <algorithm>
#include <vector>

namespace kfac {
namespace {

constexpr int TB = 64;          // tile
constexpr int KS = 16;          // k-slice staged in shared memory
constexpr int NT = 256;         // 16x16 threads, 4x4 outputs each
constexpr int kMaxJobs = 64;

struct InvJob {
    const float *F;
    float *Finv;
    double *M;        // nP x nP working matrix (lower triangle becomes L)
    double *Y;        // nP x nP, lower triangle becomes L^{-1}
    int *info;
    int n, ldF, ldFinv, nP, nbk;
};

struct InvBatch {
    int count;
    int step;
    float damping;
    int begin[kMaxJobs + 1];      // prefix of CTAs per job for the current launch
    InvJob j[kMaxJobs];
};

__device__ __forceinline__ int find(const InvBatch &b, int cta) {
    int lo = 0, hi = b.count - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (b.begin[mid] <= cta) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// acc(4x4 per thread) += op(A)[64 x K] * op(B)[K x 64]
//   ta = 0: A(m,k) = A[m*lda + k]   ta = 1: A(m,k) = A[k*lda + m]
//   tb = 0: B(k,n) = B[k*ldb + n]   tb = 1: B(k,n) = B[n*ldb + k]
__device__ void tile_gemm(double (&acc)[4][4], const double *A, int lda, int ta, const double *B, int ldb,
                          int tb, int K) {
    __shared__ double As[KS][TB + 1];
    __shared__ double Bs[KS][TB + 1];
    const int t = threadIdx.x, ty = t / 16, tx = t % 16;
    for (int k0 = 0; k0 < K; k0 += KS) {
        for (int e = t; e < KS * TB; e += NT) {          // coalesced along the contiguous index
            const int kk = e / TB, mm = e % TB;
            const int mt = e / KS, kt = e % KS;
            As[ta ? kk : kt][ta ? mm : mt] = ta ? A[(size_t)(k0 + kk) * lda + mm] : A[(size_t)mt * lda + k0 + kt];
            Bs[tb ? kt : kk][tb ? mt : mm] = tb ? B[(size_t)mt * ldb + k0 + kt] : B[(size_t)(k0 + kk) * ldb + mm];
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < KS; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty + 16 * i]; b[i] = Bs[kk][tx + 16 * i]; }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int jx = 0; jx < 4; ++jx) acc[i][jx] = fma(a[i], b[jx], acc[i][jx]);
        }
        __syncthreads();
    }
}

__device__ __forceinline__ double *tile(double *M, int nP, int bi, int bj) {
    return M + (size_t)bi * TB * nP + (size_t)bj * TB;
}

// M = sym(F) + damping I (fp64), padded with identity; Y = 0.
__global__ void inv_init(const __grid_constant__ InvBatch b) {
    const InvJob &J = b.j[blockIdx.y];
    const long long total = (long long)J.nP * J.nP;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(e / J.nP), c = (int)(e % J.nP);
        double v = 0.0;
        if (r < J.n && c < J.n)
            v = 0.5 * ((double)J.F[(size_t)r * J.ldF + c] + (double)J.F[(size_t)c * J.ldF + r]);
        if (r == c) v += (r < J.n) ? (double)b.damping : 1.0;
        J.M[e] = v;
        J.Y[e] = 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && J.info) *J.info = 0;
}

// Step k (a): factor the diagonal tile in shared memory; write L_kk and Y_kk = L_kk^{-1}.
constexpr size_t kPotrfSmem = 2 * sizeof(double) * TB * (TB + 1);
constexpr size_t kTrtriSmem = sizeof(double) * TB * (TB + 1);

__global__ void __launch_bounds__(NT) inv_potrf(const __grid_constant__ InvBatch b) {
    extern __shared__ double dyn[];
    double(*S)[TB + 1] = reinterpret_cast<double(*)[TB + 1]>(dyn);
    double(*Li)[TB + 1] = reinterpret_cast<double(*)[TB + 1]>(dyn + TB * (TB + 1));
    const InvJob &J = b.j[find(b, blockIdx.x)];
    const int k = b.step;
    double *D = tile(J.M, J.nP, k, k);
    const int t = threadIdx.x;
    for (int e = t; e < TB * TB; e += NT) S[e / TB][e % TB] = D[(size_t)(e / TB) * J.nP + e % TB];
    __syncthreads();
    __shared__ int bad;
    if (t == 0) bad = 0;
    __syncthreads();
    for (int j = 0; j < TB; ++j) {                  // left-looking column j (unblocked, in smem)
        if (t == 0) {
            double s = S[j][j];
            if (!(s > 0.0)) {
                if (!bad && J.info && *J.info == 0) *J.info = k * TB + j + 1;
                bad = 1;
                s = 1.0;
            }
            S[j][j] = sqrt(s);
        }
        __syncthreads();
        const double ljj = S[j][j];
        for (int i = j + 1 + t; i < TB; i += NT) S[i][j] /= ljj;
        __syncthreads();
        for (int e = t; e < (TB - j - 1) * (TB - j - 1); e += NT) {   // trailing update (lower part)
            const int i = j + 1 + e / (TB - j - 1), c = j + 1 + e % (TB - j - 1);
            if (c <= i) S[i][c] -= S[i][j] * S[c][j];
        }
        __syncthreads();
    }
    // Li = L^{-1} (lower): column by column forward substitution, one thread per column.
    for (int e = t; e < TB * TB; e += NT) Li[e / TB][e % TB] = 0.0;
    __syncthreads();
    if (t < TB) {
        const int c = t;
        for (int i = c; i < TB; ++i) {
            double v = (i == c) ? 1.0 : 0.0;
            for (int m = c; m < i; ++m) v -= S[i][m] * Li[m][c];
            Li[i][c] = v / S[i][i];
        }
    }
    __syncthreads();
    double *Yd = tile(J.Y, J.nP, k, k);
    for (int e = t; e < TB * TB; e += NT) {
        const int r = e / TB, c = e % TB;
        D[(size_t)r * J.nP + c] = c <= r ? S[r][c] : 0.0;
        Yd[(size_t)r * J.nP + c] = Li[r][c];
    }
}

// Step k (b): L_ik = A_ik L_kk^{-T} for i > k (one CTA per row tile).
__global__ void __launch_bounds__(NT) inv_trsm(const __grid_constant__ InvBatch b) {
    const int ji = find(b, blockIdx.x);
    const InvJob &J = b.j[ji];
    const int k = b.step;
    const int i = k + 1 + (blockIdx.x - b.begin[ji]);
    double acc[4][4] = {};
    double *Aik = tile(J.M, J.nP, i, k);
    // acc = A_ik * (L_kk^{-1})^T : B(kk, n) = Y_kk[n][kk] -> tb = 1
    tile_gemm(acc, Aik, J.nP, 0, tile(J.Y, J.nP, k, k), J.nP, 1, TB);
    const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) Aik[(size_t)(ty + 16 * a) * J.nP + tx + 16 * c] = acc[a][c];
}

// Step k (c): A_ij -= L_ik L_jk^T for i >= j > k (lower tiles).
__global__ void __launch_bounds__(NT) inv_update(const __grid_constant__ InvBatch b) {
    const int ji = find(b, blockIdx.x);
    const InvJob &J = b.j[ji];
    const int k = b.step;
    int e = blockIdx.x - b.begin[ji];
    int i = k + 1, j;
    while (e >= i - k) { e -= i - k; ++i; }      // tile rows i = k+1.., cols j = k+1..i
    j = k + 1 + e;
    double acc[4][4] = {};
    tile_gemm(acc, tile(J.M, J.nP, i, k), J.nP, 0, tile(J.M, J.nP, j, k), J.nP, 1, TB);
    double *Aij = tile(J.M, J.nP, i, j);
    const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) Aij[(size_t)(ty + 16 * a) * J.nP + tx + 16 * c] -= acc[a][c];
}

// Triangular inverse, row tile i: Y_ij = -Y_ii sum_{m=j}^{i-1} L_im Y_mj for j < i.
__global__ void __launch_bounds__(NT) inv_trtri(const __grid_constant__ InvBatch b) {
    extern __shared__ double dyn[];
    double(*Sacc)[TB + 1] = reinterpret_cast<double(*)[TB + 1]>(dyn);
    const int ji = find(b, blockIdx.x);
    const InvJob &J = b.j[ji];
    const int i = b.step;
    const int j = blockIdx.x - b.begin[ji];
    double acc[4][4] = {};
    for (int m = j; m < i; ++m)
        tile_gemm(acc, tile(J.M, J.nP, i, m), J.nP, 0, tile(J.Y, J.nP, m, j), J.nP, 0, TB);
    const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) Sacc[ty + 16 * a][tx + 16 * c] = acc[a][c];
    __syncthreads();
    const double *Yii = tile(J.Y, J.nP, i, i);
    double *Yij = tile(J.Y, J.nP, i, j);
    for (int e = threadIdx.x; e < TB * TB; e += NT) {
        const int r = e / TB, c = e % TB;
        double v = 0.0;
        for (int m = 0; m <= r; ++m) v -= Yii[(size_t)r * J.nP + m] * Sacc[m][c];
        Yij[(size_t)r * J.nP + c] = v;
    }
}

// X_ij = sum_{m >= max(i,j)} Y_mi^T Y_mj  for i >= j; writes X_ij and X_ji (fp32 output).
__global__ void __launch_bounds__(NT) inv_gram(const __grid_constant__ InvBatch b) {
    const int ji = find(b, blockIdx.x);
    const InvJob &J = b.j[ji];
    int e = blockIdx.x - b.begin[ji];
    int i = 0;
    while (e >= i + 1) { e -= i + 1; ++i; }
    const int j = e;
    double acc[4][4] = {};
    for (int m = i; m < J.nbk; ++m)
        tile_gemm(acc, tile(J.Y, J.nP, m, i), J.nP, 1, tile(J.Y, J.nP, m, j), J.nP, 0, TB);
    const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int r = i * TB + ty + 16 * a, col = j * TB + tx + 16 * c;
            if (r < J.n && col < J.n) {
                J.Finv[(size_t)r * J.ldFinv + col] = (float)acc[a][c];
                J.Finv[(size_t)col * J.ldFinv + r] = (float)acc[a][c];
            }
        }
}

struct Plan {
    std::vector<InvJob> jobs;
    size_t bytes = 0;
};

Plan plan(const int32_t *dims, int count) {
    Plan p;
    size_t off = 0;
    for (int i = 0; i < count; ++i) {
        InvJob J{};
        J.n = dims[i];
        J.nP = (int)round_up(J.n, TB);
        J.nbk = J.nP / TB;
        off = round_up(off, 256);
        J.M = reinterpret_cast<double *>(off);
        off += sizeof(double) * (size_t)J.nP * J.nP;
        off = round_up(off, 256);
        J.Y = reinterpret_cast<double *>(off);
        off += sizeof(double) * (size_t)J.nP * J.nP;
        p.jobs.push_back(J);
    }
    p.bytes = off + 256;
    return p;
}

}  // namespace

size_t inverse_workspace_bytes(const int32_t *dims, int count) { return plan(dims, count).bytes; }

kfac_status_t inverse_run(const float *const *F, const int32_t *dims, const int32_t *ldF, int count,
                          float damping, float *const *Finv, const int32_t *ldFinv, int32_t *info,
                          void *ws, cudaStream_t s) {
    KFAC_CUDA_TRY(set_smem_attr((const void *)inv_potrf, (int)kPotrfSmem));
    KFAC_CUDA_TRY(set_smem_attr((const void *)inv_trtri, (int)kTrtriSmem));
    Plan p = plan(dims, count);
    char *base = reinterpret_cast<char *>(round_up(reinterpret_cast<uintptr_t>(ws), 256));
    for (int i = 0; i < count; ++i) {
        InvJob &J = p.jobs[i];
        J.F = F[i]; J.Finv = Finv[i]; J.ldF = ldF[i]; J.ldFinv = ldFinv[i];
        J.info = info ? info + i : nullptr;
        J.M = reinterpret_cast<double *>(base + reinterpret_cast<uintptr_t>(J.M));
        J.Y = reinterpret_cast<double *>(base + reinterpret_cast<uintptr_t>(J.Y));
    }
    for (int b0 = 0; b0 < count; b0 += kMaxJobs) {
        InvBatch B;
        B.count = std::min(kMaxJobs, count - b0);
        B.damping = damping;
        int max_nbk = 0, max_np = 0;
        for (int i = 0; i < B.count; ++i) {
            B.j[i] = p.jobs[b0 + i];
            max_nbk = std::max(max_nbk, B.j[i].nbk);
            max_np = std::max(max_np, B.j[i].nP);
        }
        B.step = 0;
        inv_init<<<dim3(std::min(1024, cdiv((long long)max_np * max_np, NT)), B.count), NT, 0, s>>>(B);
        KFAC_LAUNCHED();
        // launch helper: per-job CTA counts -> prefix
        auto launch = [&](void (*kern)(InvBatch), size_t smem, auto ctas_of) -> kfac_status_t {
            int total = 0;
            for (int i = 0; i < B.count; ++i) {
                B.begin[i] = total;
                total += ctas_of(B.j[i]);
            }
            B.begin[B.count] = total;
            if (total == 0) return KFAC_OK;
            kern<<<total, NT, smem, s>>>(B);
            KFAC_LAUNCHED();
            return KFAC_OK;
        };
        // Jobs with no work in a step get zero CTAs; find() skips them because their begin equals
        // the next job's begin (binary search returns the last job with begin <= cta).
        for (int k = 0; k < max_nbk; ++k) {
            B.step = k;
            kfac_status_t st;
            if ((st = launch(inv_potrf, kPotrfSmem, [&](const InvJob &J) { return k < J.nbk ? 1 : 0; })) != KFAC_OK) return st;
            if ((st = launch(inv_trsm, 0, [&](const InvJob &J) { return k < J.nbk ? J.nbk - k - 1 : 0; })) != KFAC_OK) return st;
            if ((st = launch(inv_update, 0, [&](const InvJob &J) {
                     const int r = k < J.nbk ? J.nbk - k - 1 : 0;
                     return r * (r + 1) / 2;
                 })) != KFAC_OK)
                return st;
        }
        for (int i = 1; i < max_nbk; ++i) {
            B.step = i;
            kfac_status_t st = launch(inv_trtri, kTrtriSmem, [&](const InvJob &J) { return i < J.nbk ? i : 0; });
            if (st != KFAC_OK) return st;
        }
        kfac_status_t st = launch(inv_gram, 0, [&](const InvJob &J) { return J.nbk * (J.nbk + 1) / 2; });
        if (st != KFAC_OK) return st;
    }
    return KFAC_OK;
}

}  // namespace kfac
