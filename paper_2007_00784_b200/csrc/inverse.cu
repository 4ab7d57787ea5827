// inverse.cu -- comparison variant of Stage 2: explicit damped inverse (Eq. 11):
//   (F + damping I)^{-1} = L^{-T} L^{-1},  F + damping I = L L^T  (R15),
// blocked right-looking Cholesky in FP64 (64x64 tiles), blocked triangular inversion and the
// product X = Y^T Y with Y = L^{-1}; every launch covers the same step of all factors of the
// batch.  The 64x64 diagonal factorisations and panel solves are SIMT kernels; the O(n^3) parts --
// the trailing rank-64 updates, the triangular-inverse row products and the Gram product -- are
// grouped fp64 GEMMs (gemm64_grouped: DMMA, or the int8 Ozaki engine for the large ones).  FP64 because the explicit inverse amplifies rounding by cond(F + damping I)
// (SURVEY 8(c) numerics: fp32 inversion adds up to 4.8e-3 error on ResNet-50 layer4).
#include "internal.cuh"

#include <algorithm>
#include <vector>

namespace kfac {
namespace {

#define RET_OK_INV(x)                       \
    do {                                    \
        kfac_status_t _st = (x);            \
        if (_st != KFAC_OK) return _st;     \
    } while (0)

constexpr int TB = 64;          // tile
constexpr int KS = 16;          // k-slice staged in shared memory
constexpr int NT = 256;         // 16x16 threads, 4x4 outputs each
constexpr int kMaxJobs = 64;

struct InvJob {
    const float *F;
    float *Finv;
    double *M;        // nP x nP working matrix (lower triangle becomes L)
    double *Y;        // nP x nP, lower triangle becomes L^{-1}
    double *W;        // 64 x nP scratch of the triangular inverse
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

__host__ __device__ __forceinline__ double *tile(double *M, int nP, int bi, int bj) {
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

// Finv[j][i] = Finv[i][j] for j < i (the Gram GEMM writes the lower triangle; mirrored so the
// output is exactly symmetric).  32 x 32 tiles through shared memory.
__global__ void __launch_bounds__(256) inv_mirror(const __grid_constant__ InvBatch b) {
    __shared__ float tr[32][33];
    const InvJob &J = b.j[find(b, blockIdx.x)];
    int t = blockIdx.x - b.begin[find(b, blockIdx.x)], ti = 0;
    const int nt = (J.n + 31) / 32;
    while (t >= ti + 1) { t -= ti + 1; ++ti; }           // lower tiles (ti >= tj), row-major
    const int tj = t;
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
    (void)nt;
    for (int rr = ty; rr < 32; rr += 8) {
        const int gi = ti * 32 + rr, gj = tj * 32 + tx;
        tr[rr][tx] = (gi < J.n && gj < J.n && gj <= gi) ? J.Finv[(size_t)gi * J.ldFinv + gj] : 0.f;
    }
    __syncthreads();
    for (int rr = ty; rr < 32; rr += 8) {
        const int gi = tj * 32 + rr, gj = ti * 32 + tx;    // upper element (gi < gj) <- lower (gj, gi)
        if (gi < J.n && gj < J.n && gi < gj) J.Finv[(size_t)gi * J.ldFinv + gj] = tr[tx][rr];
    }
}

struct Plan {
    std::vector<InvJob> jobs;
    size_t bytes = 0, oz_off = 0, oz_bytes = 0;
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
        off = round_up(off, 256);
        J.W = reinterpret_cast<double *>(off);
        off += sizeof(double) * (size_t)TB * J.nP;
        p.jobs.push_back(J);
        // Ozaki scratch of the largest grouped GEMM (the Gram product Y^T Y, n x n x n)
        p.oz_bytes += 12 * (size_t)(J.nP + 64) * J.nP + (1 << 20);
    }
    off = round_up(off, 256);
    p.oz_off = off;
    off += p.oz_bytes;
    p.bytes = off + 256;
    return p;
}

}  // namespace

size_t inverse_workspace_bytes(const int32_t *dims, int count) { return plan(dims, count).bytes; }

kfac_status_t inverse_run(const float *const *F, const int32_t *dims, const int32_t *ldF, int count,
                          float damping, float *const *Finv, const int32_t *ldFinv, int32_t *info,
                          void *ws, cudaStream_t s) {
    KFAC_CUDA_TRY(set_smem_attr((const void *)inv_potrf, (int)kPotrfSmem));
    Plan p = plan(dims, count);
    char *base = reinterpret_cast<char *>(round_up(reinterpret_cast<uintptr_t>(ws), 256));
    for (int i = 0; i < count; ++i) {
        InvJob &J = p.jobs[i];
        J.F = F[i]; J.Finv = Finv[i]; J.ldF = ldF[i]; J.ldFinv = ldFinv[i];
        J.info = info ? info + i : nullptr;
        J.M = reinterpret_cast<double *>(base + reinterpret_cast<uintptr_t>(J.M));
        J.Y = reinterpret_cast<double *>(base + reinterpret_cast<uintptr_t>(J.Y));
        J.W = reinterpret_cast<double *>(base + reinterpret_cast<uintptr_t>(J.W));
    }
    struct ArenaGuard {
        ArenaGuard(void *q, size_t b) { oz_set_arena(q, b); }
        ~ArenaGuard() { oz_set_arena(nullptr, 0); }
    } arena_guard(base + p.oz_off, p.oz_bytes);
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
            // trailing update A22 -= L21 L21^T (lower tiles; K = 64)
            std::vector<Gemm64Desc> gd;
            for (int i = 0; i < B.count; ++i) {
                const InvJob &J = B.j[i];
                const int r = J.nbk - k - 1;
                if (r <= 0) continue;
                Gemm64Desc g{};
                g.M = g.N = r * TB; g.K = TB;
                g.A = tile(J.M, J.nP, k + 1, k); g.ta = DT_F64; g.lda = J.nP;
                g.B = tile(J.M, J.nP, k + 1, k); g.tb = DT_F64; g.ldb = J.nP; g.trans_b = 1;
                g.C = tile(J.M, J.nP, k + 1, k + 1); g.tc = DT_F64; g.ldc = J.nP;
                g.epi = EPI_SUB;
                g.lower = 1;
                gd.push_back(g);
            }
            if (!gd.empty()) RET_OK_INV(gemm64_grouped(gd.data(), (int)gd.size(), s));
        }
        // triangular inverse Y = L^{-1}, row tile i: W = L[i, 0:i) Y[0:i, 0:i);  Y[i, 0:i) = -Y_ii W
        for (int i = 1; i < max_nbk; ++i) {
            std::vector<Gemm64Desc> g1, g2;
            for (int q = 0; q < B.count; ++q) {
                const InvJob &J = B.j[q];
                if (i >= J.nbk) continue;
                Gemm64Desc a{};
                a.M = TB; a.N = i * TB; a.K = i * TB;
                a.A = tile(J.M, J.nP, i, 0); a.ta = DT_F64; a.lda = J.nP;
                a.B = J.Y; a.tb = DT_F64; a.ldb = J.nP;
                a.C = J.W; a.tc = DT_F64; a.ldc = J.nP;
                g1.push_back(a);
                Gemm64Desc c{};
                c.M = TB; c.N = i * TB; c.K = TB;
                c.A = tile(J.Y, J.nP, i, i); c.ta = DT_F64; c.lda = J.nP;
                c.B = J.W; c.tb = DT_F64; c.ldb = J.nP;
                c.C = tile(J.Y, J.nP, i, 0); c.tc = DT_F64; c.ldc = J.nP;
                c.epi = EPI_SUB;                    // Y[i, 0:i) is zero: 0 - Y_ii W
                g2.push_back(c);
            }
            if (g1.empty()) continue;
            RET_OK_INV(gemm64_grouped(g1.data(), (int)g1.size(), s));
            RET_OK_INV(gemm64_grouped(g2.data(), (int)g2.size(), s));
        }
        // Gram product X = Y^T Y (lower triangle, fp32 out), then mirrored
        std::vector<Gemm64Desc> gg;
        for (int q = 0; q < B.count; ++q) {
            const InvJob &J = B.j[q];
            Gemm64Desc g{};
            g.M = g.N = J.n; g.K = J.n;
            g.A = J.Y; g.ta = DT_F64; g.lda = J.nP; g.trans_a = 1;
            g.B = J.Y; g.tb = DT_F64; g.ldb = J.nP;
            g.C = J.Finv; g.tc = DT_F32; g.ldc = J.ldFinv;
            g.lower = 1;
            gg.push_back(g);
        }
        RET_OK_INV(gemm64_grouped(gg.data(), (int)gg.size(), s));
        kfac_status_t st = launch(inv_mirror, 0, [&](const InvJob &J) {
            const int nt = (J.n + 31) / 32;
            return nt * (nt + 1) / 2;
        });
        if (st != KFAC_OK) return st;
    }
    return KFAC_OK;
}

}  // namespace kfac
