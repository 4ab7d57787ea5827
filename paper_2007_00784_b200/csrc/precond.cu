// precond.cu -- Stage 3 of Alg. 1 and Eq. 18's KL-clip.
//
// Preconditioning, per layer, as a chain of grouped GEMMs over all layers (Eq. 4: layers are
// independent blocks):
//   T  = Q_G^T grad                      (Eq. 13, first product)
//   V2 = (T Q_A) / (v_G v_A^T + damping)  (Eq. 13 second product, Eq. 14 fused in the epilogue)
//   U  = Q_G V2                          (Eq. 15)
//   P  = U Q_A^T                         (Eq. 15)
// Explicit-inverse variant (Eq. 12): T = G_inv grad, P = T A_inv.
//
// KL-clip: s = sum_l |<P_l, grad_l>| with fp64 per-CTA partial sums reduced in a fixed order
// by the last CTA (deterministic), nu computed on the device, then P *= nu (float4).
#include "internal.cuh"

#include <vector>

namespace kfac {

size_t precond_workspace_bytes(const int32_t *d_g, const int32_t *d_a, int nl, int mode) {
    size_t f = 0;
    for (int l = 0; l < nl; ++l) f += 2 * round_up((size_t)d_g[l] * round_up(d_a[l], 4), 64);
    (void)mode;
    return f * sizeof(float) + 256;
}

kfac_status_t precond_run(const int32_t *d_g, const int32_t *d_a, int nl, const float *const *grad,
                          const int32_t *ldW, const float *const *QG, const int32_t *ldQG,
                          const float *const *vG, const float *const *QA, const int32_t *ldQA,
                          const float *const *vA, float damping, int mode, float *const *out,
                          void *ws, cudaStream_t s) {
    float *base = reinterpret_cast<float *>(round_up(reinterpret_cast<uintptr_t>(ws), 256));
    std::vector<float *> T(nl), V(nl);
    std::vector<int> ldt(nl);
    size_t off = 0;
    for (int l = 0; l < nl; ++l) {
        ldt[l] = (int)round_up(d_a[l], 4);
        T[l] = base + off;
        off += round_up((size_t)d_g[l] * ldt[l], 64);
        V[l] = base + off;
        off += round_up((size_t)d_g[l] * ldt[l], 64);
    }
    std::vector<GemmDesc> g(nl);
    auto run = [&]() { return gemm_grouped(g.data(), nl, damping, s); };
    kfac_status_t st;
    if (mode == KFAC_PRECOND_INVERSE) {
        for (int l = 0; l < nl; ++l) {      // T = G_inv grad
            GemmDesc d{};
            d.A = QG[l]; d.lda = ldQG[l]; d.B = grad[l]; d.ldb = ldW[l]; d.C = T[l]; d.ldc = ldt[l];
            d.M = d_g[l]; d.N = d_a[l]; d.K = d_g[l];
            g[l] = d;
        }
        if ((st = run()) != KFAC_OK) return st;
        for (int l = 0; l < nl; ++l) {      // P = T A_inv
            GemmDesc d{};
            d.A = T[l]; d.lda = ldt[l]; d.B = QA[l]; d.ldb = ldQA[l]; d.C = out[l]; d.ldc = ldW[l];
            d.M = d_g[l]; d.N = d_a[l]; d.K = d_a[l];
            g[l] = d;
        }
        return run();
    }
    for (int l = 0; l < nl; ++l) {          // T = Q_G^T grad
        GemmDesc d{};
        d.A = QG[l]; d.lda = ldQG[l]; d.trans_a = 1; d.B = grad[l]; d.ldb = ldW[l];
        d.C = T[l]; d.ldc = ldt[l]; d.M = d_g[l]; d.N = d_a[l]; d.K = d_g[l];
        g[l] = d;
    }
    if ((st = run()) != KFAC_OK) return st;
    for (int l = 0; l < nl; ++l) {          // V2 = (T Q_A) / D
        GemmDesc d{};
        d.A = T[l]; d.lda = ldt[l]; d.B = QA[l]; d.ldb = ldQA[l]; d.C = V[l]; d.ldc = ldt[l];
        d.M = d_g[l]; d.N = d_a[l]; d.K = d_a[l];
        d.epi = mode == KFAC_PRECOND_EIGEN ? EPI_DIV_EIGEN : EPI_DIV_FACTORED;
        d.vr = vG[l]; d.vc = vA[l];
        g[l] = d;
    }
    if ((st = run()) != KFAC_OK) return st;
    for (int l = 0; l < nl; ++l) {          // U = Q_G V2
        GemmDesc d{};
        d.A = QG[l]; d.lda = ldQG[l]; d.B = V[l]; d.ldb = ldt[l]; d.C = T[l]; d.ldc = ldt[l];
        d.M = d_g[l]; d.N = d_a[l]; d.K = d_g[l];
        g[l] = d;
    }
    if ((st = run()) != KFAC_OK) return st;
    for (int l = 0; l < nl; ++l) {          // P = U Q_A^T
        GemmDesc d{};
        d.A = T[l]; d.lda = ldt[l]; d.B = QA[l]; d.ldb = ldQA[l]; d.trans_b = 1;
        d.C = out[l]; d.ldc = ldW[l]; d.M = d_g[l]; d.N = d_a[l]; d.K = d_a[l];
        g[l] = d;
    }
    return run();
}

// ------------------------------------------------------------------ KL-clip --
namespace {

constexpr int kKlMax = 128;
constexpr int kKlThreads = 256;
constexpr int kKlRowsPerCta = 8;     // rows of one layer per CTA in the dot pass

struct KlLayer {
    float *P;
    const float *W;
    int rows, cols, ld, cta_begin;
};

struct KlBatch {
    int count, ctas_total;
    float lr, kappa;
    double *partial;        // [ctas_total]
    unsigned int *counter;  // last-CTA ticket
    float *nu_ws;           // nu for the scale pass
    float *nu_out;
    double *s_out;
    KlLayer l[kKlMax];
};

__device__ __forceinline__ int find_layer(const KlBatch &b, int cta) {
    int lo = 0, hi = b.count - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (b.l[mid].cta_begin <= cta) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double red[kKlThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x < 32) {
        s = threadIdx.x < kKlThreads / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    return s;   // valid in thread 0
}

__global__ void __launch_bounds__(kKlThreads) kl_dot_kernel(const __grid_constant__ KlBatch b) {
    const int cta = blockIdx.x;
    const int li = find_layer(b, cta);
    const KlLayer &L = b.l[li];
    const int r0 = (cta - L.cta_begin) * kKlRowsPerCta;
    const int r1 = min(L.rows, r0 + kKlRowsPerCta);
    double acc = 0.0;
    if ((L.cols & 3) == 0) {
        const int c4 = L.cols / 4;
        for (int e = threadIdx.x; e < (r1 - r0) * c4; e += kKlThreads) {
            const int r = r0 + e / c4, c = (e % c4) * 4;
            const float4 p = *reinterpret_cast<const float4 *>(L.P + (size_t)r * L.ld + c);
            const float4 w = __ldg(reinterpret_cast<const float4 *>(L.W + (size_t)r * L.ld + c));
            acc += (double)(p.x * w.x) + (double)(p.y * w.y) + (double)(p.z * w.z) + (double)(p.w * w.w);
        }
    } else {
        for (int e = threadIdx.x; e < (r1 - r0) * L.cols; e += kKlThreads) {
            const int r = r0 + e / L.cols, c = e % L.cols;
            acc += (double)(L.P[(size_t)r * L.ld + c] * __ldg(L.W + (size_t)r * L.ld + c));
        }
    }
    const double s = block_sum(acc);
    __shared__ bool last;
    if (threadIdx.x == 0) {
        b.partial[cta] = s;
        __threadfence();
        last = atomicAdd(b.counter, 1u) == (unsigned)(b.ctas_total - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // Last CTA: per-layer sums in a fixed order (strided per thread + fixed tree), then
    // s = sum_l |dot_l| (R12) and nu (Eq. 18).
    double total = 0.0;
    for (int l = 0; l < b.count; ++l) {
        const int beg = b.l[l].cta_begin;
        const int end = l + 1 < b.count ? b.l[l + 1].cta_begin : b.ctas_total;
        double part = 0.0;
        for (int c = beg + threadIdx.x; c < end; c += kKlThreads) part += ((volatile double *)b.partial)[c];
        const double dot = block_sum(part);
        total += fabs(dot);                 // meaningful in thread 0 only
    }
    if (threadIdx.x == 0) {
        double nu = 1.0;
        if (total > 0.0) nu = fmin(1.0, sqrt((double)b.kappa / ((double)b.lr * (double)b.lr * total)));
        *b.nu_ws = (float)nu;
        if (b.nu_out) *b.nu_out = (float)nu;
        if (b.s_out) *b.s_out = total;
        *b.counter = 0u;        // re-arm for the next call / graph replay
    }
}

__global__ void __launch_bounds__(kKlThreads) kl_scale_kernel(const __grid_constant__ KlBatch b) {
    const int cta = blockIdx.x;
    const KlLayer &L = b.l[find_layer(b, cta)];
    const float nu = *b.nu_ws;
    if (nu == 1.0f) return;
    const int r0 = (cta - L.cta_begin) * kKlRowsPerCta;
    const int r1 = min(L.rows, r0 + kKlRowsPerCta);
    if ((L.cols & 3) == 0) {
        const int c4 = L.cols / 4;
        for (int e = threadIdx.x; e < (r1 - r0) * c4; e += kKlThreads) {
            const int r = r0 + e / c4, c = (e % c4) * 4;
            float4 *p = reinterpret_cast<float4 *>(L.P + (size_t)r * L.ld + c);
            float4 v = *p;
            v.x *= nu; v.y *= nu; v.z *= nu; v.w *= nu;
            *p = v;
        }
    } else {
        for (int e = threadIdx.x; e < (r1 - r0) * L.cols; e += kKlThreads) {
            const int r = r0 + e / L.cols, c = e % L.cols;
            L.P[(size_t)r * L.ld + c] *= nu;
        }
    }
}

}  // namespace

size_t klclip_workspace_bytes(const int32_t *rows, int nl) {
    size_t ctas = 0;
    for (int l = 0; l < nl; ++l) ctas += cdiv(rows[l], kKlRowsPerCta);
    return round_up(ctas * sizeof(double), 256) + 256 * 2 + 256;
}

kfac_status_t klclip_run(float *const *P, const float *const *W, const int32_t *rows,
                         const int32_t *cols, const int32_t *ld, int nl, float lr, float kappa,
                         float *nu_out, double *s_out, void *ws, cudaStream_t s) {
    char *base = reinterpret_cast<char *>(round_up(reinterpret_cast<uintptr_t>(ws), 256));
    KFAC_CHECK_ARG(nl <= kKlMax, KFAC_ERR_SHAPE, "kfac_kl_clip: at most %d layers per call", kKlMax);
    KlBatch b;
    b.count = nl;
    b.lr = lr;
    b.kappa = kappa;
    int ctas = 0;
    for (int l = 0; l < nl; ++l) {
        b.l[l] = KlLayer{P[l], W[l], rows[l], cols[l], ld[l], ctas};
        ctas += cdiv(rows[l], kKlRowsPerCta);
    }
    b.ctas_total = ctas;
    b.partial = reinterpret_cast<double *>(base);
    char *tail = base + round_up(ctas * sizeof(double), 256);
    b.counter = reinterpret_cast<unsigned int *>(tail);
    b.nu_ws = reinterpret_cast<float *>(tail + 256);
    b.nu_out = nu_out;
    b.s_out = s_out;
    KFAC_CUDA_TRY(cudaMemsetAsync(b.counter, 0, sizeof(unsigned int), s));
    kl_dot_kernel<<<ctas, kKlThreads, 0, s>>>(b);
    KFAC_LAUNCHED();
    kl_scale_kernel<<<ctas, kKlThreads, 0, s>>>(b);
    KFAC_LAUNCHED();
    return KFAC_OK;
}

}  // namespace kfac
