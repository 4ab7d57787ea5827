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

#include <cstdlib>
#include <vector>

namespace kfac {

static bool getenv_flag(const char *name) {
    const char *e = getenv(name);
    return e && e[0] == '1';
}

// Layers whose four GEMMs all run on the tensor cores (every dimension >= 64, 16-byte rows) use
// the pre-split "planes" engine: Q_G, Q_A and the gradient are split once into TF32 hi/lo planes
// and every intermediate (T, V2, U) leaves its GEMM's epilogue as planes, so no GEMM re-splits
// an operand.  The others run the fp32 SIMT chain.
static bool planes_layer(int dg, int da, int ldW, int ldQG, int ldQA) {
    return !getenv_flag("KFAC_PRECOND_NO_PLANES") && dg >= 64 && da >= 64 && (ldW % 4) == 0 &&
           (ldQG % 4) == 0 && (ldQA % 4) == 0;
}

static size_t layer_floats(int dg, int da) {
    const size_t ldt = round_up(da, 4);
    const size_t ldg = round_up(dg, 4);
    // T, V (fp32 chain) or T, V, U planes (2 each) + Q_G, Q_A, grad planes (2 each)
    return 2 * (3 * round_up((size_t)dg * ldt, 64) + round_up((size_t)dg * ldg, 64) +
                round_up((size_t)da * ldt, 64) + round_up((size_t)dg * ldt, 64));
}

size_t precond_workspace_bytes(const int32_t *d_g, const int32_t *d_a, int nl, int mode) {
    size_t f = 0;
    for (int l = 0; l < nl; ++l) f += layer_floats(d_g[l], d_a[l]);
    (void)mode;
    return f * sizeof(float) + 256;
}

kfac_status_t precond_run(const int32_t *d_g, const int32_t *d_a, int nl, const float *const *grad,
                          const int32_t *ldW, const float *const *QG, const int32_t *ldQG,
                          const float *const *vG, const float *const *QA, const int32_t *ldQA,
                          const float *const *vA, float damping, int mode, float *const *out,
                          void *ws, cudaStream_t s) {
    float *base = reinterpret_cast<float *>(round_up(reinterpret_cast<uintptr_t>(ws), 256));
    // per layer: fp32 chain buffers T, V and (planes layers) the hi/lo planes
    struct Buf {
        float *T, *V;                                   // fp32 chain
        float *Th, *Tl, *Vh, *Vl, *Uh, *Ul;             // planes chain
        float *QGh, *QGl, *QAh, *QAl, *Wh, *Wl;         // split inputs
        int ldt, ldg, planes;
    };
    std::vector<Buf> B(nl);
    size_t off = 0;
    auto take = [&](size_t n) { float *p = base + off; off += round_up(n, 64); return p; };
    std::vector<SplitJob> split;
    for (int l = 0; l < nl; ++l) {
        Buf &b = B[l];
        b.ldt = (int)round_up(d_a[l], 4);
        b.ldg = (int)round_up(d_g[l], 4);
        const size_t gt = (size_t)d_g[l] * b.ldt;
        const size_t start = off;
        b.planes = planes_layer(d_g[l], d_a[l], ldW[l], ldQG[l], ldQA[l]);
        if (!b.planes) {
            b.T = take(gt);
            b.V = take(gt);
        } else {
            b.Th = take(gt); b.Tl = take(gt);
            b.Vh = take(gt); b.Vl = take(gt);
            b.Uh = take(gt); b.Ul = take(gt);
            b.QGh = take((size_t)d_g[l] * b.ldg); b.QGl = take((size_t)d_g[l] * b.ldg);
            b.QAh = take((size_t)d_a[l] * b.ldt); b.QAl = take((size_t)d_a[l] * b.ldt);
            b.Wh = take(gt); b.Wl = take(gt);
            split.push_back({QG[l], b.QGh, b.QGl, d_g[l], d_g[l], ldQG[l], b.ldg});
            split.push_back({QA[l], b.QAh, b.QAl, d_a[l], d_a[l], ldQA[l], b.ldt});
            split.push_back({grad[l], b.Wh, b.Wl, d_g[l], d_a[l], ldW[l], b.ldt});
        }
        off = start + layer_floats(d_g[l], d_a[l]);
    }
    kfac_status_t st;
    if (!split.empty() && (st = split_planes(split.data(), (int)split.size(), s)) != KFAC_OK) return st;

    std::vector<GemmDesc> gs, gp;                   // fp32 chain (SIMT / split-in-kernel), planes chain
    auto run = [&]() {
        kfac_status_t r = KFAC_OK;
        if (!gs.empty()) r = gemm_grouped(gs.data(), (int)gs.size(), damping, s);
        if (r == KFAC_OK && !gp.empty()) r = gemm_tc_planes_grouped(gp.data(), (int)gp.size(), damping, s);
        gs.clear();
        gp.clear();
        return r;
    };
    // one GEMM of the chain for layer l: op(A) op(B) -> C (fp32) or planes (Ch, Cl)
    auto add = [&](int l, const float *A, const float *Al, int lda, int ta, const float *Bm, const float *Bl, int ldb,
                   int tb, float *C, float *Cl, int ldc, int M, int N, int K, int epi) {
        GemmDesc d{};
        d.A = A; d.A_lo = Al; d.lda = lda; d.trans_a = ta;
        d.B = Bm; d.B_lo = Bl; d.ldb = ldb; d.trans_b = tb;
        d.C = C; d.C_lo = Cl; d.ldc = ldc; d.M = M; d.N = N; d.K = K; d.epi = epi;
        if (epi_uses_vectors(epi)) { d.vr = vG[l]; d.vc = vA[l]; }
        (B[l].planes ? gp : gs).push_back(d);
    };
    if (mode == KFAC_PRECOND_INVERSE) {
        for (int l = 0; l < nl; ++l) {      // T = G_inv grad
            const Buf &b = B[l];
            if (b.planes) add(l, b.QGh, b.QGl, b.ldg, 0, b.Wh, b.Wl, b.ldt, 0, b.Th, b.Tl, b.ldt, d_g[l], d_a[l], d_g[l], EPI_STORE);
            else add(l, QG[l], nullptr, ldQG[l], 0, grad[l], nullptr, ldW[l], 0, b.T, nullptr, b.ldt, d_g[l], d_a[l], d_g[l], EPI_STORE);
        }
        if ((st = run()) != KFAC_OK) return st;
        for (int l = 0; l < nl; ++l) {      // P = T A_inv
            const Buf &b = B[l];
            if (b.planes) add(l, b.Th, b.Tl, b.ldt, 0, b.QAh, b.QAl, b.ldt, 0, out[l], nullptr, ldW[l], d_g[l], d_a[l], d_a[l], EPI_STORE);
            else add(l, b.T, nullptr, b.ldt, 0, QA[l], nullptr, ldQA[l], 0, out[l], nullptr, ldW[l], d_g[l], d_a[l], d_a[l], EPI_STORE);
        }
        return run();
    }
    const int div = mode == KFAC_PRECOND_EIGEN ? EPI_DIV_EIGEN : EPI_DIV_FACTORED;
    for (int l = 0; l < nl; ++l) {          // T = Q_G^T grad
        const Buf &b = B[l];
        if (b.planes) add(l, b.QGh, b.QGl, b.ldg, 1, b.Wh, b.Wl, b.ldt, 0, b.Th, b.Tl, b.ldt, d_g[l], d_a[l], d_g[l], EPI_STORE);
        else add(l, QG[l], nullptr, ldQG[l], 1, grad[l], nullptr, ldW[l], 0, b.T, nullptr, b.ldt, d_g[l], d_a[l], d_g[l], EPI_STORE);
    }
    if ((st = run()) != KFAC_OK) return st;
    for (int l = 0; l < nl; ++l) {          // V2 = (T Q_A) / D   (Eq. 14 in the epilogue)
        const Buf &b = B[l];
        if (b.planes) add(l, b.Th, b.Tl, b.ldt, 0, b.QAh, b.QAl, b.ldt, 0, b.Vh, b.Vl, b.ldt, d_g[l], d_a[l], d_a[l], div);
        else add(l, b.T, nullptr, b.ldt, 0, QA[l], nullptr, ldQA[l], 0, b.V, nullptr, b.ldt, d_g[l], d_a[l], d_a[l], div);
    }
    if ((st = run()) != KFAC_OK) return st;
    for (int l = 0; l < nl; ++l) {          // U = Q_G V2
        const Buf &b = B[l];
        if (b.planes) add(l, b.QGh, b.QGl, b.ldg, 0, b.Vh, b.Vl, b.ldt, 0, b.Uh, b.Ul, b.ldt, d_g[l], d_a[l], d_g[l], EPI_STORE);
        else add(l, QG[l], nullptr, ldQG[l], 0, b.V, nullptr, b.ldt, 0, b.T, nullptr, b.ldt, d_g[l], d_a[l], d_g[l], EPI_STORE);
    }
    if ((st = run()) != KFAC_OK) return st;
    for (int l = 0; l < nl; ++l) {          // P = U Q_A^T
        const Buf &b = B[l];
        if (b.planes) add(l, b.Uh, b.Ul, b.ldt, 0, b.QAh, b.QAl, b.ldt, 1, out[l], nullptr, ldW[l], d_g[l], d_a[l], d_a[l], EPI_STORE);
        else add(l, b.T, nullptr, b.ldt, 0, QA[l], nullptr, ldQA[l], 1, out[l], nullptr, ldW[l], d_g[l], d_a[l], d_a[l], EPI_STORE);
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
