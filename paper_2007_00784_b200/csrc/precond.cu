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

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace kfac {

// Layers whose four GEMMs all run on the tensor cores (every dimension >= 64, 16-byte rows) use
// the pre-split "planes" engine: Q_G, Q_A and the gradient are split once into TF32 hi/lo planes
// and every intermediate (T, V2, U) leaves its GEMM's epilogue as planes, so no GEMM re-splits
// an operand.  The others run the fp32 SIMT chain.
static bool planes_layer(int dg, int da, int ldW, int ldQG, int ldQA) {
    return dg >= 64 && da >= 64 && (ldW % 4) == 0 &&
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
// Eq. 18 (R12) in three passes, every one a float4 stream over the layers' rows:
//   kl_dot   per CTA, a contiguous run of rows of one layer (about kKlUnits float4 of P and of
//            grad, masked at the row tail: d_A is odd with the bias column), fp32 products summed
//            in fp64; the last CTA of the launch reduces its layers' CTA partials, one warp per
//            layer in a fixed order, into layer_dot[l];
//   kl_nu    one warp: s = sum_l |layer_dot[l]| in layer order, nu = min(1, sqrt(kappa/(lr^2 s)));
//   kl_scale P *= nu over the same runs of rows.
// Layers are launched in chunks of kKlMax descriptors (kernel parameters), so any layer count
// works; the reduction order depends only on the shapes (bitwise reproducible).
namespace {

constexpr int kKlMax = 256;
constexpr int kKlThreads = 256;
constexpr int kKlUnits = 8192;       // float4 of P per CTA (128 KB of P + grad in flight per CTA)

struct KlLayer {
    float *P;
    const float *W;
    int rows, cols, ld, nch;         // nch = ceil(cols / 4) float4 chunks per row
    int rows_per_cta, cta_begin;
};

struct KlBatch {
    int count, ctas_total, layer_base;
    double *partial;        // [ctas_total] of this chunk
    double *layer_dot;      // [all layers]
    unsigned int *counter;  // last-CTA ticket of this chunk
    const float *nu;        // scale pass
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

__device__ __forceinline__ float4 masked(float4 v, int c, int cols) {
    if (c + 3 >= cols) {             // row tail: elements at or past `cols` are padding
        if (c + 1 >= cols) v.y = 0.f;
        if (c + 2 >= cols) v.z = 0.f;
        if (c + 3 >= cols) v.w = 0.f;
    }
    return v;
}

__global__ void __launch_bounds__(kKlThreads) kl_dot_kernel(const __grid_constant__ KlBatch b) {
    __shared__ double red[kKlThreads / 32];
    __shared__ bool last;
    const int cta = blockIdx.x;
    const KlLayer &L = b.l[find_layer(b, cta)];
    const int r0 = (cta - L.cta_begin) * L.rows_per_cta;
    const int r1 = min(L.rows, r0 + L.rows_per_cta);
    const int units = (r1 - r0) * L.nch;
    double acc = 0.0;
    for (int e0 = threadIdx.x; e0 < units; e0 += 4 * kKlThreads) {
        float4 p[4], w[4];
        int cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {           // all loads of the round before any use
            const int e = e0 + u * kKlThreads;
            const int r = r0 + e / L.nch, c = (e % L.nch) * 4;
            cc[u] = c;
            if (e < units) {
                p[u] = __ldcs(reinterpret_cast<const float4 *>(L.P + (size_t)r * L.ld + c));
                w[u] = __ldcs(reinterpret_cast<const float4 *>(L.W + (size_t)r * L.ld + c));
            } else {
                p[u] = w[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            // padding columns of either operand may hold anything (NaN included): mask both
            const float4 q = masked(p[u], cc[u], L.cols), v = masked(w[u], cc[u], L.cols);
            acc += (double)(q.x * v.x) + (double)(q.y * v.y) + (double)(q.z * v.z) + (double)(q.w * v.w);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < kKlThreads / 32; ++i) s += red[i];
        b.partial[cta] = s;
        __threadfence();
        last = atomicAdd(b.counter, 1u) == (unsigned)(b.ctas_total - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // last CTA of the chunk: one warp per layer, lane-strided partial sums, fixed butterfly
    for (int l = warp; l < b.count; l += kKlThreads / 32) {
        const int beg = b.l[l].cta_begin;
        const int end = l + 1 < b.count ? b.l[l + 1].cta_begin : b.ctas_total;
        double s = 0.0;
        for (int c = beg + lane; c < end; c += 32) s += __ldcg(b.partial + c);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) b.layer_dot[b.layer_base + l] = s;
    }
    if (threadIdx.x == 0) *b.counter = 0u;    // re-arm for the next chunk / call / graph replay
}

__global__ void kl_nu_kernel(const double *layer_dot, int nl, float lr, float kappa, float *nu_ws,
                             float *nu_out, double *s_out) {
    const int lane = threadIdx.x;
    double s = 0.0;
    for (int l = lane; l < nl; l += 32) s += fabs(__ldcg(layer_dot + l));      // R12: |.| per layer
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        double nu = 1.0;
        if (s > 0.0) nu = fmin(1.0, sqrt((double)kappa / ((double)lr * (double)lr * s)));
        *nu_ws = (float)nu;
        if (nu_out) *nu_out = (float)nu;
        if (s_out) *s_out = s;
    }
}

__global__ void __launch_bounds__(kKlThreads) kl_scale_kernel(const __grid_constant__ KlBatch b) {
    const int cta = blockIdx.x;
    const KlLayer &L = b.l[find_layer(b, cta)];
    const float nu = *b.nu;
    if (nu == 1.0f) return;
    const int r0 = (cta - L.cta_begin) * L.rows_per_cta;
    const int r1 = min(L.rows, r0 + L.rows_per_cta);
    const int units = (r1 - r0) * L.nch;
    for (int e0 = threadIdx.x; e0 < units; e0 += 4 * kKlThreads) {
        float4 p[4];
        float4 *ptr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * kKlThreads;
            const int r = r0 + e / L.nch, c = (e % L.nch) * 4;
            ptr[u] = e < units ? reinterpret_cast<float4 *>(L.P + (size_t)r * L.ld + c) : nullptr;
            if (ptr[u]) p[u] = __ldcs(ptr[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (ptr[u]) __stcs(ptr[u], make_float4(p[u].x * nu, p[u].y * nu, p[u].z * nu, p[u].w * nu));
    }
}

struct KlPlan {
    std::vector<KlBatch> chunks;
    size_t partial_off, dot_off, tail_off, bytes;
};

KlPlan kl_plan(const int32_t *rows, const int32_t *cols, int nl) {
    KlPlan p;
    size_t ctas_max = 0;
    for (int base = 0; base < nl; base += kKlMax) {
        KlBatch b;
        memset(&b, 0, sizeof(b));
        b.layer_base = base;
        int ctas = 0;
        for (int l = base; l < nl && b.count < kKlMax; ++l) {
            KlLayer &L = b.l[b.count++];
            L.rows = rows[l];
            L.cols = cols[l];
            L.nch = (cols[l] + 3) / 4;
            L.rows_per_cta = std::max(1, kKlUnits / L.nch);
            L.cta_begin = ctas;
            ctas += cdiv(L.rows, L.rows_per_cta);
        }
        b.ctas_total = ctas;
        ctas_max = std::max(ctas_max, (size_t)ctas);
        p.chunks.push_back(b);
    }
    p.partial_off = 0;
    p.dot_off = round_up(ctas_max * sizeof(double), 256);
    p.tail_off = p.dot_off + round_up((size_t)nl * sizeof(double), 256);
    p.bytes = p.tail_off + 256 * 2 + 256;
    return p;
}

}  // namespace

size_t klclip_workspace_bytes(const int32_t *rows, const int32_t *cols, int nl) {
    return kl_plan(rows, cols, nl).bytes;
}

kfac_status_t klclip_run(float *const *P, const float *const *W, const int32_t *rows,
                         const int32_t *cols, const int32_t *ld, int nl, float lr, float kappa,
                         float *nu_out, double *s_out, void *ws, cudaStream_t s) {
    char *base = reinterpret_cast<char *>(round_up(reinterpret_cast<uintptr_t>(ws), 256));
    KlPlan plan = kl_plan(rows, cols, nl);
    double *partial = reinterpret_cast<double *>(base + plan.partial_off);
    double *layer_dot = reinterpret_cast<double *>(base + plan.dot_off);
    unsigned int *counter = reinterpret_cast<unsigned int *>(base + plan.tail_off);
    float *nu_ws = reinterpret_cast<float *>(base + plan.tail_off + 256);
    KFAC_CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(unsigned int), s));
    for (auto &b : plan.chunks) {
        for (int q = 0; q < b.count; ++q) {
            const int l = b.layer_base + q;
            b.l[q].P = P[l];
            b.l[q].W = W[l];
            b.l[q].ld = ld[l];
        }
        b.partial = partial;
        b.layer_dot = layer_dot;
        b.counter = counter;
        b.nu = nu_ws;
        kl_dot_kernel<<<b.ctas_total, kKlThreads, 0, s>>>(b);
        KFAC_LAUNCHED();
    }
    kl_nu_kernel<<<1, 32, 0, s>>>(layer_dot, nl, lr, kappa, nu_ws, nu_out, s_out);
    KFAC_LAUNCHED();
    for (auto &b : plan.chunks) {
        kl_scale_kernel<<<b.ctas_total, kKlThreads, 0, s>>>(b);
        KFAC_LAUNCHED();
    }
    return KFAC_OK;
}

}  // namespace kfac
