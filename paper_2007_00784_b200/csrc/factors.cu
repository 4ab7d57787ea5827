// factors.cu -- Stage 1 of Alg. 1: Kronecker factors and their running average.
//
//   A_batch = X^T X / n, X = [im2col(a_{i-1}) | 1]   (Eq. 5; im2col fused into the loads)
//   G_batch = g^T g / n                                (Eq. 5)
//   F = first ? F_batch : xi F_batch + (1 - xi) F;  F *= out_scale   (Eqs. 16-17, R5)
//
// Two launches per group of factors:
//   syrk_partial : one CTA per (upper-triangle 128x128 tile, row chunk); im2col patches are
//                  gathered straight from the NHWC activations (never materialised) and the
//                  symmetric rank-k update is accumulated for the chunk;
//   syrk_reduce  : sums the chunk partials in a fixed order (deterministic, no atomics),
//                  applies 1/n, the running average and out_scale, and writes both triangles.
// The SIMT tile is the numerics baseline; the tcgen05 3xTF32 SYRK replaces the partial kernel
// for large factors.
#include "internal.cuh"

#include <cstdlib>
#include <vector>

namespace kfac {
namespace {

constexpr int T = 128, BK = 16, NT = 256;
#ifndef KFAC_SYRK_CHUNK
#define KFAC_SYRK_CHUNK 8192
#endif
constexpr int kChunkRows = KFAC_SYRK_CHUNK;   // rows per partial (split-K chunk of the SYRKs)
constexpr int kMaxJobs = 64;

struct FactorBatch {
    int count;
    float xi, out_scale;  // xi: weight on the new batch estimate
    int first;
    FactorJob j[kMaxJobs];
};

__device__ __forceinline__ int find_job(const FactorBatch &b, int item, bool by_tile) {
    int lo = 0, hi = b.count - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        int beg = by_tile ? b.j[mid].tile_begin : b.j[mid].item_begin;
        if (beg <= item) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ void upper_tile(int tau, int t1d, int &ti, int &tj) {
    int i = 0;
    while (tau >= t1d - i) { tau -= t1d - i; ++i; }
    ti = i;
    tj = i + tau;
}

// Per-column gather descriptor: offset inside the receptive field and (kh, kw) for bounds.
struct ColInfo {
    int off, kh, kw, kind;   // kind: 0 regular, 1 bias (constant 1), 2 outside d (0)
};

__device__ __forceinline__ ColInfo col_info(const FactorJob &J, int c) {
    ColInfo ci;
    if (c >= J.d) { ci.kind = 2; ci.off = ci.kh = ci.kw = 0; return ci; }
    if (!J.is_a) { ci.kind = 0; ci.off = c; ci.kh = ci.kw = 0; return ci; }
    if (c >= J.patch_cols) { ci.kind = 1; ci.off = ci.kh = ci.kw = 0; return ci; }
    const int kwc = J.k_w * J.c_in;
    ci.kh = c / kwc;
    const int rem = c - ci.kh * kwc;
    ci.kw = rem / J.c_in;
    const int ch = rem - ci.kw * J.c_in;
    ci.off = (ci.kh * J.w_in + ci.kw) * J.c_in + ch;
    ci.kind = 0;
    return ci;
}

__global__ void __launch_bounds__(NT) syrk_partial_kernel(const __grid_constant__ FactorBatch batch) {
    __shared__ float As[2][BK][T + 4];
    __shared__ float Bs[2][BK][T + 4];
    const int item = blockIdx.x;
    const FactorJob &J = batch.j[find_job(batch, item, false)];
    const int local = item - J.item_begin;
    const int tau = local / J.splits, split = local % J.splits;
    int ti, tj;
    upper_tile(tau, J.t1d, ti, tj);
    const int t = threadIdx.x;
    const int lr = t / 16, lc = (t % 16) * 8;        // loader: row lr of the slab, 8 columns
    ColInfo ca[8], cb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        ca[i] = col_info(J, ti * T + lc + i);
        cb[i] = col_info(J, tj * T + lc + i);
    }
    const long long r_begin = (long long)split * J.chunk;
    const long long r_end = min(J.n, r_begin + J.chunk);
    const int hw = J.h_out * J.w_out;

    float ra[8], rb[8];
    auto load = [&](long long r0) {
        const long long r = r0 + lr;
        const bool rv = r < r_end;
        if (!J.is_a) {
            const float *row = J.src + r * J.c_in;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                ra[i] = (rv && ca[i].kind == 0) ? __ldg(row + ca[i].off) : 0.f;
                rb[i] = (rv && cb[i].kind == 0) ? __ldg(row + cb[i].off) : 0.f;
            }
            return;
        }
        int img = 0, oh = 0, ow = 0;
        if (rv) {
            img = (int)(r / hw);
            const int p = (int)(r - (long long)img * hw);
            oh = p / J.w_out;
            ow = p - oh * J.w_out;
        }
        const int ih0 = oh * J.stride_h - J.pad_h, iw0 = ow * J.stride_w - J.pad_w;
        const float *base = J.src + (((long long)img * J.h_in + ih0) * J.w_in + iw0) * J.c_in;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float va = 0.f, vb = 0.f;
            if (rv) {
                if (ca[i].kind == 1) va = 1.f;
                else if (ca[i].kind == 0) {
                    const int ih = ih0 + ca[i].kh, iw = iw0 + ca[i].kw;
                    if (ih >= 0 && ih < J.h_in && iw >= 0 && iw < J.w_in) va = __ldg(base + ca[i].off);
                }
                if (cb[i].kind == 1) vb = 1.f;
                else if (cb[i].kind == 0) {
                    const int ih = ih0 + cb[i].kh, iw = iw0 + cb[i].kw;
                    if (ih >= 0 && ih < J.h_in && iw >= 0 && iw < J.w_in) vb = __ldg(base + cb[i].off);
                }
            }
            ra[i] = va;
            rb[i] = vb;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            As[buf][lr][lc + i] = ra[i];
            Bs[buf][lr][lc + i] = rb[i];
        }
    };

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    const int ty = t / 16, tx = t % 16;
    const int nk = (int)((r_end - r_begin + BK - 1) / BK);
    load(r_begin);
    store(0);
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nk) load(r_begin + (long long)(kt + 1) * BK);
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            float a[8], b[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                a[i] = As[buf][k][ty * 4 + i];
                a[4 + i] = As[buf][k][64 + ty * 4 + i];
                b[i] = Bs[buf][k][tx * 4 + i];
                b[4 + i] = Bs[buf][k][64 + tx * 4 + i];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (kt + 1 < nk) {
            store(buf ^ 1);
            __syncthreads();
        }
    }
    float *out = J.partial + ((size_t)split * J.tiles + tau) * (T * T);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int m = i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4);
        float4 *dst = reinterpret_cast<float4 *>(out + m * T);
        dst[tx] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        dst[16 + tx] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
}

// Small factors (d <= 64, the ones the tensor-core engine does not take: ResNet-32's gradient
// factors d_G = 16 / 32 and its conv1 d_A = 28, the MLP's d_G = 10): the 128 x 128 SIMT tile would
// spend (128/d)^2 of its FMAs on padding.  Here one CTA per row chunk stages 128 rows x d columns
// of X = [im2col | 1] (or of the gradient rows) in shared memory; each thread accumulates 2 x 2
// register blocks of the upper triangle (4 FMAs per two 8-byte loads), over all rows or, when
// there are fewer blocks than threads, over one of P row phases combined in a fixed order; fp32
// like the SIMT tile, and the partial lands where the SIMT tile would put it, so the fold is
// unchanged.
constexpr int kSmallD = 64;
constexpr int kSmallRows = 128;
constexpr int kSmallLd = kSmallD + 2;                        // even row stride: 8-byte column pairs
constexpr int kSmallBpt = ((kSmallD / 2) * (kSmallD / 2 + 1) / 2 + 255) / 256;   // blocks per thread (3)

__global__ void __launch_bounds__(256, 2) syrk_small_kernel(const __grid_constant__ FactorBatch batch) {
    __shared__ __align__(16) float X[kSmallRows][kSmallLd];
    __shared__ ColInfo cinf[kSmallD];
    __shared__ int rorg[kSmallRows][3];          // per staged row: element offset of the receptive
                                                 // field origin, ih0, iw0 (A)
    __shared__ float red[256 * 4];
    const int item = blockIdx.x;
    const FactorJob &J = batch.j[find_job(batch, item, false)];
    const int split = item - J.item_begin;       // one tile (d <= 64 < T): item = split
    const int t = threadIdx.x, d = J.d;
    const int nb = (d + 1) / 2, dp = 2 * nb;     // column pairs; column d (odd d) is staged as 0
    const int B = nb * (nb + 1) / 2;             // upper 2 x 2 blocks
    const int P = max(1, 256 / B);
    const bool active = t < B * P;
    const int p = B <= 256 ? t / B : 0;
    int bi[kSmallBpt], bj[kSmallBpt];
#pragma unroll
    for (int q = 0; q < kSmallBpt; ++q) {
        const int b = B <= 256 ? (q == 0 && active ? t % B : -1) : (t + 256 * q < B ? t + 256 * q : -1);
        int a = 0, rem = b < 0 ? 0 : b;          // block b of the row-major upper triangle of nb x nb
        while (rem >= nb - a) { rem -= nb - a; ++a; }
        bi[q] = b < 0 ? -1 : a;
        bj[q] = b < 0 ? 0 : a + rem;
    }
    const int nblk = B <= 256 ? (active ? 1 : 0) : (B - t + 255) / 256;
    if (t < d) cinf[t] = col_info(J, t);
    const long long r_begin = (long long)split * J.chunk;
    const long long r_end = min(J.n, r_begin + J.chunk);
    const int hw = J.h_out * J.w_out;
    float acc[kSmallBpt][4];
#pragma unroll
    for (int q = 0; q < kSmallBpt; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.f;
    for (long long r0 = r_begin; r0 < r_end; r0 += kSmallRows) {
        const int nr = (int)min((long long)kSmallRows, r_end - r0);
        __syncthreads();                         // previous step's reads done (and cinf ready)
        if (J.is_a && t < kSmallRows && t < nr) {
            const long long r = r0 + t;
            const int img = (int)(r / hw);
            const int pp = (int)(r - (long long)img * hw);
            const int oh = pp / J.w_out, ow = pp - oh * J.w_out;
            const int ih0 = oh * J.stride_h - J.pad_h, iw0 = ow * J.stride_w - J.pad_w;
            rorg[t][0] = ((img * J.h_in + ih0) * J.w_in + iw0) * J.c_in;
            rorg[t][1] = ih0;
            rorg[t][2] = iw0;
        }
        if (J.is_a) __syncthreads();
        // every load of the step issued before any is stored (a load-store loop waits out the
        // memory latency once per element)
        constexpr int kPer = kSmallRows * kSmallD / 256;
        float vals[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int q = t + 256 * u;
            if (256 * u >= kSmallRows * dp) break;   // uniform: 128 dp is a multiple of 256
            const int rr = q / dp, c = q - rr * dp;
            float v = 0.f;
            if (rr < nr && c < d) {
                const ColInfo ci = cinf[c];
                if (!J.is_a) {
                    v = __ldg(J.src + (r0 + rr) * J.c_in + ci.off);
                } else if (ci.kind == 1) {
                    v = 1.f;
                } else if (ci.kind == 0) {
                    const int ih = rorg[rr][1] + ci.kh, iw = rorg[rr][2] + ci.kw;
                    if (ih >= 0 && ih < J.h_in && iw >= 0 && iw < J.w_in) v = __ldg(J.src + rorg[rr][0] + ci.off);
                }
            }
            vals[u] = v;
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int q = t + 256 * u;
            if (256 * u >= kSmallRows * dp) break;
            const int rr = q / dp;
            X[rr][q - rr * dp] = vals[u];
        }
        __syncthreads();
        for (int rr = p; rr < nr; rr += P) {
            const float *xr = X[rr];
#pragma unroll
            for (int q = 0; q < kSmallBpt; ++q) {
                if (q >= nblk) break;
                const float2 a = *reinterpret_cast<const float2 *>(xr + 2 * bi[q]);
                const float2 b = *reinterpret_cast<const float2 *>(xr + 2 * bj[q]);
                acc[q][0] = fmaf(a.x, b.x, acc[q][0]);
                acc[q][1] = fmaf(a.x, b.y, acc[q][1]);
                acc[q][2] = fmaf(a.y, b.x, acc[q][2]);
                acc[q][3] = fmaf(a.y, b.y, acc[q][3]);
            }
        }
    }
    float *out = J.partial + (size_t)split * J.tiles * (T * T);
    if (B <= 256) {
#pragma unroll
        for (int u = 0; u < 4; ++u) red[u * 256 + t] = acc[0][u];
        __syncthreads();
        if (active && p == 0) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = 2 * bi[0] + (u >> 1), j = 2 * bj[0] + (u & 1);
                if (i >= d || j >= d || i > j) continue;
                float sum = 0.f;
                for (int q = 0; q < P; ++q) sum += red[u * 256 + q * B + t];   // fixed order over the phases
                out[i * T + j] = sum;
            }
        }
    } else {
#pragma unroll
        for (int q = 0; q < kSmallBpt; ++q) {
            if (q >= nblk) break;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = 2 * bi[q] + (u >> 1), j = 2 * bj[q] + (u & 1);
                if (i < d && j < d && i <= j) out[i * T + j] = acc[q][u];
            }
        }
    }
}

// Column of the SYRK's (possibly channel-padded) geometry that holds column c of the real factor.
__device__ __forceinline__ int padded_col(const FactorJob &J, int c) {
    if (!J.c_real || !J.is_a) return c;                  // no padding, or padding after the last column
    const int patch_real = J.c_real * (J.patch_cols / J.c_in);
    if (c >= patch_real) return J.patch_cols;            // bias column
    return (c / J.c_real) * J.c_in + c % J.c_real;
}

// Upper-tile index of tile (ti, tj), ti <= tj, in a t1d x t1d tile grid.
__device__ __forceinline__ int upper_index(int ti, int tj, int t1d) { return ti * t1d - ti * (ti - 1) / 2 + (tj - ti); }

// One CTA (32x8 threads) per 32x32 sub-tile of an upper 128x128 tile of the real factor.
__global__ void __launch_bounds__(256) syrk_reduce_kernel(const __grid_constant__ FactorBatch batch) {
    __shared__ float tr[32][33];
    const int blk = blockIdx.x;                  // tile_begin counts sub-tiles (16 per tile)
    const FactorJob &J = batch.j[find_job(batch, blk, true)];
    const int local = blk - J.tile_begin;
    const int tau = local / 16, sub = local % 16;
    int ti, tj;
    upper_tile(tau, J.t1d_out, ti, tj);
    const int si = sub / 4, sj = sub % 4;
    if (ti == tj && si > sj) return;             // the (sj, si) sub-tile writes both copies
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
    const float inv_n = 1.0f / (float)J.n;
    const int d = J.d_out;
    const int gj = tj * T + sj * 32 + tx;
    for (int rr = ty; rr < 32; rr += 8) {
        const int li = si * 32 + rr, lj = sj * 32 + tx;
        const int gi = ti * T + li;
        // diagonal tiles: read the upper entry for both (i, j) and (j, i) -> exact symmetry
        const bool swap = ti == tj && li > lj;
        const int ui = swap ? gj : gi, uj = swap ? gi : gj;       // ui <= uj (real columns)
        float v = 0.f;
        if (gi < d && gj < d) {
            const int mi = padded_col(J, ui), mj = padded_col(J, uj);   // monotone: mi <= mj
            const size_t off = (size_t)upper_index(mi / T, mj / T, J.t1d) * (T * T) + (mi % T) * T + (mj % T);
            float s = 0.f;
            for (int sp = 0; sp < J.splits; ++sp) s += J.partial[(size_t)sp * J.tiles * (T * T) + off];
            v = s * inv_n;
            float *dst = J.F + (size_t)gi * J.ldF + gj;
            if (!batch.first) v = batch.xi * v + (1.f - batch.xi) * (*dst);
            v *= batch.out_scale;
            *dst = v;
            if (J.packed && gi <= gj)            // each upper entry once: row gi starts at gi d - gi (gi - 1) / 2
                J.packed[(long long)gi * d - (long long)gi * (gi - 1) / 2 + (gj - gi)] = v;
        }
        tr[rr][tx] = v;
    }
    if (ti == tj && si == sj) return;            // diagonal sub-tile already holds both triangles
    __syncthreads();
    const int gcol = ti * T + si * 32 + tx;      // mirrored write: F[gj][gi]
    for (int rr = ty; rr < 32; rr += 8) {
        const int grow = tj * T + sj * 32 + rr;
        if (grow < d && gcol < d) J.F[(size_t)grow * J.ldF + gcol] = tr[tx][rr];
    }
}

struct Plan {
    std::vector<FactorJob> jobs;
    size_t partial_floats = 0;
    size_t plane_floats = 0;        // TF32 hi/lo planes of the tensor-core jobs' inputs
};

// Elements of a job's input tensor (A: the NHWC activation, G: the n x c_out gradient rows).
inline long long input_elems(const FactorJob &j) {
    return j.is_a ? (j.n / ((long long)j.h_out * j.w_out)) * j.h_in * j.w_in * j.c_in : j.n * j.c_in;
}

Plan make_plan(const kfac_layer_t *layers, int nl, float *const *A, const int32_t *ldA,
               float *const *G, const int32_t *ldG, const float *const *act,
               const float *const *gout, float *const *pA = nullptr, float *const *pG = nullptr) {
    Plan p;
    for (int l = 0; l < nl; ++l) {
        const kfac_layer_t &L = layers[l];
        for (int f = 0; f < 2; ++f) {
            FactorJob j{};
            j.is_a = f == 0;
            j.n = (long long)L.batch * L.h_out * L.w_out;
            j.d = j.is_a ? L.c_in * L.k_h * L.k_w + L.bias_col : L.c_out;
            j.src = act ? (j.is_a ? act[l] : gout[l]) : nullptr;
            j.F = A ? (j.is_a ? A[l] : G[l]) : nullptr;
            j.packed = j.is_a ? (pA ? pA[l] : nullptr) : (pG ? pG[l] : nullptr);
            j.ldF = ldA ? (j.is_a ? ldA[l] : ldG[l]) : 0;
            j.c_in = j.is_a ? L.c_in : L.c_out;
            j.h_in = L.h_in; j.w_in = L.w_in; j.h_out = L.h_out; j.w_out = L.w_out;
            j.k_w = L.k_w; j.stride_h = L.stride_h; j.stride_w = L.stride_w;
            j.pad_h = L.pad_h; j.pad_w = L.pad_w;
            j.patch_cols = L.c_in * L.k_h * L.k_w;
            j.bias_col = L.bias_col;
            j.chunk = kChunkRows;
            j.splits = (int)((j.n + kChunkRows - 1) / kChunkRows);
            j.d_out = j.d;
            j.t1d_out = cdiv(j.d, T);
            j.tiles_out = j.t1d_out * (j.t1d_out + 1) / 2;
            if (j.d >= 64 && j.n >= 32 && j.c_in % 4 != 0) {
                // tensor-core SYRK on zero-padded channels (the fold gathers the real columns);
                // kept only if the padded job is one the tensor-core engine takes
                FactorJob pj = j;
                pj.c_real = j.c_in;
                pj.c_in = (int)round_up((size_t)j.c_in, 4);
                if (pj.is_a) {
                    pj.patch_cols = pj.c_in * L.k_h * L.k_w;
                    pj.d = pj.patch_cols + L.bias_col;
                } else {
                    pj.d = pj.c_in;
                }
                if (syrk_tc_supported(pj)) j = pj;
            }
            j.t1d = cdiv(j.d, T);
            j.tiles = j.t1d * (j.t1d + 1) / 2;
            j.partial = reinterpret_cast<float *>(p.partial_floats);   // offset, rebased later
            p.partial_floats += (size_t)j.splits * j.tiles * T * T;
            if (syrk_tc_supported(j)) p.plane_floats += 2 * round_up((size_t)input_elems(j), 64);
            p.jobs.push_back(j);
        }
    }
    return p;
}

}  // namespace

size_t factors_workspace_bytes(const kfac_layer_t *layers, int nl) {
    Plan p = make_plan(layers, nl, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    return (p.partial_floats + p.plane_floats) * sizeof(float) + 512;
}

kfac_status_t factors_run(const kfac_layer_t *layers, int nl, const float *const *act,
                          const float *const *gout, float *const *A, const int32_t *ldA,
                          float *const *G, const int32_t *ldG, float *const *pA, float *const *pG,
                          float xi, int first, float out_scale, void *ws, cudaStream_t s) {
    Plan p = make_plan(layers, nl, A, ldA, G, ldG, act, gout, pA, pG);
    float *base = reinterpret_cast<float *>(round_up(reinterpret_cast<uintptr_t>(ws), 256));
    for (auto &j : p.jobs) j.partial = base + reinterpret_cast<uintptr_t>(j.partial);
    // Partial SYRKs: tcgen05 3xTF32 for the factors it supports, the SIMT tile for the rest.  The
    // tensor-core jobs' inputs are first split once into TF32 hi/lo planes (one elementwise pass),
    // so the SYRK kernel gathers both planes and never splits in shared memory.
    std::vector<FactorJob> tc, simt;
    for (auto &j : p.jobs) (syrk_tc_supported(j) ? tc : simt).push_back(j);
    // the SIMT / small-d partial SYRKs are independent of the tensor-core ones: they run on a side
    // stream forked from s and joined back before the fold
    SideFork fk;
    const bool par = !tc.empty() && !simt.empty();
    if (par) KFAC_CUDA_TRY(fk.fork(s, 1));
    const cudaStream_t ss = par ? fk.side(0) : s;
    if (!tc.empty()) {
        float *pl = base + round_up(p.partial_floats, 64);
        std::vector<SplitJob> sj;
        for (auto &j : tc) {
            const size_t e = round_up((size_t)input_elems(j), 64);
            const int cols = j.c_real ? j.c_real : j.c_in;     // padded jobs: zero channels appended
            const int rows = (int)(input_elems(j) / j.c_in);
            sj.push_back({j.src, pl, pl + e, rows, cols, cols, j.c_in});
            j.src = pl;
            j.src_lo = pl + e;
            pl += 2 * e;
        }
        kfac_status_t st = split_planes(sj.data(), (int)sj.size(), s);
        if (st != KFAC_OK) return st;
    }
    if (!tc.empty()) {
        kfac_status_t st = syrk_tc_partial(tc.data(), (int)tc.size(), s);
        if (st != KFAC_OK) return st;
    }
    std::vector<FactorJob> small, tile;
    for (auto &j : simt) (j.d <= kSmallD && input_elems(j) < (1ll << 31) ? small : tile).push_back(j);
    for (size_t b0 = 0; b0 < small.size(); b0 += kMaxJobs) {
        FactorBatch fb;
        fb.count = 0;
        int items = 0;
        for (size_t i = b0; i < small.size() && fb.count < kMaxJobs; ++i) {
            FactorJob j = small[i];
            j.item_begin = items;
            items += j.splits;                       // one tile
            fb.j[fb.count++] = j;
        }
        syrk_small_kernel<<<items, 256, 0, ss>>>(fb);
        KFAC_LAUNCHED();
    }
    for (size_t b0 = 0; b0 < tile.size(); b0 += kMaxJobs) {
        FactorBatch fb;
        fb.count = 0;
        int items = 0;
        for (size_t i = b0; i < tile.size() && fb.count < kMaxJobs; ++i) {
            FactorJob j = tile[i];
            j.item_begin = items;
            items += j.tiles * j.splits;
            fb.j[fb.count++] = j;
        }
        syrk_partial_kernel<<<items, NT, 0, ss>>>(fb);
        KFAC_LAUNCHED();
    }
    if (par) KFAC_CUDA_TRY(fk.join(s));
    // Fixed-order reduction + running average for every factor.
    for (size_t b0 = 0; b0 < p.jobs.size(); b0 += kMaxJobs) {
        FactorBatch fb;
        fb.count = 0;
        fb.xi = xi;
        fb.out_scale = out_scale;
        fb.first = first;
        int subtiles = 0;
        for (size_t i = b0; i < p.jobs.size() && fb.count < kMaxJobs; ++i) {
            FactorJob j = p.jobs[i];
            j.tile_begin = subtiles;
            subtiles += j.tiles_out * 16;
            fb.j[fb.count++] = j;
        }
        syrk_reduce_kernel<<<subtiles, 256, 0, s>>>(fb);
        KFAC_LAUNCHED();
    }
    return KFAC_OK;
}

// Packed upper triangles (row-major, d(d+1)/2 floats) -> full symmetric factors (both triangles):
// the receive side of the halved factor allreduce.  One 32 x 32 tile per CTA (lower tiles are the
// mirrored writes of the upper ones).
struct UnpackJob {
    const float *packed;
    float *F;
    int d, ldF, t1d, tile_begin;
};
struct UnpackBatch {
    int count;
    float scale;
    UnpackJob j[64];
};

__global__ void __launch_bounds__(256) unpack_kernel(const __grid_constant__ UnpackBatch b) {
    __shared__ float tr[32][33];
    int lo = 0, hi = b.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (b.j[mid].tile_begin <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    const UnpackJob &J = b.j[lo];
    int t = blockIdx.x - J.tile_begin, ti = 0;
    while (t >= J.t1d - ti) { t -= J.t1d - ti; ++ti; }         // upper tiles, row-major
    const int tj = ti + t;
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
    for (int rr = ty; rr < 32; rr += 8) {
        const int gi = ti * 32 + rr, gj = tj * 32 + tx;
        float v = 0.f;
        if (gi < J.d && gj < J.d) {
            const int a = min(gi, gj), c = max(gi, gj);
            v = b.scale * J.packed[(long long)a * J.d - (long long)a * (a - 1) / 2 + (c - a)];
            J.F[(size_t)gi * J.ldF + gj] = v;
        }
        tr[rr][tx] = v;
    }
    if (ti == tj) return;
    __syncthreads();
    for (int rr = ty; rr < 32; rr += 8) {
        const int gi = tj * 32 + rr, gj = ti * 32 + tx;
        if (gi < J.d && gj < J.d) J.F[(size_t)gi * J.ldF + gj] = tr[tx][rr];
    }
}

kfac_status_t unpack_run(const float *const *packed, const int32_t *dims, float *const *F, const int32_t *ldF,
                         int count, float scale, cudaStream_t s) {
    for (int b0 = 0; b0 < count; b0 += 64) {
        UnpackBatch b;
        b.count = 0;
        b.scale = scale;
        int tiles = 0;
        for (int i = b0; i < count && b.count < 64; ++i) {
            UnpackJob &j = b.j[b.count++];
            j.packed = packed[i];
            j.F = F[i];
            j.d = dims[i];
            j.ldF = ldF[i];
            j.t1d = cdiv(dims[i], 32);
            j.tile_begin = tiles;
            tiles += j.t1d * (j.t1d + 1) / 2;
        }
        unpack_kernel<<<tiles, 256, 0, s>>>(b);
        KFAC_LAUNCHED();
    }
    return KFAC_OK;
}

}  // namespace kfac
