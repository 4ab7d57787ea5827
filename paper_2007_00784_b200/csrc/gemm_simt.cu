// gemm_simt.cu -- grouped fp32 SIMT GEMM with the preconditioner's epilogues.
//
// One CTA computes a 128x128 tile of one problem of the group; tiles of all
// problems are laid out back to back along grid.x (layer-grouped launch, Eq. 4
// block-diagonal structure: every layer is an independent problem).  256
// threads, 8x8 outputs per thread, K staged 16 at a time through shared memory
// with a register prefetch of the next slab.  Used for small / ragged shapes
// and as the numerics baseline of the tcgen05 path.
#include "internal.cuh"

#include <vector>

namespace kfac {
namespace {

constexpr int BM = 128, BN = 128, BK = 16, NT = 256;

__device__ __forceinline__ int find_desc(const GemmBatch &b, int tile) {
    int lo = 0, hi = b.count - 1;
    while (lo < hi) {                       // last desc with tile_begin <= tile
        int mid = (lo + hi + 1) >> 1;
        if (b.d[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(NT) gemm_simt_kernel(const __grid_constant__ GemmBatch batch) {
    __shared__ float As[2][BK][BM + 4];
    __shared__ float Bs[2][BK][BN + 4];
    const int tile = blockIdx.x;
    const GemmDesc &d = batch.d[find_desc(batch, tile)];
    const int local = tile - d.tile_begin;
    const int tiles_n = (d.N + BN - 1) / BN;
    const int m0 = (local / tiles_n) * BM, n0 = (local % tiles_n) * BN;
    const int t = threadIdx.x;
    const int Me = d.M, Ne = d.dyn ? min(d.N, d.dyn[0]) : d.N, Ke = d.dyn ? min(d.K, d.dyn[1]) : d.K;
    if (n0 >= Ne) return;

    // loader coordinates: 8 consecutive elements per thread per operand
    int a_r, a_c, b_r, b_c;
    if (d.trans_a) { a_r = t / 16; a_c = (t % 16) * 8; }    // As[k][m..m+8) from A[k][m]
    else           { a_r = t / 2;  a_c = (t % 2) * 8; }     // A[m][k..k+8)
    if (d.trans_b) { b_r = t / 2;  b_c = (t % 2) * 8; }     // B[n][k..k+8)
    else           { b_r = t / 16; b_c = (t % 16) * 8; }    // Bs[k][n..n+8) from B[k][n]

    float ra[8], rb[8];
    auto load = [&](int k0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            int m, k;
            if (d.trans_a) { k = k0 + a_r; m = m0 + a_c + i; }
            else           { m = m0 + a_r; k = k0 + a_c + i; }
            ra[i] = (m < Me && k < Ke)
                        ? __ldg(d.trans_a ? d.A + (size_t)k * d.lda + m : d.A + (size_t)m * d.lda + k)
                        : 0.f;
            int n, kb;
            if (d.trans_b) { n = n0 + b_r; kb = k0 + b_c + i; }
            else           { kb = k0 + b_r; n = n0 + b_c + i; }
            rb[i] = (n < Ne && kb < Ke)
                        ? __ldg(d.trans_b ? d.B + (size_t)n * d.ldb + kb : d.B + (size_t)kb * d.ldb + n)
                        : 0.f;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (d.trans_a) As[buf][a_r][a_c + i] = ra[i];
            else           As[buf][a_c + i][a_r] = ra[i];
            if (d.trans_b) Bs[buf][b_c + i][b_r] = rb[i];
            else           Bs[buf][b_r][b_c + i] = rb[i];
        }
    };

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    const int ty = t / 16, tx = t % 16;
    const int nk = (Ke + BK - 1) / BK;
    load(0);
    store(0);
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nk) load((kt + 1) * BK);
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

#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        if (m >= Me) continue;
        const float vr = epi_uses_vectors(d.epi) ? d.vr[m] : 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
            if (n >= Ne) continue;
            float v = acc[i][j];
            if (d.epi == EPI_DIV_EIGEN) {
                v = v / fmaxf(fmaf(vr, d.vc[n], batch.damping), 1e-12f);
            } else if (d.epi == EPI_DIV_FACTORED) {
                v = v / fmaxf((vr + batch.damping) * (d.vc[n] + batch.damping), 1e-12f);
            } else if (d.epi == EPI_SUB) {
                v = d.C[(size_t)m * d.ldc + n] - v;
            }
            d.C[(size_t)m * d.ldc + n] = v;
        }
    }
}

}  // namespace

kfac_status_t gemm_simt_grouped(const GemmDesc *descs, int count, float damping, cudaStream_t s) {
    for (int base = 0; base < count; base += kGemmMaxDescs) {
        GemmBatch b;
        b.count = 0;
        b.damping = damping;
        int tiles = 0;
        for (int i = base; i < count && b.count < kGemmMaxDescs; ++i) {
            const GemmDesc &g = descs[i];
            if (g.M <= 0 || g.N <= 0) continue;
            b.d[b.count] = g;
            b.d[b.count].tile_begin = tiles;
            tiles += cdiv(g.M, BM) * cdiv(g.N, BN);
            ++b.count;
        }
        if (b.count == 0) continue;
        b.tiles_total = tiles;
        gemm_simt_kernel<<<tiles, NT, 0, s>>>(b);
        KFAC_LAUNCHED();
    }
    return KFAC_OK;
}

kfac_status_t gemm_grouped(const GemmDesc *descs, int count, float damping, cudaStream_t s) {
    // Layers below the tensor-core engine's tile (a dimension < 64) run the SIMT fp32 chain.
    return gemm_simt_grouped(descs, count, damping, s);
}

}  // namespace kfac
