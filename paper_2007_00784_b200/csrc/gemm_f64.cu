// gemm_f64.cu -- grouped GEMM with fp64 accumulation for the eigensolver's internal products
// (trailing rank-2k updates, divide-and-conquer eigenvector updates, back-transformation, the
// two-stage reduction's rank-32 update), and the explicit inverse's blocked updates.
//
// Why fp64 there: the preconditioner divides by v_G v_A^T + damping, so an eigenvector error e along
// a direction of eigenvalue L is amplified by ~L/damping (5e5 for the ResNet-50 fc A factor); the
// eigenvectors must be accurate to the fp32 rounding level, while a 3xTF32 product carries ~2^-22
// relative error per term and accumulates across ~10 chained GEMMs.
//
// Engines (gemm64_grouped picks per batch): fp64 tensor cores (DMMA, mma.sync m8n8k4) fed by a
// cp.async pipeline -- straight from the fp64 stages when both operands are fp64 ("direct"), through
// an fp32->fp64 conversion pass otherwise ("pipe"); a SIMT fallback for unaligned operands; and,
// while an Ozaki arena is set, the int8 tensor-core Ozaki scheme (gemm_ozaki.cu) for large products.
#include "internal.cuh"

#include <cstdlib>
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

// Epilogue shared by both kernels: the thread owns rows rows[i] (i < 8) and column pairs
// (cols[jj], cols[jj] + 1) (jj < 4); acc[i][2 jj + e] is element (rows[i], cols[jj] + e).
__device__ __forceinline__ void epilogue(const Gemm64Desc &d, int Me, int Ne, const int (&rows)[8],
                                         const int (&cols)[4], const double (&acc)[8][8]) {
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
            const int m = rows[i];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int n = cols[jj];
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
            const int m = rows[i];
            if (m >= Me) continue;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int n = cols[jj];
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

    int rows[8], cols[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) rows[i] = m0 + 2 * ty + (i & 1) + 32 * (i >> 1);
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) cols[jj] = n0 + 2 * tx + 32 * jj;
    epilogue(d, Me, Ne, rows, cols, acc);
}


// ------------------------------------------------------- pipelined DMMA kernel --
// Same 128 x 128 output tile, K staged 16 at a time: every slab is copied raw (fp32 or fp64, in
// the operand's own layout) into one of kStages shared-memory stages with cp.async -- kStages-1
// slabs in flight while one is computed -- then converted once to fp64 tiles T[k][mn] (row
// stride kTs = 136 doubles, so the 8x4 fragment loads below hit every bank exactly twice).  The
// products run on the fp64 tensor cores: mma.sync m8n8k4 f64 (DMMA; fp64 products, fp64
// accumulation -- the same arithmetic as DFMA, at the tensor pipe's rate).  Warp w owns the
// 64 x 32 block (rows 64 (w / 4), columns 32 (w % 4)) as 8 x 4 DMMA tiles.  Used when every
// operand's rows are 16-byte aligned.
constexpr int PBK = 16, kStages = 2, kPM = 64;                 // pipelined tile: kPM x BN
constexpr int kPT = kPM * 2;                                      // 4 warps, each 64 x 32
constexpr int kTsA = kPM + 8, kTsB = BN + 8;                      // fp64 tile row strides
constexpr int kRawA = kPM * PBK * 8, kRawB = BN * PBK * 8;        // raw slabs, fp64 worst case
constexpr int kTileD = PBK * (kTsA + kTsB);                       // doubles per fp64 tile pair
constexpr int kPipeSmem = kStages * (kRawA + kRawB) + 2 * kTileD * 8 + 64;

// Raw slab of one operand: "outer" rows of "inner" contiguous elements.  MN-contiguous operands
// (A^T stored k x m, B stored k x n) have outer = k, inner = mn; K-contiguous ones the reverse.
struct RawOp {
    const char *base;     // element (0, 0) of the operand
    size_t ld_bytes;      // bytes between outer rows
    int es;               // element size
    int mn_inner;         // 1: inner = mn (ext wide), outer = k (16); 0: inner = k, outer = mn
    int ext;              // mn extent of the tile (kPM for A, BN for B)
    int mn0, mn_lim, k_lim;
};

__device__ __forceinline__ void issue_raw(const RawOp &o, uint32_t dst, int k0, int t) {
    const int inner = o.mn_inner ? o.ext : PBK, outer = o.mn_inner ? PBK : o.ext;
    const int epc = 16 / o.es;                         // elements per 16-byte chunk
    const int cpr = inner / epc;                       // chunks per outer row
    const int nchunk = outer * cpr;
    for (int c = t; c < nchunk; c += kPT) {
        const int r = c / cpr, i0 = (c - r * cpr) * epc;
        const int og = o.mn_inner ? k0 + r : o.mn0 + r;          // global outer index
        const int ig = o.mn_inner ? o.mn0 + i0 : k0 + i0;        // global inner index
        const int olim = o.mn_inner ? o.k_lim : o.mn_lim, ilim = o.mn_inner ? o.mn_lim : o.k_lim;
        int valid = (og < olim) ? min(epc, ilim - ig) : 0;
        valid = max(valid, 0);
        const char *src = valid ? o.base + (size_t)og * o.ld_bytes + (size_t)ig * o.es : o.base;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + (uint32_t)(r * inner + i0) * o.es),
                     "l"(src), "r"((uint32_t)(valid * o.es))
                     : "memory");
    }
}

// raw slab -> fp64 tile T[k][mn] (row stride ts)
__device__ __forceinline__ void convert_raw(const RawOp &o, const char *raw, double *T, int ts, int t) {
    for (int e = t; e < o.ext * PBK; e += kPT) {
        int k, mn;
        if (o.mn_inner) { k = e / o.ext; mn = e - k * o.ext; }
        else            { mn = e / PBK; k = e % PBK; }
        const double v = o.es == 8 ? reinterpret_cast<const double *>(raw)[e]
                                   : (double)reinterpret_cast<const float *>(raw)[e];
        T[k * ts + mn] = v;
    }
}

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// kPM x BN output tile, 4 warps (warp w: columns 32 w .. 32 w + 31, all kPM rows), so two CTAs
// share an SM and one's staging/barriers overlap the other's tensor-core work.
__global__ void __launch_bounds__(kPT, 2) gemm64_pipe_kernel(const __grid_constant__ Batch64 batch) {
    // dynamic shared memory is 16-byte aligned; keep every pointer derived from the __shared__
    // symbol so the compiler emits LDS/STS (a uintptr round trip would make them generic loads)
    extern __shared__ __align__(16) double smem_d[];
    const int tile = blockIdx.x;
    const Gemm64Desc &d = batch.d[find_desc(batch, tile)];
    const int local = tile - d.tile_begin;
    const int tiles_n = (d.N + BN - 1) / BN;
    const int m0 = (local / tiles_n) * kPM, n0 = (local % tiles_n) * BN;
    const int Me = d.M, Ne = d.dyn ? min(d.N, d.dyn[0]) : d.N, Ke = d.dyn ? min(d.K, d.dyn[1]) : d.K;
    if (n0 >= Ne) return;
    if (d.lower && n0 >= m0 + kPM) return;           // block strictly above the diagonal
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    char *raw = reinterpret_cast<char *>(smem_d);
    double *tiles = smem_d + kStages * (kRawA + kRawB) / 8;     // two fp64 tile pairs (A, B)
    const uint32_t raw_s = (uint32_t)__cvta_generic_to_shared(raw);

    RawOp oa, ob;
    oa.base = static_cast<const char *>(d.A); oa.es = d.ta == DT_F64 ? 8 : 4; oa.ext = kPM;
    oa.ld_bytes = (size_t)d.lda * oa.es; oa.mn_inner = d.trans_a; oa.mn0 = m0; oa.mn_lim = Me; oa.k_lim = Ke;
    ob.base = static_cast<const char *>(d.B); ob.es = d.tb == DT_F64 ? 8 : 4; ob.ext = BN;
    ob.ld_bytes = (size_t)d.ldb * ob.es; ob.mn_inner = !d.trans_b; ob.mn0 = n0; ob.mn_lim = Ne; ob.k_lim = Ke;

    double acc[8][8];                          // [mi][2 ni + e]
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
    const int wn = warp * 32, g = lane >> 2, q = lane & 3;
    const int nk = (Ke + PBK - 1) / PBK;
    auto issue = [&](int kt) {                 // slab kt -> raw stage kt & 1
        if (kt < nk) {
            const uint32_t st = raw_s + (uint32_t)((kt & 1) * (kRawA + kRawB));
            issue_raw(oa, st, kt * PBK, t);
            issue_raw(ob, st + kRawA, kt * PBK, t);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto convert = [&](int kt) {               // raw stage kt & 1 -> tile pair kt & 1
        const char *st = raw + (kt & 1) * (kRawA + kRawB);
        double *T = tiles + (kt & 1) * kTileD;
        convert_raw(oa, st, T, kTsA, t);
        convert_raw(ob, st + kRawA, T + PBK * kTsA, kTsB, t);
    };
    // Software pipeline, one barrier per slab: iteration kt converts slab kt+1 (its copies landed)
    // into the other tile pair and refills the raw stage of slab kt with slab kt+2, then runs the
    // DMMAs of slab kt -- warps still converting overlap warps already multiplying.
    issue(0);
    issue(1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    if (nk > 0) convert(0);
    for (int kt = 0; kt < nk; ++kt) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");    // slab kt+1 (this thread's copies)
        __syncthreads();       // all copies of kt+1 landed; convert(kt) done; compute(kt-1) done
        if (kt + 1 < nk) convert(kt + 1);
        issue(kt + 2);                          // raw stage of slab kt: converted last iteration
        const double *As = tiles + (kt & 1) * kTileD, *Bs = As + PBK * kTsA;
#pragma unroll
        for (int kk = 0; kk < PBK; kk += 4) {
            // A fragment (8 x 4, row-major): element (g, q); B fragment (4 x 8, col): element (q, g)
            double a[8], b[4];
#pragma unroll
            for (int mi = 0; mi < 8; ++mi) a[mi] = As[(kk + q) * kTsA + mi * 8 + g];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(kk + q) * kTsB + wn + ni * 8 + g];
#pragma unroll
            for (int mi = 0; mi < 8; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][2 * ni], acc[mi][2 * ni + 1], a[mi], b[ni]);
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    // accumulator (mi, ni): rows 8 mi + g, columns wn + 8 ni + 2 q + {0, 1}
    int rows[8], cols[4];
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) rows[mi] = m0 + mi * 8 + g;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) cols[ni] = n0 + wn + ni * 8 + 2 * q;
    epilogue(d, Me, Ne, rows, cols, acc);
}

// ------------------------------------------------ all-fp64 direct DMMA kernel --
// Both operands fp64 (divide and conquer, back-transformation): the cp.async stages are laid out
// so that the DMMA fragments are loaded straight from them -- no conversion pass.  Row strides are
// padded (K-contiguous rows: 18 doubles; MN-contiguous rows: 64 + 4 / 128 + 8 doubles) so every
// 8x4 fragment load touches each bank exactly twice (two wavefronts, the minimum for 256 B).
// Three stages: slab kt is multiplied while kt+1 lands and kt+2 is being issued.
constexpr int kDS = 3;
constexpr int kSAk = PBK + 2, kSAm = kPM + 4, kSBk = PBK + 2, kSBn = BN + 8;
constexpr int kDA = (kPM * kSAk > PBK * kSAm) ? kPM * kSAk : PBK * kSAm;       // doubles per A slab
constexpr int kDB = (BN * kSBk > PBK * kSBn) ? BN * kSBk : PBK * kSBn;         // doubles per B slab
constexpr int kDirectSmem = kDS * (kDA + kDB) * 8 + 64;

__device__ __forceinline__ void issue_direct(const double *base, size_t ld, int mn_inner, int ext, int stride,
                                             int mn0, int mn_lim, int k0, int k_lim, uint32_t dst, int t) {
    const int inner = mn_inner ? ext : PBK, outer = mn_inner ? PBK : ext;
    const int cpr = inner / 2;                         // 16-byte chunks (2 doubles) per row
    for (int c = t; c < outer * cpr; c += kPT) {
        const int r = c / cpr, i0 = (c - r * cpr) * 2;
        const int og = mn_inner ? k0 + r : mn0 + r, ig = mn_inner ? mn0 + i0 : k0 + i0;
        const int olim = mn_inner ? k_lim : mn_lim, ilim = mn_inner ? mn_lim : k_lim;
        int valid = og < olim ? min(2, ilim - ig) : 0;
        valid = max(valid, 0);
        const double *src = valid ? base + (size_t)og * ld + ig : base;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + (uint32_t)(r * stride + i0) * 8),
                     "l"(src), "r"((uint32_t)(valid * 8))
                     : "memory");
    }
}

__global__ void __launch_bounds__(kPT, 2) gemm64_direct_kernel(const __grid_constant__ Batch64 batch) {
    extern __shared__ __align__(16) double smem_d[];
    const int tile = blockIdx.x;
    const Gemm64Desc &d = batch.d[find_desc(batch, tile)];
    const int local = tile - d.tile_begin;
    const int tiles_n = (d.N + BN - 1) / BN;
    const int m0 = (local / tiles_n) * kPM, n0 = (local % tiles_n) * BN;
    const int Me = d.M, Ne = d.dyn ? min(d.N, d.dyn[0]) : d.N, Ke = d.dyn ? min(d.K, d.dyn[1]) : d.K;
    if (n0 >= Ne) return;
    if (d.lower && n0 >= m0 + kPM) return;
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_d);
    const double *A = static_cast<const double *>(d.A), *Bm = static_cast<const double *>(d.B);
    const int a_mn = d.trans_a, b_mn = !d.trans_b;
    const int sa = a_mn ? kSAm : kSAk, sb = b_mn ? kSBn : kSBk;

    double acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
    const int wn = warp * 32, g = lane >> 2, q = lane & 3;
    const int nk = (Ke + PBK - 1) / PBK;
    auto issue = [&](int kt) {
        if (kt < nk) {
            const int st = kt % kDS;
            const uint32_t da = sbase + (uint32_t)(st * (kDA + kDB)) * 8;
            issue_direct(A, (size_t)d.lda, a_mn, kPM, sa, m0, Me, kt * PBK, Ke, da, t);
            issue_direct(Bm, (size_t)d.ldb, b_mn, BN, sb, n0, Ne, kt * PBK, Ke, da + kDA * 8, t);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // K slabs below dyn[2] multiply known zeros (divide-and-conquer column types): skipped
    const int kt0 = (d.dyn && d.dyn_koff) ? min(max(d.dyn[2], 0), Ke) / PBK : 0;
    issue(kt0);
    issue(kt0 + 1);
    for (int kt = kt0; kt < nk; ++kt) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");      // slab kt (this thread's copies)
        __syncthreads();                        // slab kt landed everywhere; compute(kt-1) done
        issue(kt + 2);                          // into the stage of slab kt-1
        const double *As = smem_d + (kt % kDS) * (kDA + kDB), *Bs = As + kDA;
#pragma unroll
        for (int kk = 0; kk < PBK; kk += 4) {
            double a[8], b[4];
#pragma unroll
            for (int mi = 0; mi < 8; ++mi) {
                const int m = mi * 8 + g, k = kk + q;
                a[mi] = As[a_mn ? k * kSAm + m : m * kSAk + k];
            }
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
                const int n = wn + ni * 8 + g, k = kk + q;
                b[ni] = Bs[b_mn ? k * kSBn + n : n * kSBk + k];
            }
#pragma unroll
            for (int mi = 0; mi < 8; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][2 * ni], acc[mi][2 * ni + 1], a[mi], b[ni]);
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    int rows[8], cols[4];
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) rows[mi] = m0 + mi * 8 + g;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) cols[ni] = n0 + wn + ni * 8 + 2 * q;
    epilogue(d, Me, Ne, rows, cols, acc);
}

bool direct_ok(const Gemm64Desc &g) {
    return g.ta == DT_F64 && g.tb == DT_F64 && (reinterpret_cast<uintptr_t>(g.A) % 16 == 0) &&
           (reinterpret_cast<uintptr_t>(g.B) % 16 == 0) && (g.lda % 2 == 0) && (g.ldb % 2 == 0);
}

bool pipe_ok(const Gemm64Desc &g) {
    const int ea = g.ta == DT_F64 ? 8 : 4, eb = g.tb == DT_F64 ? 8 : 4;
    return (reinterpret_cast<uintptr_t>(g.A) % 16 == 0) && (reinterpret_cast<uintptr_t>(g.B) % 16 == 0) &&
           ((size_t)g.lda * ea) % 16 == 0 && ((size_t)g.ldb * eb) % 16 == 0;
}

}  // namespace

namespace {
kfac_status_t gemm64_dmma_grouped(const Gemm64Desc *descs, int count, cudaStream_t s) {
    for (int base = 0, end = 0; base < count; base = end) {
        thread_local Batch64 b;   // host staging; parameters are copied at launch
        b.count = 0;
        end = base;
        bool pipe = true, direct = true;
        for (int i = base; i < count && b.count < kGemm64MaxDescs; ++i, ++end) {
            const Gemm64Desc &g = descs[i];
            if (g.M <= 0 || g.N <= 0) continue;
            b.d[b.count++] = g;
            pipe = pipe && pipe_ok(g);
            direct = direct && direct_ok(g);
        }
        if (b.count == 0) continue;
        const int tm = pipe ? kPM : BM;
        int tiles = 0;
        for (int i = 0; i < b.count; ++i) {
            b.d[i].tile_begin = tiles;
            tiles += cdiv(b.d[i].M, tm) * cdiv(b.d[i].N, BN);
        }
        const int prof = prof_begin(KFAC_PROF_GEMM64, s);
        if (direct) {
            KFAC_CUDA_TRY(set_smem_attr((const void *)gemm64_direct_kernel, kDirectSmem));
            gemm64_direct_kernel<<<tiles, kPT, kDirectSmem, s>>>(b);
        } else if (pipe) {
            KFAC_CUDA_TRY(set_smem_attr((const void *)gemm64_pipe_kernel, kPipeSmem));
            gemm64_pipe_kernel<<<tiles, kPT, kPipeSmem, s>>>(b);
        } else {
            gemm64_kernel<<<tiles, NT, 0, s>>>(b);
        }
        KFAC_LAUNCHED();
        if (prof >= 0) {
            double by = 0.0, fl = 0.0;
            for (int i = 0; i < b.count; ++i) {
                const Gemm64Desc &g = b.d[i];
                const double ea = g.ta == DT_F64 ? 8 : 4, eb = g.tb == DT_F64 ? 8 : 4, ec = g.tc == DT_F64 ? 8 : 4;
                const double mn = g.lower ? 0.5 * g.M * (g.N + 1.0) : (double)g.M * g.N;
                fl += 2.0 * mn * g.K;
                by += (double)g.M * g.K * ea + (double)g.N * g.K * eb + mn * ec * (g.epi == EPI_SUB ? 2 : 1);
            }
            prof_end(prof, s, by, fl);
        }
    }
    return KFAC_OK;
}
}  // namespace

kfac_status_t gemm64_grouped(const Gemm64Desc *descs, int count, cudaStream_t s) {
    if (!oz_arena_active()) return gemm64_dmma_grouped(descs, count, s);
    // Ozaki (int8 tensor cores) for the large fp64 products, DMMA for the rest
    std::vector<Gemm64Desc> oz, dm;
    for (int i = 0; i < count; ++i)
        if (descs[i].M > 0 && descs[i].N > 0) (oz_eligible(descs[i]) ? oz : dm).push_back(descs[i]);
    if (!oz.empty()) {
        kfac_status_t st = oz_gemm_grouped(oz.data(), (int)oz.size(), s);
        if (st != KFAC_OK) return st;
    }
    return dm.empty() ? KFAC_OK : gemm64_dmma_grouped(dm.data(), (int)dm.size(), s);
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
