// eigen.cu -- Stage 2 of Alg. 1: eigendecomposition of every Kronecker factor.
//
// Batched one-sided block Jacobi (Hestenes) on U = F V, V orthogonal:
//   * columns are split into blocks of 16; a parallel round-robin tournament pairs the blocks so
//     every round is a set of disjoint 32-column pairs (one CTA each, all factors batched);
//   * per pair: Gram G = U_pq^T U_pq, its 32x32 eigenproblem G = R D R^T solved by cyclic
//     Jacobi in shared memory, then U_pq <- U_pq R and V_pq <- V_pq R -- all in fp64 with U, V
//     stored in fp64, so U = F V holds to fp64 rounding and the null-space eigenvectors of
//     rank-deficient factors are not polluted by fp32 drift (ResNet-50 fc at 32 rows/GPU);
//   * a pair whose columns are already orthogonal to tol is skipped; a sweep with no rotation
//     marks the factor converged (device flag, no host synchronisation);
//   * at the end eigenvalues are Rayleigh quotients v_j^T u_j = v_j^T F v_j (fp64), clamped at 0
//     (R10), and (Q, v) are sorted ascending and rounded to fp32.
// Why Jacobi: fully parallel across pairs and factors, robust to the
// huge zero-eigenvalue clusters of rank-deficient conv factors (R11), and warm-startable from
// the previous (stale) eigenbasis (KFAC_EIG_WARM_START).
#include "internal.cuh"

#include <algorithm>
#include <vector>

namespace kfac {

size_t eigen_workspace_bytes(const int32_t *dims, int count);
size_t trd_workspace_bytes(const int32_t *dims, int count);
kfac_status_t trd_run(const float *const *F, const int32_t *dims, const int32_t *ldF, int count,
                      float *const *Q, const int32_t *ldQ, float *const *evals, int32_t *info, uint32_t flags,
                      void *ws, cudaStream_t s);
kfac_status_t eigen_run(const float *const *F, const int32_t *dims, const int32_t *ldF, int count,
                        float *const *Q, const int32_t *ldQ, float *const *evals, int32_t *info,
                        uint32_t flags, void *ws, cudaStream_t s);

namespace {

constexpr int B = 16;            // columns per block
constexpr int P = 2 * B;         // columns per pair
constexpr int NT = 256;
constexpr int kMaxSweeps = 16;
constexpr int kTableChunk = 48;
constexpr int kInnerSweeps = 3;

struct EigJob {
    const float *F;
    float *Q;
    float *evals;
    double *U;       // n x ldu  (U = F V)
    double *V;       // n x ldu
    double *lam;     // n
    int *rank;       // n
    int *info;       // device (caller)
    int n, ldF, ldQ, ldu, nb;      // nb: number of blocks incl. the dummy (even)
    int pair_begin;                // prefix over jobs (sorted by nb descending)
    int rot_count, converged, sweeps;
    float scale;                   // ||F||_F (>= ||F||_2)
};

struct EigTableInit {
    EigJob *table;
    int count, base;
    EigJob j[kTableChunk];
};

__global__ void eig_table_init(const __grid_constant__ EigTableInit t) {
    int i = threadIdx.x;
    if (i < t.count) t.table[t.base + i] = t.j[i];
}

// U = (F + F^T)/2 (or keep U from the warm-start GEMM), V = I (or Q_in); pads zeroed; scale = ||F||_F.
__global__ void eig_init(EigJob *table, int warm) {
    EigJob &J = table[blockIdx.y];
    const int n = J.n, ldu = J.ldu;
    const long long total = (long long)n * ldu;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(e / ldu), c = (int)(e % ldu);
        if (!warm) {
            double u = 0.0;
            if (c < n) u = 0.5 * ((double)J.F[(size_t)r * J.ldF + c] + (double)J.F[(size_t)c * J.ldF + r]);
            J.U[e] = u;
            J.V[e] = (r == c) ? 1.0 : 0.0;
        } else {
            J.V[e] = (c < n) ? (double)J.Q[(size_t)r * J.ldQ + c] : 0.0;
            if (c >= n) J.U[e] = 0.0;
        }
    }
    if (blockIdx.x == 0) {
        __shared__ double red[NT];
        double s = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) s += J.lam[i];   // row sums of squares
        red[threadIdx.x] = s;
        __syncthreads();
        for (int w = NT / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            J.scale = (float)sqrt(red[0]);
            J.rot_count = 0;
            J.converged = 0;
            J.sweeps = 0;
        }
    }
}

// lam[r] = sum_c F[r][c]^2 (one warp per row, fixed order) -- feeds ||F||_F in eig_init.
__global__ void eig_rownorm(EigJob *table) {
    EigJob &J = table[blockIdx.y];
    const int r = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (r >= J.n) return;
    double s = 0.0;
    for (int c = lane; c < J.n; c += 32) {
        const double x = J.F[(size_t)r * J.ldF + c];
        s += x * x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) J.lam[r] = s;
}

// Round-robin ("circle") tournament: pair k of round r among m players (m even).
__device__ __forceinline__ void circle_pair(int r, int k, int m, int &a, int &b) {
    if (k == 0) { a = m - 1; b = r % (m - 1); }
    else { a = (r + k) % (m - 1); b = (r - k + (m - 1)) % (m - 1); }
}

__device__ __forceinline__ void schur2(double app, double aqq, double apq, double &c, double &s) {
    // G&VL Alg. 8.4.1 (sym.schur2): J(p,q,theta)^T A J zeroes A_pq.
    const double tau = (aqq - app) / (2.0 * apq);
    const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
    c = 1.0 / sqrt(1.0 + t * t);
    s = t * c;
}

constexpr int kRowsPerIter = 16;                         // rows each warp stages per iteration
constexpr size_t kRoundSmem = sizeof(double) * (NT / 32) * P * (P + 1);

__global__ void __launch_bounds__(NT, 2) eig_round(const EigJob *__restrict__ table, int count, int round,
                                                   float tol, float tol_abs) {
    extern __shared__ double dsm[];
    double(*Gp)[P][P + 1] = reinterpret_cast<double(*)[P][P + 1]>(dsm);       // [8 warps] partial Grams
    double(*G)[P + 1] = Gp[0];                                                  // reduced Gram (reuses slot 0)
    __shared__ double R[P][P + 1];
    __shared__ double rows[NT / 32][kRowsPerIter][P];
    __shared__ double cs_c[P / 2], cs_s[P / 2];
    __shared__ int cs_i[P / 2], cs_j[P / 2];
    __shared__ double gmax;

    // locate the job (table sorted by nb descending; pair_begin is a prefix sum)
    int lo = 0, hi = count - 1;
    const int item = blockIdx.x;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (table[mid].pair_begin <= item) lo = mid; else hi = mid - 1;
    }
    const EigJob *Jp = table + lo;
    if (Jp->converged || round >= Jp->nb - 1) return;
    const int k = item - Jp->pair_begin;
    const int nb = Jp->nb;
    if (k >= nb / 2) return;
    const int n = Jp->n, ldu = Jp->ldu;
    double *const U = Jp->U;
    double *const V = Jp->V;
    const double fro = (double)Jp->scale;
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    const int nb_real = (n + B - 1) / B;
    int a, b;
    circle_pair(round, k, nb, a, b);
    const int c0 = a < nb_real ? a * B : -1, c1 = b < nb_real ? b * B : -1;   // -1: dummy block
    // lane l owns column col(l) of the pair: block p for l < 16, block q for l >= 16
    const int mycol = lane < B ? (c0 >= 0 ? c0 + lane : -1) : (c1 >= 0 ? c1 + lane - B : -1);

    // ---- Gram: every warp accumulates G_w = sum over its rows of u_r u_r^T (lane l: row l of G_w)
    double g[P];
#pragma unroll
    for (int j = 0; j < P; ++j) g[j] = 0.0;
    for (int r0 = warp * kRowsPerIter; r0 < n; r0 += NT / 32 * kRowsPerIter) {
        double ld[kRowsPerIter];                            // all loads in flight before any store
#pragma unroll
        for (int i = 0; i < kRowsPerIter; ++i) {
            const int r = r0 + i;
            ld[i] = (r < n && mycol >= 0) ? __ldg(U + (size_t)r * ldu + mycol) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < kRowsPerIter; ++i) rows[warp][i][lane] = ld[i];
        __syncwarp();
#pragma unroll
        for (int i = 0; i < kRowsPerIter; ++i) {
            const double x = rows[warp][i][lane];
#pragma unroll
            for (int j = 0; j < P; j += 2) {
                const double2 y = *reinterpret_cast<const double2 *>(&rows[warp][i][j]);
                g[j] = fma(x, y.x, g[j]);
                g[j + 1] = fma(x, y.y, g[j + 1]);
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int j = 0; j < P; ++j) Gp[warp][lane][j] = g[j];
    __syncthreads();
    for (int e = t; e < P * P; e += NT) {                   // fixed-order reduction over warps
        const int i = e / P, j = e % P;
        double v = Gp[0][i][j];
#pragma unroll
        for (int w = 1; w < NT / 32; ++w) v += Gp[w][i][j];
        Gp[0][i][j] = v;
        R[i][j] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (t < P * P) {                                        // exact symmetry from the upper triangle
        const int i = t / P, j = t % P;
        if (i > j) G[i][j] = G[j][i];
    }
    if (t == 0) {
        double m = 0.0;
        for (int i = 0; i < P; ++i) m = fmax(m, G[i][i]);
        gmax = m;
    }
    __syncthreads();

    // ---- convergence test of this pair: rotate only if some coupling exceeds both the relative
    // bound tol ||u_i|| ||u_j|| and the absolute level tol_abs ||F|| (||u_i|| + ||u_j||).
    int need = 0;
    for (int e = t; e < P * P; e += NT) {
        const int i = e / P, j = e % P;
        if (i >= j) continue;
        const double gg = fabs(G[i][j]);
        const double ni = sqrt(G[i][i]), nj = sqrt(G[j][j]);
        if (gg > tol * ni * nj && gg > tol_abs * fro * (ni + nj)) need = 1;
    }
    if (!__syncthreads_or(need)) return;

    // ---- inner cyclic Jacobi on the 32x32 Gram (fp64, shared memory) ----
    const double inner_abs = 1e-15 * gmax;
    for (int sweep = 0; sweep < kInnerSweeps; ++sweep) {
        int rotated = 0;
        for (int ir = 0; ir < P - 1; ++ir) {
            if (t < P / 2) {
                int i, j;
                circle_pair(ir, t, P, i, j);
                const double gij = G[i][j], gii = G[i][i], gjj = G[j][j];
                double c = 1.0, sn = 0.0;
                if (fabs(gij) > 1e-12 * sqrt(fabs(gii * gjj)) && fabs(gij) > inner_abs) {
                    schur2(gii, gjj, gij, c, sn);
                    rotated = 1;
                }
                cs_i[t] = i; cs_j[t] = j; cs_c[t] = c; cs_s[t] = sn;
            }
            __syncthreads();
            for (int e = t; e < (P / 2) * P * 2; e += NT) {        // columns of G and R
                const int which = e / ((P / 2) * P);
                const int e2 = e % ((P / 2) * P);
                const int kk = e2 / P, r = e2 % P;
                const double c = cs_c[kk], sn = cs_s[kk];
                if (sn == 0.0) continue;
                double(*M)[P + 1] = which ? R : G;
                const int i = cs_i[kk], j = cs_j[kk];
                const double x = M[r][i], y = M[r][j];
                M[r][i] = c * x - sn * y;
                M[r][j] = sn * x + c * y;
            }
            __syncthreads();
            for (int e = t; e < (P / 2) * P; e += NT) {            // rows of G
                const int kk = e / P, r = e % P;
                const double c = cs_c[kk], sn = cs_s[kk];
                if (sn == 0.0) continue;
                const int i = cs_i[kk], j = cs_j[kk];
                const double x = G[i][r], y = G[j][r];
                G[i][r] = c * x - sn * y;
                G[j][r] = sn * x + c * y;
            }
            __syncthreads();
        }
        if (!__syncthreads_or(rotated)) break;
    }
    if (t == 0) atomicAdd(const_cast<int *>(&Jp->rot_count), 1);

    // ---- apply: U_pq <- U_pq R and V_pq <- V_pq R (lane l computes column l; rows broadcast) ----
    double rc[P];
#pragma unroll
    for (int kk = 0; kk < P; ++kk) rc[kk] = R[kk][lane];
    for (int w = 0; w < 2; ++w) {
        double *M = w ? V : U;
        for (int r0 = warp * kRowsPerIter; r0 < n; r0 += NT / 32 * kRowsPerIter) {
            double ld[kRowsPerIter];
#pragma unroll
            for (int i = 0; i < kRowsPerIter; ++i) {
                const int r = r0 + i;
                ld[i] = (r < n && mycol >= 0) ? M[(size_t)r * ldu + mycol] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < kRowsPerIter; ++i) rows[warp][i][lane] = ld[i];
            __syncwarp();
#pragma unroll
            for (int i = 0; i < kRowsPerIter; ++i) {
                double y = 0.0;
#pragma unroll
                for (int kk = 0; kk < P; kk += 2) {
                    const double2 x = *reinterpret_cast<const double2 *>(&rows[warp][i][kk]);
                    y = fma(x.x, rc[kk], y);
                    y = fma(x.y, rc[kk + 1], y);
                }
                const int r = r0 + i;
                if (r < n && mycol >= 0) M[(size_t)r * ldu + mycol] = y;
            }
            __syncwarp();
        }
    }
}

// Warm start: U = F V in fp64 (64x64 tile per CTA, 4x4 per thread).
__global__ void __launch_bounds__(256) eig_fv(EigJob *table) {
    __shared__ double Fs[16][65];
    __shared__ double Vs[16][65];
    EigJob &J = table[blockIdx.z];
    const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
    if (m0 >= J.n || n0 >= J.n) return;
    const int t = threadIdx.x, ty = t / 16, tx = t % 16;
    double acc[4][4] = {};
    const int n = J.n, ldF = J.ldF, ldu = J.ldu;
    const float *__restrict__ F = J.F;
    const double *__restrict__ Vg = J.V;
    for (int k0 = 0; k0 < n; k0 += 16) {
        float fv[4];
        double vv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {                           // loads first, then shared stores
            const int e = t + 256 * q;
            const int mm = e / 16, kk = e % 16;                 // F[m][k] (k fastest)
            const int m = m0 + mm, k = k0 + kk;
            fv[q] = (m < n && k < n) ? __ldg(F + (size_t)m * ldF + k) : 0.f;
            const int kv = e / 64, nn = e % 64;                 // V[k][n] (n fastest)
            vv[q] = (k0 + kv < n && n0 + nn < n) ? __ldg(Vg + (size_t)(k0 + kv) * ldu + n0 + nn) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = t + 256 * q;
            Fs[e % 16][e / 16] = (double)fv[q];
            Vs[e / 64][e % 64] = vv[q];
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < 16; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) { a[i] = Fs[kk][ty + 16 * i]; b[i] = Vs[kk][tx + 16 * i]; }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
            if (m < J.n && n < J.n) J.U[(size_t)m * J.ldu + n] = acc[i][j];
        }
}

__global__ void eig_sweep_end(EigJob *table, int count) {
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        EigJob &J = table[i];
        if (J.converged) continue;
        J.sweeps += 1;
        if (J.rot_count == 0) J.converged = 1;
        J.rot_count = 0;
    }
}

// lam_j = v_j^T u_j = v_j^T F v_j (U = F V is exact to fp64 rounding).
__global__ void eig_rayleigh(EigJob *table) {
    EigJob &J = table[blockIdx.y];
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= J.n) return;
    double s = 0.0;
    for (int r = 0; r < J.n; ++r)
        s += J.V[(size_t)r * J.ldu + j] * J.U[(size_t)r * J.ldu + j];
    J.lam[j] = s;
}

__global__ void eig_rank(EigJob *table) {
    __shared__ double lt[256];
    EigJob &J = table[blockIdx.y];
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const double lj = j < J.n ? J.lam[j] : 0.0;
    int rank = 0;
    for (int b0 = 0; b0 < J.n; b0 += 256) {
        __syncthreads();
        if (b0 + threadIdx.x < J.n) lt[threadIdx.x] = J.lam[b0 + threadIdx.x];
        __syncthreads();
        const int m = min(256, J.n - b0);
        for (int i = 0; i < m; ++i) {
            const double li = lt[i];
            rank += (li < lj) || (li == lj && b0 + i < j);
        }
    }
    if (j < J.n) {
        J.rank[j] = rank;
        J.evals[rank] = (float)fmax(lj, 0.0);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && J.info) *J.info = J.converged ? 0 : J.sweeps;
}

__global__ void eig_scatter(EigJob *table) {
    EigJob &J = table[blockIdx.z];
    const int r = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= J.n || j >= J.n) return;
    J.Q[(size_t)r * J.ldQ + J.rank[j]] = (float)J.V[(size_t)r * J.ldu + j];
}

struct Layout {
    std::vector<EigJob> jobs;      // in caller order
    std::vector<int> order;        // sorted by nb descending
    size_t bytes = 0;
    size_t table_off = 0;
};

Layout plan(const int32_t *dims, int count) {
    Layout L;
    L.jobs.resize(count);
    size_t off = 0;
    auto take = [&](size_t bytes) { off = round_up(off, 256); size_t o = off; off += bytes; return o; };
    L.table_off = take(sizeof(EigJob) * count);
    for (int i = 0; i < count; ++i) {
        EigJob &J = L.jobs[i];
        J = EigJob{};
        J.n = dims[i];
        const int nb_real = cdiv(J.n, B);
        J.nb = nb_real + (nb_real & 1);
        J.ldu = nb_real * B;
        J.U = reinterpret_cast<double *>(take(sizeof(double) * (size_t)J.n * J.ldu));
        J.V = reinterpret_cast<double *>(take(sizeof(double) * (size_t)J.n * J.ldu));
        J.lam = reinterpret_cast<double *>(take(sizeof(double) * J.n));
        J.rank = reinterpret_cast<int *>(take(sizeof(int) * J.n));
    }
    L.bytes = off + 256;
    L.order.resize(count);
    for (int i = 0; i < count; ++i) L.order[i] = i;
    std::stable_sort(L.order.begin(), L.order.end(),
                     [&](int a, int b) { return L.jobs[a].nb > L.jobs[b].nb; });
    return L;
}

}  // namespace

namespace {

size_t jacobi_bytes(const int32_t *dims, int count) { return plan(dims, count).bytes; }

kfac_status_t jacobi_run(const float *const *F, const int32_t *dims, const int32_t *ldF, int count,
                         float *const *Q, const int32_t *ldQ, float *const *evals, int32_t *info,
                         uint32_t flags, void *ws, cudaStream_t s) {
    Layout L = plan(dims, count);
    char *base = reinterpret_cast<char *>(round_up(reinterpret_cast<uintptr_t>(ws), 256));
    EigJob *table = reinterpret_cast<EigJob *>(base + L.table_off);
    std::vector<EigJob> sorted(count);
    int pairs = 0;
    for (int k = 0; k < count; ++k) {
        const int i = L.order[k];
        EigJob J = L.jobs[i];
        J.F = F[i]; J.Q = Q[i]; J.evals = evals[i];
        J.info = info ? info + i : nullptr;
        J.ldF = ldF[i]; J.ldQ = ldQ[i];
        J.U = reinterpret_cast<double *>(base + reinterpret_cast<uintptr_t>(J.U));
        J.V = reinterpret_cast<double *>(base + reinterpret_cast<uintptr_t>(J.V));
        J.lam = reinterpret_cast<double *>(base + reinterpret_cast<uintptr_t>(J.lam));
        J.rank = reinterpret_cast<int *>(base + reinterpret_cast<uintptr_t>(J.rank));
        J.pair_begin = pairs;
        pairs += J.nb / 2;
        sorted[k] = J;
    }
    for (int b0 = 0; b0 < count; b0 += kTableChunk) {
        EigTableInit ti;
        ti.table = table;
        ti.base = b0;
        ti.count = std::min(kTableChunk, count - b0);
        for (int i = 0; i < ti.count; ++i) ti.j[i] = sorted[b0 + i];
        eig_table_init<<<1, 64, 0, s>>>(ti);
        KFAC_LAUNCHED();
    }
    KFAC_CUDA_TRY(set_smem_attr((const void *)eig_round, (int)kRoundSmem));
    const bool warm = flags & KFAC_EIG_WARM_START;
    int max_n = 0;
    for (auto &J : sorted) max_n = std::max(max_n, J.n);
    eig_rownorm<<<dim3(cdiv(max_n, 8), count), 256, 0, s>>>(table);
    KFAC_LAUNCHED();
    eig_init<<<dim3(std::min(1024, cdiv((long long)max_n * max_n, NT)), count), NT, 0, s>>>(table, warm);
    KFAC_LAUNCHED();
    if (warm) {   // U = F * V (fp64), V = Q_in
        const int tiles = cdiv(max_n, 64);
        eig_fv<<<dim3(tiles, tiles, count), 256, 0, s>>>(table);
        KFAC_LAUNCHED();
    }
    // Sweeps: all rounds of all factors, factors sorted so that active pairs form a prefix.
    const int max_rounds = sorted[0].nb - 1;
    const float tol = 1e-7f, tol_abs = 1e-8f;
    for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
        for (int r = 0; r < max_rounds; ++r) {
            int active = 0;
            for (auto &J : sorted) if (J.nb - 1 > r) active = J.pair_begin + J.nb / 2;
            eig_round<<<active, NT, kRoundSmem, s>>>(table, count, r, tol, tol_abs);
            KFAC_LAUNCHED();
        }
        eig_sweep_end<<<1, 256, 0, s>>>(table, count);
        KFAC_LAUNCHED();
    }
    eig_rayleigh<<<dim3(cdiv(max_n, 128), count), 128, 0, s>>>(table);
    KFAC_LAUNCHED();
    eig_rank<<<dim3(cdiv(max_n, 256), count), 256, 0, s>>>(table);
    KFAC_LAUNCHED();
    eig_scatter<<<dim3(cdiv(max_n, 128), max_n, count), 128, 0, s>>>(table);
    KFAC_LAUNCHED();
    return KFAC_OK;
}

// Factors of order >= kTrdMinDim go to the tridiagonal solver (Jacobi for d = 300/600/1200 measured
// +6/+29/+122 ms on ResNet-50).
constexpr int kTrdMinDim = 64;

bool use_trd(int n, uint32_t flags) {
    if (flags & KFAC_EIG_JACOBI) return false;
    if (flags & KFAC_EIG_TRIDIAG) return true;
    return n >= kTrdMinDim;
}

}  // namespace

namespace {
struct InfoScatter {
    int count;
    int idx[2000];
};
__global__ void eig_info_scatter(const int32_t *local, int32_t *info, const __grid_constant__ InfoScatter p) {
    for (int q = threadIdx.x; q < p.count; q += blockDim.x) info[p.idx[q]] = local[q];
}
kfac_status_t scatter_info(const int32_t *local, const std::vector<int> &idx, int32_t *info, cudaStream_t s) {
    for (size_t b = 0; b < idx.size(); b += 2000) {
        InfoScatter p;
        p.count = (int)std::min<size_t>(2000, idx.size() - b);
        for (int q = 0; q < p.count; ++q) p.idx[q] = idx[b + q];
        eig_info_scatter<<<1, 256, 0, s>>>(local + b, info, p);
        KFAC_LAUNCHED();
    }
    return KFAC_OK;
}
}  // namespace

// Workspace covers both methods (the method split depends on flags, the size only on dims).
size_t eigen_workspace_bytes(const int32_t *dims, int count) {
    return round_up(jacobi_bytes(dims, count), 256) + round_up(trd_workspace_bytes(dims, count), 256) +
           sizeof(int32_t) * count + 512;
}

kfac_status_t eigen_run(const float *const *F, const int32_t *dims, const int32_t *ldF, int count,
                        float *const *Q, const int32_t *ldQ, float *const *evals, int32_t *info,
                        uint32_t flags, void *ws, cudaStream_t s) {
    std::vector<const float *> jF, tF;
    std::vector<int32_t> jd, td, jl, tl, jlq, tlq;
    std::vector<float *> jQ, tQ, je, te;
    std::vector<int> jidx, tidx;
    for (int i = 0; i < count; ++i) {
        const bool t = use_trd(dims[i], flags);
        (t ? tF : jF).push_back(F[i]);
        (t ? td : jd).push_back(dims[i]);
        (t ? tl : jl).push_back(ldF[i]);
        (t ? tQ : jQ).push_back(Q[i]);
        (t ? tlq : jlq).push_back(ldQ[i]);
        (t ? te : je).push_back(evals[i]);
        (t ? tidx : jidx).push_back(i);
    }
    // Each method reports into its own int array at the end of the workspace; one scatter
    // kernel per method moves the codes to the caller's (caller-ordered) info array.
    char *base = static_cast<char *>(ws);
    const size_t joff = round_up(jacobi_bytes(dims, count), 256);
    int32_t *local = reinterpret_cast<int32_t *>(base + joff + round_up(trd_workspace_bytes(dims, count), 256));
    // the Jacobi factors (d < 64) and the tridiagonal path share nothing (disjoint workspace and
    // info slots): the Jacobi sweeps run on a side stream next to the reduction
    SideFork fk;
    const bool par = !jd.empty() && !td.empty();
    if (par) KFAC_CUDA_TRY(fk.fork(s, 1));
    if (!jd.empty()) {
        const cudaStream_t js = par ? fk.side(0) : s;
        kfac_status_t st = jacobi_run(jF.data(), jd.data(), jl.data(), (int)jd.size(), jQ.data(), jlq.data(),
                                      je.data(), local, flags & KFAC_EIG_WARM_START, base, js);
        if (st != KFAC_OK) return st;
        if (info) {
            st = scatter_info(local, jidx, info, js);
            if (st != KFAC_OK) return st;
        }
    }
    if (!td.empty()) {
        kfac_status_t st = trd_run(tF.data(), td.data(), tl.data(), (int)td.size(), tQ.data(), tlq.data(),
                                   te.data(), local + jd.size(), flags, base + joff, s);
        if (st != KFAC_OK) return st;
        if (info) {
            st = scatter_info(local + jd.size(), tidx, info, s);
            if (st != KFAC_OK) return st;
        }
    }
    if (par) KFAC_CUDA_TRY(fk.join(s));
    return KFAC_OK;
}


}  // namespace kfac
