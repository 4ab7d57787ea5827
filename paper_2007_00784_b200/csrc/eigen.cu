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
kfac_status_t eigen_run(const float *const *F, const int32_t *dims, const int32_t *ldF, int count,
                        float *const *Q, const int32_t *ldQ, float *const *evals, int32_t *info,
                        uint32_t flags, void *ws, cudaStream_t s);

namespace {

constexpr int B = 16;            // columns per block
constexpr int P = 2 * B;         // columns per pair
constexpr int NT = 256;
constexpr int kMaxSweeps = 16;
constexpr int kTableChunk = 48;
constexpr int kInnerSweeps = 6;

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

__global__ void __launch_bounds__(NT, 2) eig_round(EigJob *table, int count, int round, float tol,
                                                float tol_abs) {
    __shared__ double tile[32][P + 1];
    __shared__ double G[P][P + 1];
    __shared__ double R[P][P + 1];
    __shared__ double cs_c[P / 2], cs_s[P / 2];
    __shared__ int cs_i[P / 2], cs_j[P / 2];
    __shared__ int col0[2];

    // locate the job (table sorted by nb descending; pair_begin is a prefix sum)
    int lo = 0, hi = count - 1;
    const int item = blockIdx.x;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (table[mid].pair_begin <= item) lo = mid; else hi = mid - 1;
    }
    EigJob &J = table[lo];
    if (J.converged || round >= J.nb - 1) return;
    const int k = item - J.pair_begin;
    if (k >= J.nb / 2) return;
    const int t = threadIdx.x;
    const int n = J.n, ldu = J.ldu;
    const int nb_real = (n + B - 1) / B;
    if (t == 0) {
        int a, b;
        circle_pair(round, k, J.nb, a, b);
        col0[0] = a < nb_real ? a * B : -1;     // -1: dummy block (no columns)
        col0[1] = b < nb_real ? b * B : -1;
    }
    __syncthreads();
    const int c0 = col0[0], c1 = col0[1];

    // ---- Gram G = U_pq^T U_pq (fp64): thread t owns the 2x2 block (2*(t/16), 2*(t%16)) ----
    const int gi = 2 * (t / 16), gj = 2 * (t % 16);
    double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
    for (int r0 = 0; r0 < n; r0 += 32) {
        for (int e = t; e < 32 * (P / 2); e += NT) {       // 32 rows x 16 double2
            const int rr = e / (P / 2), g = e % (P / 2);
            const int r = r0 + rr;
            const int cb = (g < B / 2) ? c0 : c1;
            double2 v = make_double2(0.0, 0.0);
            if (r < n && cb >= 0) v = *reinterpret_cast<const double2 *>(J.U + (size_t)r * ldu + cb + (g % (B / 2)) * 2);
            tile[rr][2 * g] = v.x;
            tile[rr][2 * g + 1] = v.y;
        }
        __syncthreads();
        const int rows = min(32, n - r0);
        for (int rr = 0; rr < rows; ++rr) {
            const double x0 = tile[rr][gi], x1 = tile[rr][gi + 1];
            const double y0 = tile[rr][gj], y1 = tile[rr][gj + 1];
            a00 = fma(x0, y0, a00); a01 = fma(x0, y1, a01);
            a10 = fma(x1, y0, a10); a11 = fma(x1, y1, a11);
        }
        __syncthreads();
    }
    G[gi][gj] = a00; G[gi][gj + 1] = a01; G[gi + 1][gj] = a10; G[gi + 1][gj + 1] = a11;
    for (int e = t; e < P * P; e += NT) R[e / P][e % P] = (e / P == e % P) ? 1.0 : 0.0;
    __syncthreads();
    if (t < P * P / 2) {                                   // exact symmetry: upper copies to lower
        const int i = t / P, j = t % P;
        if (i > j) G[i][j] = G[j][i];
    }
    __syncthreads();

    // ---- convergence test of this pair.  Rotate (i, j) only if the coupling exceeds both the
    // relative bound tol * ||u_i|| ||u_j|| and the fp32 backward-error level tol_abs ||F|| (||u_i|| +
    // ||u_j||): below it the coupling is indistinguishable from rounding of F itself.
    const double fro = (double)J.scale;
    int need = 0;
    for (int e = t; e < P * P; e += NT) {
        const int i = e / P, j = e % P;
        if (i >= j) continue;
        const double g = fabs(G[i][j]);
        const double ni = sqrt(G[i][i]), nj = sqrt(G[j][j]);
        if (g > tol * ni * nj && g > tol_abs * fro * (ni + nj)) need = 1;
    }
    need = __syncthreads_or(need);
    if (!need) return;

    // ---- inner cyclic Jacobi on the 32x32 Gram (fp64, shared memory) ----
    __shared__ double gmax;
    if (t == 0) {
        double m = 0.0;
        for (int i = 0; i < P; ++i) m = fmax(m, G[i][i]);
        gmax = m;
    }
    __syncthreads();
    const double inner_abs = 1e-15 * gmax;
    for (int sweep = 0; sweep < kInnerSweeps; ++sweep) {
        int rotated = 0;
        for (int ir = 0; ir < P - 1; ++ir) {
            if (t < P / 2) {
                int i, j;
                circle_pair(ir, t, P, i, j);
                const double gij = G[i][j], gii = G[i][i], gjj = G[j][j];
                double c = 1.0, s = 0.0;
                if (fabs(gij) > 1e-12 * sqrt(fabs(gii * gjj)) && fabs(gij) > inner_abs) {
                    schur2(gii, gjj, gij, c, s);
                    rotated = 1;
                }
                cs_i[t] = i; cs_j[t] = j; cs_c[t] = c; cs_s[t] = s;
            }
            __syncthreads();
            for (int e = t; e < (P / 2) * P * 2; e += NT) {        // columns of G and R
                const int which = e / ((P / 2) * P);
                const int e2 = e % ((P / 2) * P);
                const int kk = e2 / P, r = e2 % P;
                const double c = cs_c[kk], s = cs_s[kk];
                if (s == 0.0) continue;
                double(*M)[P + 1] = which ? R : G;
                const int i = cs_i[kk], j = cs_j[kk];
                const double x = M[r][i], y = M[r][j];
                M[r][i] = c * x - s * y;
                M[r][j] = s * x + c * y;
            }
            __syncthreads();
            for (int e = t; e < (P / 2) * P; e += NT) {            // rows of G
                const int kk = e / P, r = e % P;
                const double c = cs_c[kk], s = cs_s[kk];
                if (s == 0.0) continue;
                const int i = cs_i[kk], j = cs_j[kk];
                const double x = G[i][r], y = G[j][r];
                G[i][r] = c * x - s * y;
                G[j][r] = s * x + c * y;
            }
            __syncthreads();
        }
        if (!__syncthreads_or(rotated)) break;
    }
    if (t == 0) atomicAdd(&J.rot_count, 1);
    __syncthreads();

    // ---- apply: U_pq <- U_pq R, V_pq <- V_pq R (fp64; one row per thread, R broadcast) ----
    for (int w = 0; w < 2; ++w) {
        double *M = w ? J.V : J.U;
        for (int r = t; r < n; r += NT) {
            double x[P];
#pragma unroll
            for (int g = 0; g < P / 2; ++g) {
                const int cb = (g < B / 2) ? c0 : c1;
                double2 v = make_double2(0.0, 0.0);
                if (cb >= 0) v = *reinterpret_cast<const double2 *>(M + (size_t)r * ldu + cb + (g % (B / 2)) * 2);
                x[2 * g] = v.x;
                x[2 * g + 1] = v.y;
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {                 // output block p (h = 0) then q (h = 1)
                const int cb = h ? c1 : c0;
                double y[B];
#pragma unroll
                for (int j = 0; j < B; ++j) y[j] = 0.0;
#pragma unroll
                for (int i = 0; i < P; ++i)
#pragma unroll
                    for (int j = 0; j < B; ++j) y[j] = fma(x[i], R[i][h * B + j], y[j]);
                if (cb >= 0) {
#pragma unroll
                    for (int g = 0; g < B / 2; ++g)
                        *reinterpret_cast<double2 *>(M + (size_t)r * ldu + cb + 2 * g) = make_double2(y[2 * g], y[2 * g + 1]);
                }
            }
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
    for (int k0 = 0; k0 < J.n; k0 += 16) {
        for (int e = t; e < 16 * 64; e += 256) {
            const int mm = e / 16, kk = e % 16;                 // F[m][k] (k fastest)
            const int m = m0 + mm, k = k0 + kk;
            Fs[kk][mm] = (m < J.n && k < J.n) ? (double)J.F[(size_t)m * J.ldF + k] : 0.0;
            const int kv = e / 64, nn = e % 64;                 // V[k][n] (n fastest)
            Vs[kv][nn] = (k0 + kv < J.n && n0 + nn < J.n) ? J.V[(size_t)(k0 + kv) * J.ldu + n0 + nn] : 0.0;
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

size_t eigen_workspace_bytes(const int32_t *dims, int count) { return plan(dims, count).bytes; }

kfac_status_t eigen_run(const float *const *F, const int32_t *dims, const int32_t *ldF, int count,
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
            eig_round<<<active, NT, 0, s>>>(table, count, r, tol, tol_abs);
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

}  // namespace kfac
