/* kfac_oracle.c -- FP64 CPU oracle for the K-FAC preconditioner hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see kfac_oracle.h).  Plain loops in double
 * precision, no blocking or fusion beyond what each definition states; the
 * only parallelism is OpenMP across independent layers in
 * orc_update_factors.  Every function cites the passage it follows.
 */
#include "kfac_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

int64_t orc_rows(const orc_layer_t *L) {
    return (int64_t)L->batch * L->h_out * L->w_out;
}

int32_t orc_d_a(const orc_layer_t *L) {
    return L->c_in * L->k_h * L->k_w + (L->bias_col ? 1 : 0);
}

/* One im2col row (R8, R9): patch of output position r, zero outside the image,
 * trailing 1 for the bias column. */
static void patch_row(const orc_layer_t *L, const float *act, int64_t r, double *x) {
    if (L->kind == 0) {                         /* linear: the input row itself */
        for (int c = 0; c < L->c_in; ++c) x[c] = act[r * L->c_in + c];
    } else {
        int64_t hw = (int64_t)L->h_out * L->w_out;
        int64_t n = r / hw;
        int oh = (int)((r % hw) / L->w_out);
        int ow = (int)(r % L->w_out);
        for (int kh = 0; kh < L->k_h; ++kh)
            for (int kw = 0; kw < L->k_w; ++kw) {
                int ih = oh * L->stride_h - L->pad_h + kh;
                int iw = ow * L->stride_w - L->pad_w + kw;
                double *dst = x + (int64_t)(kh * L->k_w + kw) * L->c_in;
                if (ih < 0 || ih >= L->h_in || iw < 0 || iw >= L->w_in) {
                    for (int c = 0; c < L->c_in; ++c) dst[c] = 0.0;
                } else {
                    const float *src = act + ((n * L->h_in + ih) * L->w_in + iw) * L->c_in;
                    for (int c = 0; c < L->c_in; ++c) dst[c] = src[c];
                }
            }
    }
    if (L->bias_col) x[L->c_in * L->k_h * L->k_w] = 1.0;
}

void orc_im2col(const orc_layer_t *L, const float *act, double *X) {
    int64_t n = orc_rows(L);
    int32_t d = orc_d_a(L);
    for (int64_t r = 0; r < n; ++r) patch_row(L, act, r, X + r * d);
}

/* Eq. 5: F = (1/n) sum_r x_r x_r^T, upper triangle summed row by row, mirrored. */
static void accumulate_outer(const double *x, int32_t d, double *S) {
    for (int32_t i = 0; i < d; ++i) {
        double xi = x[i];
        if (xi == 0.0) continue;
        double *Si = S + (int64_t)i * d;
        for (int32_t j = i; j < d; ++j) Si[j] += xi * x[j];
    }
}

static void finish_covariance(double *S, int32_t d, int64_t n) {
    for (int32_t i = 0; i < d; ++i)
        for (int32_t j = i; j < d; ++j) {
            double v = S[(int64_t)i * d + j] / (double)n;
            S[(int64_t)i * d + j] = v;
            S[(int64_t)j * d + i] = v;
        }
}

void orc_covariance(const double *X, int64_t n, int32_t d, double *F) {
    memset(F, 0, sizeof(double) * (size_t)d * d);
    for (int64_t r = 0; r < n; ++r) accumulate_outer(X + r * d, d, F);
    finish_covariance(F, d, n);
}

/* Eqs. 16-17: xi weights the new batch estimate, 1 - xi the previous value (R5);
 * the first observation seeds the average. */
void orc_running_average(double *F, const double *Fb, int32_t d, double xi, int32_t first) {
    int64_t m = (int64_t)d * d;
    for (int64_t i = 0; i < m; ++i)
        F[i] = first ? Fb[i] : xi * Fb[i] + (1.0 - xi) * F[i];
}

void orc_update_factors(const orc_layer_t *layers, int32_t nl, const float *const *act,
                        const float *const *gout, double *const *A, double *const *G,
                        double xi, int32_t first) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t l = 0; l < 2 * nl; ++l) {
        const orc_layer_t *L = &layers[l / 2];
        int64_t n = orc_rows(L);
        int32_t d = (l % 2 == 0) ? orc_d_a(L) : L->c_out;
        double *x = (double *)malloc(sizeof(double) * d);
        double *S = (double *)calloc((size_t)d * d, sizeof(double));
        for (int64_t r = 0; r < n; ++r) {
            if (l % 2 == 0) {
                patch_row(L, act[l / 2], r, x);                       /* a_{i-1} */
            } else {
                const float *g = gout[l / 2] + r * L->c_out;            /* g_i */
                for (int32_t c = 0; c < d; ++c) x[c] = g[c];
            }
            accumulate_outer(x, d, S);
        }
        finish_covariance(S, d, n);
        orc_running_average(l % 2 == 0 ? A[l / 2] : G[l / 2], S, d, xi, first);
        free(S);
        free(x);
    }
}

/* ---------------------------------------------------------------- eigen -- */

/* Sort eigenpairs ascending, clamp negatives to 0 (R10) and write Q with
 * columns = eigenvectors from Ut (rows = eigenvectors). */
static void finish_eig(int32_t d, const double *w, const double *Ut, double *Q, double *v) {
    int *idx = (int *)malloc(sizeof(int) * d);
    for (int i = 0; i < d; ++i) {                        /* stable insertion sort, ascending */
        int t = i;
        idx[i] = i;
        while (t > 0 && w[idx[t - 1]] > w[i]) { idx[t] = idx[t - 1]; --t; }
        idx[t] = i;
    }
    for (int j = 0; j < d; ++j) {
        double lam = w[idx[j]];
        v[j] = lam > 0.0 ? lam : 0.0;
        const double *u = Ut + (int64_t)idx[j] * d;
        for (int i = 0; i < d; ++i) Q[(int64_t)i * d + j] = u[i];
    }
    free(idx);
}

/* Householder reflector (Golub & Van Loan Alg. 5.1.1 restated): P = I - beta v v^T,
 * P x = r e_1 with r = -sign(x_0) ||x||. */
static double house(const double *x, int32_t m, double *v, double *r_out) {
    double alpha = 0.0;
    for (int32_t i = 0; i < m; ++i) alpha += x[i] * x[i];
    alpha = sqrt(alpha);
    for (int32_t i = 0; i < m; ++i) v[i] = x[i];
    if (alpha == 0.0) { *r_out = 0.0; return 0.0; }
    double r = x[0] >= 0.0 ? -alpha : alpha;
    v[0] = x[0] - r;
    double vv = 0.0;
    for (int32_t i = 0; i < m; ++i) vv += v[i] * v[i];
    *r_out = r;
    return 2.0 / vv;
}

int orc_symeig(const double *F, int32_t d, double *Q, double *v) {
    int64_t n = d;
    double *A = (double *)malloc(sizeof(double) * n * n);
    double *Ut = (double *)calloc((size_t)(n * n), sizeof(double));
    double *dg = (double *)malloc(sizeof(double) * n);
    double *e = (double *)calloc((size_t)n, sizeof(double));
    double *x = (double *)malloc(sizeof(double) * n);
    double *hv = (double *)malloc(sizeof(double) * n);
    double *p = (double *)malloc(sizeof(double) * n);
    double *u = (double *)malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) A[i * n + j] = 0.5 * (F[i * n + j] + F[j * n + i]);
    for (int64_t i = 0; i < n; ++i) Ut[i * n + i] = 1.0;

    /* Householder tridiagonalisation, G&VL Alg. 8.3.1: A <- P_k A P_k, and
     * Ut <- P_k Ut so that Ut = Q^T with A_orig = Q T Q^T. */
    for (int64_t k = 0; k + 2 < n; ++k) {
        int64_t m = n - k - 1;
        for (int64_t i = 0; i < m; ++i) x[i] = A[(k + 1 + i) * n + k];
        double r, beta = house(x, (int32_t)m, hv, &r);
        if (beta != 0.0) {
            double pv = 0.0;
            for (int64_t i = 0; i < m; ++i) {
                double s = 0.0;
                const double *Bi = A + (k + 1 + i) * n + (k + 1);
                for (int64_t j = 0; j < m; ++j) s += Bi[j] * hv[j];
                p[i] = beta * s;
                pv += p[i] * hv[i];
            }
            double K = 0.5 * beta * pv;
            for (int64_t i = 0; i < m; ++i) p[i] -= K * hv[i];            /* w */
            for (int64_t i = 0; i < m; ++i) {
                double *Bi = A + (k + 1 + i) * n + (k + 1);
                for (int64_t j = 0; j < m; ++j) Bi[j] -= hv[i] * p[j] + p[i] * hv[j];
            }
            for (int64_t c = 0; c < n; ++c) u[c] = 0.0;
            for (int64_t a = 0; a < m; ++a) {
                const double *row = Ut + (k + 1 + a) * n;
                for (int64_t c = 0; c < n; ++c) u[c] += hv[a] * row[c];
            }
            for (int64_t a = 0; a < m; ++a) {
                double *row = Ut + (k + 1 + a) * n;
                double f = beta * hv[a];
                for (int64_t c = 0; c < n; ++c) row[c] -= f * u[c];
            }
        } else {
            r = x[0];
        }
        A[(k + 1) * n + k] = A[k * n + k + 1] = r;
        for (int64_t i = 1; i < m; ++i) A[(k + 1 + i) * n + k] = A[k * n + k + 1 + i] = 0.0;
    }
    for (int64_t i = 0; i < n; ++i) dg[i] = A[i * n + i];
    for (int64_t i = 0; i + 1 < n; ++i) e[i] = A[(i + 1) * n + i];

    /* Implicit symmetric QR with Wilkinson shift, G&VL Alg. 8.3.2 / 8.3.3.
     * Rotations G(k,k+1) act on T as G^T T G and on Ut as G^T Ut. */
    int steps = 0, ok = 1;
    long max_steps = 60L * (n + 1);
    for (;;) {
        for (int64_t i = 0; i + 1 < n; ++i)
            if (fabs(e[i]) <= DBL_EPSILON * (fabs(dg[i]) + fabs(dg[i + 1])) || fabs(e[i]) < DBL_MIN)
                e[i] = 0.0;
        int64_t hi = n - 1;
        while (hi > 0 && e[hi - 1] == 0.0) --hi;
        if (hi == 0) break;
        int64_t lo = hi - 1;
        while (lo > 0 && e[lo - 1] != 0.0) --lo;
        if (++steps > max_steps) { ok = 0; break; }
        double dd = 0.5 * (dg[hi - 1] - dg[hi]);
        double ee = e[hi - 1];
        double mu = dg[hi] - ee * ee / (dd + (dd >= 0.0 ? 1.0 : -1.0) * hypot(dd, ee));
        double xx = dg[lo] - mu, zz = e[lo], bulge = 0.0;
        for (int64_t k = lo; k < hi; ++k) {
            double c = 1.0, s = 0.0;
            if (zz != 0.0) { double rr = hypot(xx, zz); c = xx / rr; s = -zz / rr; }
            if (k > lo) e[k - 1] = c * e[k - 1] - s * bulge;      /* T'(k,k-1); T'(k+1,k-1) = 0 */
            double a = dg[k], b = e[k], cc = dg[k + 1];
            dg[k] = a * c * c - 2.0 * b * c * s + cc * s * s;
            dg[k + 1] = a * s * s + 2.0 * b * c * s + cc * c * c;
            e[k] = (a - cc) * c * s + b * (c * c - s * s);
            if (k + 1 < hi) { bulge = -s * e[k + 1]; e[k + 1] = c * e[k + 1]; }
            double *r0 = Ut + k * n, *r1 = Ut + (k + 1) * n;
            for (int64_t j = 0; j < n; ++j) {
                double y0 = r0[j], y1 = r1[j];
                r0[j] = c * y0 - s * y1;
                r1[j] = s * y0 + c * y1;
            }
            xx = e[k];
            zz = bulge;
        }
    }
    finish_eig(d, dg, Ut, Q, v);
    free(A); free(Ut); free(dg); free(e); free(x); free(hv); free(p); free(u);
    return ok ? steps : -1;
}

/* Cyclic-by-row Jacobi, G&VL Alg. 8.5.2 (sym.schur2) + 8.5.3; stop when
 * off(A) <= 1e-15 ||A||_F (S:81 uses 1e-12 with 100 sweeps). */
int orc_symeig_jacobi(const double *F, int32_t d, double *Q, double *v) {
    int64_t n = d;
    double *A = (double *)malloc(sizeof(double) * n * n);
    double *Vt = (double *)calloc((size_t)(n * n), sizeof(double));
    double *w = (double *)calloc((size_t)n, sizeof(double));
    double fro = 0.0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) {
            A[i * n + j] = 0.5 * (F[i * n + j] + F[j * n + i]);
            fro += A[i * n + j] * A[i * n + j];
        }
    fro = sqrt(fro);
    for (int64_t i = 0; i < n; ++i) Vt[i * n + i] = 1.0;
    int sweep, ok = 0;
    for (sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < n; ++j)
                if (i != j) off += A[i * n + j] * A[i * n + j];
        if (sqrt(off) <= 1e-15 * fro || fro == 0.0) { ok = 1; break; }
        for (int64_t p = 0; p < n; ++p)
            for (int64_t q = p + 1; q < n; ++q) {
                double apq = A[p * n + q];
                if (apq == 0.0) continue;
                double tau = (A[q * n + q] - A[p * n + p]) / (2.0 * apq);
                double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                for (int64_t k = 0; k < n; ++k) {               /* A <- A J */
                    double akp = A[k * n + p], akq = A[k * n + q];
                    A[k * n + p] = c * akp - s * akq;
                    A[k * n + q] = s * akp + c * akq;
                }
                for (int64_t k = 0; k < n; ++k) {               /* A <- J^T A */
                    double apk = A[p * n + k], aqk = A[q * n + k];
                    A[p * n + k] = c * apk - s * aqk;
                    A[q * n + k] = s * apk + c * aqk;
                }
                for (int64_t k = 0; k < n; ++k) {               /* V <- V J (rows of V^T) */
                    double x0 = Vt[p * n + k], x1 = Vt[q * n + k];
                    Vt[p * n + k] = c * x0 - s * x1;
                    Vt[q * n + k] = s * x0 + c * x1;
                }
            }
    }
    for (int64_t i = 0; i < n; ++i) w[i] = A[i * n + i];
    finish_eig(d, w, Vt, Q, v);
    free(A); free(Vt); free(w);
    return ok ? sweep : -1;
}

/* ------------------------------------------------------------- inverse -- */

/* Eq. 11: (F + gamma I)^{-1} = L^{-T} L^{-1} with F + gamma I = L L^T. */
int orc_damped_inverse(const double *F, int32_t d, double gamma, double *Finv) {
    int64_t n = d;
    double *L = (double *)calloc((size_t)(n * n), sizeof(double));
    double *Li = (double *)calloc((size_t)(n * n), sizeof(double));
    int info = 0;
    for (int64_t j = 0; j < n && !info; ++j) {
        double s = 0.5 * (F[j * n + j] + F[j * n + j]) + gamma;
        for (int64_t k = 0; k < j; ++k) s -= L[j * n + k] * L[j * n + k];
        if (!(s > 0.0)) { info = (int)j + 1; break; }
        double ljj = sqrt(s);
        L[j * n + j] = ljj;
        for (int64_t i = j + 1; i < n; ++i) {
            double t = 0.5 * (F[i * n + j] + F[j * n + i]);
            for (int64_t k = 0; k < j; ++k) t -= L[i * n + k] * L[j * n + k];
            L[i * n + j] = t / ljj;
        }
    }
    if (!info) {
        for (int64_t c = 0; c < n; ++c) {                  /* forward substitution L y = e_c */
            for (int64_t i = c; i < n; ++i) {
                double t = (i == c) ? 1.0 : 0.0;
                for (int64_t k = c; k < i; ++k) t -= L[i * n + k] * Li[k * n + c];
                Li[i * n + c] = t / L[i * n + i];
            }
        }
        for (int64_t i = 0; i < n; ++i)                     /* Finv = Li^T Li */
            for (int64_t j = 0; j < n; ++j) {
                double t = 0.0;
                for (int64_t k = (i > j ? i : j); k < n; ++k) t += Li[k * n + i] * Li[k * n + j];
                Finv[i * n + j] = t;
            }
    }
    free(L); free(Li);
    return info;
}

/* ------------------------------------------------------ preconditioning -- */

void orc_precondition(int32_t mode, int32_t dg, int32_t da, const double *W,
                      const double *QG, const double *vG, const double *QA, const double *vA,
                      double gamma, double *P) {
    int64_t m = dg, k = da;
    double *T = (double *)calloc((size_t)(m * k), sizeof(double));
    double *V = (double *)calloc((size_t)(m * k), sizeof(double));
    if (mode == 2) {
        /* Eq. 12: P = (G + gI)^-1 W (A + gI)^-1; inverses given in QG/QA. */
        for (int64_t i = 0; i < m; ++i)
            for (int64_t t = 0; t < m; ++t) {
                double g = QG[i * m + t];
                for (int64_t j = 0; j < k; ++j) T[i * k + j] += g * W[t * k + j];
            }
        for (int64_t i = 0; i < m; ++i)
            for (int64_t t = 0; t < k; ++t) {
                double a = T[i * k + t];
                for (int64_t j = 0; j < k; ++j) V[i * k + j] += a * QA[t * k + j];
            }
        memcpy(P, V, sizeof(double) * (size_t)(m * k));
    } else {
        /* Eq. 13: V1 = Q_G^T W Q_A (R1: the gradient, R2: A = Q_A L_A Q_A^T). */
        for (int64_t t = 0; t < m; ++t)
            for (int64_t i = 0; i < m; ++i) {
                double g = QG[t * m + i];
                for (int64_t j = 0; j < k; ++j) T[i * k + j] += g * W[t * k + j];
            }
        for (int64_t i = 0; i < m; ++i)
            for (int64_t t = 0; t < k; ++t) {
                double a = T[i * k + t];
                for (int64_t j = 0; j < k; ++j) V[i * k + j] += a * QA[t * k + j];
            }
        /* Eq. 14: V2 = V1 / (v_G v_A^T + gamma) elementwise (R3, R4);
         * FACTORED: (v_G + gamma)(v_A + gamma)^T.  Denominator floor 1e-12. */
        for (int64_t i = 0; i < m; ++i)
            for (int64_t j = 0; j < k; ++j) {
                double den = mode == 0 ? vG[i] * vA[j] + gamma : (vG[i] + gamma) * (vA[j] + gamma);
                if (den < 1e-12) den = 1e-12;
                V[i * k + j] /= den;
            }
        /* Eq. 15: P = Q_G V2 Q_A^T. */
        memset(T, 0, sizeof(double) * (size_t)(m * k));
        for (int64_t i = 0; i < m; ++i)
            for (int64_t t = 0; t < m; ++t) {
                double g = QG[i * m + t];
                for (int64_t j = 0; j < k; ++j) T[i * k + j] += g * V[t * k + j];
            }
        for (int64_t i = 0; i < m; ++i)
            for (int64_t j = 0; j < k; ++j) {
                double s = 0.0;
                for (int64_t t = 0; t < k; ++t) s += T[i * k + t] * QA[j * k + t];
                P[i * k + j] = s;
            }
    }
    free(T); free(V);
}

/* ------------------------------------------------------------- KL-clip -- */

double orc_kl_clip(int32_t nl, double *const *P, const double *const *W, const int64_t *numel,
                   double lr, double kappa, double *s_out) {
    double s = 0.0;
    for (int32_t l = 0; l < nl; ++l) {
        double dot = 0.0;                                   /* G_l^T grad L_l (Frobenius) */
        for (int64_t i = 0; i < numel[l]; ++i) dot += P[l][i] * W[l][i];
        s += fabs(dot);
    }
    double nu = 1.0;
    if (s > 0.0) {
        double r = sqrt(kappa / (lr * lr * s));
        nu = r < 1.0 ? r : 1.0;
    }
    for (int32_t l = 0; l < nl; ++l)
        for (int64_t i = 0; i < numel[l]; ++i) P[l][i] *= nu;
    if (s_out) *s_out = s;
    return nu;
}

/* ---------------------------------------------------------------- kron -- */

void orc_kron(const double *A, int32_t m, int32_t n, const double *B, int32_t p, int32_t q,
              double *out) {
    int64_t cols = (int64_t)n * q;
    for (int32_t i = 0; i < m; ++i)
        for (int32_t j = 0; j < n; ++j)
            for (int32_t k = 0; k < p; ++k)
                for (int32_t l = 0; l < q; ++l)
                    out[((int64_t)i * p + k) * cols + (int64_t)j * q + l] = A[i * n + j] * B[k * q + l];
}

int orc_kron_solve(const double *A, int32_t da, const double *G, int32_t dg, double gamma,
                   const double *W, double *P) {
    int64_t N = (int64_t)da * dg;
    double *M = (double *)malloc(sizeof(double) * N * N);
    double *b = (double *)malloc(sizeof(double) * N);
    orc_kron(A, da, da, G, dg, dg, M);                      /* F_hat = A (x) G (Eq. 5) */
    for (int64_t i = 0; i < N; ++i) M[i * N + i] += gamma;
    for (int32_t j = 0; j < da; ++j)                        /* vec_c: column stacking (R13) */
        for (int32_t i = 0; i < dg; ++i) b[(int64_t)j * dg + i] = W[(int64_t)i * da + j];
    int info = 0;
    for (int64_t j = 0; j < N && !info; ++j) {              /* in-place Cholesky, lower */
        double s = M[j * N + j];
        for (int64_t k = 0; k < j; ++k) s -= M[j * N + k] * M[j * N + k];
        if (!(s > 0.0)) { info = (int)j + 1; break; }
        s = sqrt(s);
        M[j * N + j] = s;
        for (int64_t i = j + 1; i < N; ++i) {
            double t = M[i * N + j];
            for (int64_t k = 0; k < j; ++k) t -= M[i * N + k] * M[j * N + k];
            M[i * N + j] = t / s;
        }
    }
    if (!info) {
        for (int64_t i = 0; i < N; ++i) {                   /* L y = b */
            double t = b[i];
            for (int64_t k = 0; k < i; ++k) t -= M[i * N + k] * b[k];
            b[i] = t / M[i * N + i];
        }
        for (int64_t i = N - 1; i >= 0; --i) {              /* L^T x = y */
            double t = b[i];
            for (int64_t k = i + 1; k < N; ++k) t -= M[k * N + i] * b[k];
            b[i] = t / M[i * N + i];
        }
        for (int32_t j = 0; j < da; ++j)
            for (int32_t i = 0; i < dg; ++i) P[(int64_t)i * da + j] = b[(int64_t)j * dg + i];
    }
    free(M); free(b);
    return info;
}

/* ---------------------------------------------------------- assignment -- */

typedef struct { double cost; int32_t idx; } job_t;

static int cmp_job(const void *a, const void *b) {
    const job_t *x = (const job_t *)a, *y = (const job_t *)b;
    if (x->cost > y->cost) return -1;
    if (x->cost < y->cost) return 1;
    return x->idx - y->idx;
}

static void lpt(job_t *jobs, int32_t nj, int32_t world, int32_t *owner_of_job) {
    double *load = (double *)calloc((size_t)world, sizeof(double));
    qsort(jobs, nj, sizeof(job_t), cmp_job);
    for (int32_t t = 0; t < nj; ++t) {
        int32_t best = 0;
        for (int32_t r = 1; r < world; ++r)
            if (load[r] < load[best]) best = r;
        load[best] += jobs[t].cost;
        owner_of_job[jobs[t].idx] = best;
    }
    free(load);
}

void orc_assign(const int32_t *dims, const int32_t *layer_of, int32_t nf, int32_t nl,
                int32_t world, int32_t policy, int32_t *owner) {
    if (policy == 1) {                                      /* paper round robin (R16) */
        for (int32_t f = 0; f < nf; ++f)
            owner[f] = world > nl ? f % world : layer_of[f] % world;
    } else if (policy == 0) {                               /* LPT on d^3 */
        job_t *jobs = (job_t *)malloc(sizeof(job_t) * nf);
        for (int32_t f = 0; f < nf; ++f) {
            double d = dims[f];
            jobs[f].cost = d * d * d;
            jobs[f].idx = f;
        }
        lpt(jobs, nf, world, owner);
        free(jobs);
    } else {                                                /* layer-wise LPT */
        job_t *jobs = (job_t *)malloc(sizeof(job_t) * nl);
        int32_t *lown = (int32_t *)malloc(sizeof(int32_t) * nl);
        for (int32_t l = 0; l < nl; ++l) { jobs[l].cost = 0.0; jobs[l].idx = l; }
        for (int32_t f = 0; f < nf; ++f) {
            double d = dims[f];
            jobs[layer_of[f]].cost += d * d * d;
        }
        lpt(jobs, nl, world, lown);
        for (int32_t f = 0; f < nf; ++f) owner[f] = lown[layer_of[f]];
        free(jobs); free(lown);
    }
}

/* --------------------------------------------- batches (independent units) -- */

/* Alg. 1 step 2: every factor independently; OpenMP across factors. */
void orc_symeig_batch(int32_t count, const double *const *F, const int32_t *dims,
                      double *const *Q, double *const *v, int32_t *status) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t i = 0; i < count; ++i) status[i] = orc_symeig(F[i], dims[i], Q[i], v[i]);
}

/* Alg. 1 step 3: every layer independently; OpenMP across layers. */
void orc_precondition_batch(int32_t nl, int32_t mode, const int32_t *dg, const int32_t *da,
                            const double *const *W, const double *const *QG,
                            const double *const *vG, const double *const *QA,
                            const double *const *vA, double gamma, double *const *P) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t l = 0; l < nl; ++l)
        orc_precondition(mode, dg[l], da[l], W[l], QG[l], vG ? vG[l] : 0, QA[l], vA ? vA[l] : 0,
                         gamma, P[l]);
}
