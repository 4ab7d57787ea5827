/* kfac_oracle.h -- plain, slow, FP64 CPU oracle of the distributed K-FAC
 * preconditioner hot path (arXiv 2007.00784).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2007_00784_b200/, include/).
 *
 * Every routine is the plain definition written out in double precision,
 * with loops in the paper's order; parallelism (OpenMP) is only across
 * independent layers / factors.  Citations: P:n = PAPER.md line n,
 * S:n = SPEC.md line n, readings Rn = DESIGN.md "Readings of the paper".
 */
#ifndef KFAC_ORACLE_H
#define KFAC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One Linear / Conv2D layer.  Same field meaning as the product's
 * kfac_layer_t, but an independent definition. */
typedef struct {
    int32_t kind;           /* 0 linear, 1 conv2d */
    int32_t batch;          /* N images (conv) or rows (linear) */
    int32_t c_in, h_in, w_in;
    int32_t c_out, h_out, w_out;
    int32_t k_h, k_w, stride_h, stride_w, pad_h, pad_w;
    int32_t bias_col;       /* 1: append a column of ones (R7) */
} orc_layer_t;

int64_t orc_rows(const orc_layer_t *L);      /* n = N*H_out*W_out */
int32_t orc_d_a(const orc_layer_t *L);       /* C_in*k_h*k_w + bias_col */

/* im2col (R8): X[r][c], r = (n*H_out + oh)*W_out + ow, c = (kh*K_w + kw)*C_in + ci,
 * value act[n, oh*s_h - p_h + kh, ow*s_w - p_w + kw, ci] or 0 outside; last col 1. */
void orc_im2col(const orc_layer_t *L, const float *act, double *X);

/* F_batch = X^T X / n over the n rows of X (n x d) -- Eq. 5 A = a a^T, G = g g^T. */
void orc_covariance(const double *X, int64_t n, int32_t d, double *F);

/* Running average, Eqs. 16-17 read as R5:
 * F = first ? F_batch : xi*F_batch + (1-xi)*F  (xi: weight on the new batch estimate). */
void orc_running_average(double *F, const double *Fbatch, int32_t d, double xi, int32_t first);

/* Stage 1 for a set of layers (act NHWC fp32, gout rows x C_out fp32).
 * A[l] (d_A x d_A), G[l] (d_G x d_G) row-major doubles updated in place. */
void orc_update_factors(const orc_layer_t *layers, int32_t nl, const float *const *act,
                        const float *const *gout, double *const *A, double *const *G,
                        double xi, int32_t first);

/* Symmetric eigendecomposition of (F+F^T)/2 (Alg. 1):
 * Householder tridiagonalisation (Golub & Van Loan Alg. 8.3.1) then implicit
 * symmetric QR with Wilkinson shift (G&VL Alg. 8.3.2/8.3.3).  Q row-major d x d,
 * columns are eigenvectors; v ascending, clamped at 0 (R10).  Returns the
 * number of QR steps, or -1 if not converged. */
int orc_symeig(const double *F, int32_t d, double *Q, double *v);
/* Cyclic Jacobi (G&VL Alg. 8.5.3) -- cross-check for small d.  Same output contract. */
int orc_symeig_jacobi(const double *F, int32_t d, double *Q, double *v);

/* (F + gamma I)^{-1} by Cholesky (Eq. 11; R15).  Returns 0 or k+1 at a
 * non-positive pivot k. */
int orc_damped_inverse(const double *F, int32_t d, double gamma, double *Finv);

/* Preconditioning of one layer; W is d_G x d_A (row-major).
 * mode 0 EIGEN     : Eqs. 13-15, denominator v_G v_A^T + gamma (R3, R4)
 * mode 1 FACTORED  : same with denominator (v_G + gamma)(v_A + gamma)^T
 * mode 2 INVERSE   : Eq. 12: Ginv W Ainv; Ginv/Ainv passed as QG/QA, v ignored. */
void orc_precondition(int32_t mode, int32_t dg, int32_t da, const double *W,
                      const double *QG, const double *vG, const double *QA, const double *vA,
                      double gamma, double *P);

/* KL-clip (Eq. 18; R12): s = sum_l |<P_l, W_l>_F|,
 * nu = s > 0 ? min(1, sqrt(kappa / (lr^2 s))) : 1; P_l *= nu.  Returns nu. */
double orc_kl_clip(int32_t nl, double *const *P, const double *const *W, const int64_t *numel,
                   double lr, double kappa, double *s_out);

/* Kronecker product (Eq. 6): A (m x n) (x) B (p x q) -> (m p) x (n q). */
void orc_kron(const double *A, int32_t m, int32_t n, const double *B, int32_t p, int32_t q,
              double *out);

/* Brute-force damped Kronecker solve (R13): P = unvec_c((A (x) G + gamma I)^{-1} vec_c(W))
 * with column-stacking vec, W d_G x d_A.  Dense Cholesky of the (dA*dG)^2 system. */
int orc_kron_solve(const double *A, int32_t da, const double *G, int32_t dg, double gamma,
                   const double *W, double *P);

/* Factor -> rank assignment (Alg. 1).
 * policy 0 LPT_D3          : factors sorted by (d^3 desc, index asc), each to the
 *                            least-loaded rank (ties: lowest rank) -- north_star's
 *                            greedy size-balanced distribution.
 * policy 1 ROUND_ROBIN_PAPER: if W > L: factor k of [A0,G0,A1,G1,...] -> k mod W;
 *                            else layer i -> i mod W (R16, reproduces P:746-747).
 * policy 2 LAYERWISE_LPT   : whole layers (cost d_A^3 + d_G^3) by LPT (K-FAC-lw). */
void orc_assign(const int32_t *dims, const int32_t *layer_of, int32_t nf, int32_t nl,
                int32_t world, int32_t policy, int32_t *owner);

/* Batched drivers (OpenMP across independent factors / layers only). */
void orc_symeig_batch(int32_t count, const double *const *F, const int32_t *dims,
                      double *const *Q, double *const *v, int32_t *status);
void orc_precondition_batch(int32_t nl, int32_t mode, const int32_t *dg, const int32_t *da,
                            const double *const *W, const double *const *QG,
                            const double *const *vG, const double *const *QA,
                            const double *const *vA, double gamma, double *const *P);

#ifdef __cplusplus
}
#endif
#endif
