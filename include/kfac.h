/* kfac.h -- C-ABI of the B200-native K-FAC preconditioner hot path.
 *
 * Method: distributed K-FAC as a gradient preconditioner (Pauloski et al.,
 * arXiv 2007.00784).  Citations "P:n" are PAPER.md lines, "S:n" SPEC.md
 * lines, "Rn" the readings listed in DESIGN.md.  Algorithm 1:
 *   step 1  factors A, G and their running average    -> kfac_update_factors
 *   step 2  eigendecomposition of every factor         -> kfac_compute_eigen
 *           (explicit damped inverse, comparison)      -> kfac_compute_inverse
 *           factor -> worker assignment                 -> kfac_assign
 *   step 3  preconditioned gradient, Eqs. 13-15 / 12   -> kfac_precondition
 *   Eq. 18  KL-clip rescaling by nu                     -> kfac_kl_clip
 *
 * Conventions (all calls):
 *  - Every buffer is caller-owned.  "device" pointers are CUDA device
 *    (global) memory; "host" pointers are ordinary host memory.  Arrays of
 *    pointers (e.g. `const float* const* act`) are HOST arrays holding DEVICE
 *    pointers.  The library allocates no device memory, keeps no pointer after
 *    return, never synchronises the device and launches on `stream`
 *    (cudaStream_t; 0 = legacy default stream) -- independent launches of one call
 *    may run on per-thread side streams forked from `stream` by an event and joined
 *    back into it before the call returns, so the call stays stream-ordered (and
 *    capturable in a CUDA graph) as seen by the caller.
 *  - Matrices are fp32, row-major, with a leading dimension `ld` (elements)
 *    that is >= the column count and a multiple of 4 (16-byte rows, TMA rule);
 *    every matrix base address must be 16-byte aligned.
 *  - Errors: arguments are validated on the host before anything is launched.
 *    A validation status (INVALID_VALUE, SHAPE, ALIGNMENT, WORKSPACE, UNSUPPORTED)
 *    means nothing was launched and outputs are untouched.  KFAC_ERR_CUDA (a CUDA
 *    runtime call or kernel launch failed) can occur after earlier kernels of the
 *    same call were queued, so outputs may be partly written.
 *    kfac_last_error() returns a thread-local message for the last failure.
 *    Numerical failures are device-side `info` codes, not statuses.
 *  - Concurrency: host state is thread-local (staging) or mutex-guarded (per-device
 *    kernel attributes), so calls from several host threads, on several devices, or
 *    on different streams with disjoint buffers and workspaces may overlap.
 *  - Determinism: identical inputs on the same GPU model give bitwise
 *    identical outputs (fixed reduction orders; no float atomics).
 *  - Workspace: each stage has a *_workspace_size twin taking the same shape
 *    arguments; `ws` is device memory of at least that many bytes, 256-byte
 *    aligned, not shared with a concurrently running call.
 */
#ifndef KFAC_H
#define KFAC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *kfac_stream_t;   /* == cudaStream_t */

typedef enum {
    KFAC_OK = 0,
    KFAC_ERR_INVALID_VALUE = 1,   /* null pointer, count <= 0, bad enum, bad hyper-parameter */
    KFAC_ERR_SHAPE = 2,           /* inconsistent layer geometry, ld < cols, size limits */
    KFAC_ERR_ALIGNMENT = 3,       /* ld % 4 != 0 or base address not 16-byte aligned */
    KFAC_ERR_WORKSPACE = 4,       /* ws null / too small / misaligned */
    KFAC_ERR_UNSUPPORTED = 5,     /* feature not available on this device / build */
    KFAC_ERR_CUDA = 6             /* a CUDA runtime call failed (see kfac_last_error) */
} kfac_status_t;

/* Only Linear and Conv2D layers are preconditioned. */
typedef enum { KFAC_LINEAR = 0, KFAC_CONV2D = 1 } kfac_layer_kind_t;

/* One preconditioned layer.  For KFAC_LINEAR: batch = rows n, c_in/c_out =
 * in/out features, h/w/k/stride = 1, pad = 0.  For KFAC_CONV2D: activations
 * are NHWC (batch, h_in, w_in, c_in); h_out = (h_in + 2 pad_h - k_h)/stride_h + 1.
 * d_A = c_in*k_h*k_w + bias_col (R7), d_G = c_out, rows n = batch*h_out*w_out (R6).
 * Patch columns are ordered (k_h, k_w, c_in), bias last (R8); the gradient
 * grad L_i must use the same column order. */
typedef struct {
    int32_t kind;
    int32_t batch;
    int32_t c_in, h_in, w_in;
    int32_t c_out, h_out, w_out;
    int32_t k_h, k_w, stride_h, stride_w, pad_h, pad_w;
    int32_t bias_col;             /* 0 or 1 */
} kfac_layer_t;

typedef enum {
    KFAC_PRECOND_EIGEN = 0,           /* Eqs. 13-15, denominator v_G v_A^T + damping (R3, R4) */
    KFAC_PRECOND_EIGEN_FACTORED = 1,  /* denominator (v_G + damping)(v_A + damping)^T  (R14) */
    KFAC_PRECOND_INVERSE = 2          /* Eq. 12: G_inv grad A_inv; inverses in the Q slots */
} kfac_precond_mode_t;

typedef enum {
    KFAC_ASSIGN_LPT_D3 = 0,             /* greedy size-balanced (north_star) */
    KFAC_ASSIGN_ROUND_ROBIN_PAPER = 1,  /* the paper's round robin (R16) */
    KFAC_ASSIGN_LAYERWISE_LPT = 2       /* K-FAC-lw: whole layers */
} kfac_assign_policy_t;

/* kfac_compute_eigen flags */
#define KFAC_EIG_WARM_START 1u   /* Jacobi factors start from the Q passed in (stale basis) */
#define KFAC_EIG_JACOBI 2u       /* every factor by one-sided block Jacobi */
#define KFAC_EIG_TRIDIAG 4u      /* every factor by tridiagonalisation + divide and conquer */
#define KFAC_EIG_TWO_STAGE 8u    /* tridiagonal factors with 1024 <= dims <= 5632: two-stage reduction */
#define KFAC_EIG_ONE_STAGE 16u   /* tridiagonal factors: one-stage reduction only */

/* Derived dimensions of one layer.  Host only; any output pointer may be NULL. */
kfac_status_t kfac_layer_dims(const kfac_layer_t *layer, int32_t *d_a, int32_t *d_g, int64_t *rows);

/* ---- Stage 1: Kronecker factors (Eq. 5) and running average
 * (Eqs. 16-17; R5).  For every layer l (host arrays of length num_layers):
 *   A_batch = X^T X / n with X = [im2col(act[l]) | 1]   (n x d_A),
 *   G_batch = gout[l]^T gout[l] / n                     (gout: n x c_out, row-major, device),
 *   F = first ? F_batch : xi*F_batch + (1-xi)*F;  F *= out_scale   (F in {A, G}; Eqs. 16-17 P:383-386:
 *   xi weights the new batch estimate, xi = 1 keeps only the batch).
 * act[l]: device, NHWC (conv) or (n, c_in) (linear) fp32, contiguous.
 * A[l]: device d_A x ld_A[l]; G[l]: device d_G x ld_G[l]; both triangles are written
 * (symmetric).  When first == 0 the previous A/G are read (must be symmetric).
 * packed_A / packed_G (nullable host arrays of device pointers): also write each factor's upper
 * triangle row-major, d(d+1)/2 floats (row i starts at i d - i (i-1)/2), the same values as F --
 * the factor allreduce buffer at half the full-matrix bytes (kfac_unpack_factors restores
 * both triangles after the collective).
 * out_scale = 1/W before an allreduce-SUM averages the factors.
 * Rows per layer must be < 2^31; xi in [0, 1].
 * Workspace: the per-(tile, row chunk) partial sums and, for the tensor-core factors, the TF32
 * hi/lo planes of their inputs (two copies of each activation / gradient tensor). */
size_t kfac_update_factors_workspace_size(const kfac_layer_t *layers, int32_t num_layers);
kfac_status_t kfac_update_factors(const kfac_layer_t *layers, int32_t num_layers,
                                  const float *const *act, const float *const *gout,
                                  float *const *A, const int32_t *ld_A,
                                  float *const *G, const int32_t *ld_G,
                                  float *const *packed_A, float *const *packed_G,
                                  float xi, int32_t first, float out_scale,
                                  void *ws, size_t ws_bytes, kfac_stream_t stream);

/* Packed upper triangles (layout of kfac_update_factors' packed outputs) -> both triangles of F[i]
 * (device dims[i] x ld_F[i]), each element multiplied by `scale` (1: a bitwise copy; 1/W after a
 * reduce-SUM of W ranks' local running averages, whose mean is the running average of the
 * averaged batches because Eqs. 16-17 are linear).  No workspace. */
kfac_status_t kfac_unpack_factors(const float *const *packed, const int32_t *dims, float *const *F,
                                  const int32_t *ld_F, int32_t count, float scale, kfac_stream_t stream);

/* ---- Stage 2: symmetric eigendecomposition of each factor (Alg. 1).
 * F[i]: device dims[i] x ld_F[i] (read only; (F + F^T)/2 is decomposed).
 * Q[i]: device dims[i] x ld_Q[i]; on return column j is the eigenvector of evals[i][j].
 * evals[i]: device, dims[i] floats, ascending, clamped >= 0 (R10).
 * info: device int32[count]; 0 = converged, k > 0 = not converged after k sweeps
 * (outputs still written).  Method: factors with dims >= 64 by
 * Householder tridiagonalisation + divide and conquer + blocked back-transformation, smaller
 * ones by one-sided block Jacobi; KFAC_EIG_JACOBI / KFAC_EIG_TRIDIAG force one method.  The
 * tridiagonalisation is one-stage (Householder panels) or two-stage (dense -> band 16 -> tridiagonal,
 * DESIGN.md §8) for 1024 <= dims <= 5632; by default the two-stage reduction takes a factor that
 * carries most of the call's d^3 (a latency-bound lone factor, e.g. one rank's share at W >= 4) and
 * is measured faster at its size; KFAC_EIG_TWO_STAGE / KFAC_EIG_ONE_STAGE force either reduction.
 * When every dims >= 64 factor of the call fits one thread-block cluster's shared memory in fp64
 * (dims <= ~870), the one-stage reduction runs cluster-resident (DESIGN.md §8b'); same outputs.
 * KFAC_EIG_WARM_START: Q[i] holds the previous orthonormal eigenbasis on entry and the Jacobi
 * factors start from it (the dims >= 64 path stays cold: DESIGN.md §8c).  Eigenvector sign/order within equal eigenvalues is free (R11).
 * 1 <= dims[i] <= 16384. */
size_t kfac_compute_eigen_workspace_size(const int32_t *dims, int32_t count);
kfac_status_t kfac_compute_eigen(const float *const *F, const int32_t *dims, const int32_t *ld_F,
                                 int32_t count, float *const *Q, const int32_t *ld_Q,
                                 float *const *evals, int32_t *info, uint32_t flags,
                                 void *ws, size_t ws_bytes, kfac_stream_t stream);

/* ---- Stage 2' (comparison variant): explicit damped inverse (F + damping I)^{-1}
 * (Eq. 11; R15) by FP64 Cholesky.  Finv[i]: device dims[i] x ld_Finv[i].
 * info: device int32[count]; 0 ok, k > 0: leading minor k not positive. */
size_t kfac_compute_inverse_workspace_size(const int32_t *dims, int32_t count);
kfac_status_t kfac_compute_inverse(const float *const *F, const int32_t *dims, const int32_t *ld_F,
                                   int32_t count, float damping, float *const *Finv,
                                   const int32_t *ld_Finv, int32_t *info,
                                   void *ws, size_t ws_bytes, kfac_stream_t stream);

/* ---- Stage 3: preconditioned gradient (Eqs. 13-15, or Eq. 12).
 * grad[l], out[l]: device d_g[l] x ld_W[l] (gradient of the d_G x d_A weight, R8).
 * EIGEN / EIGEN_FACTORED: Q_G[l] (d_G x ld_QG[l], columns = eigenvectors), v_G[l] (d_G),
 *   Q_A[l] (d_A x ld_QA[l]), v_A[l] (d_A):
 *   out = Q_G ((Q_G^T grad Q_A) / D) Q_A^T,  D = v_G v_A^T + damping  (or factored).
 * INVERSE: Q_G = (G + damping I)^{-1}, Q_A = (A + damping I)^{-1}, v_* ignored (may be NULL):
 *   out = Q_G grad Q_A.
 * out may alias grad.  damping >= 0 (denominators are floored at 1e-12).
 * Workspace: the intermediates T, V2, U and, for layers whose dimensions are all >= 64, the TF32
 * hi/lo planes of Q_G, Q_A and grad (pre-split once per call for the tensor-core engine). */
size_t kfac_precondition_workspace_size(const int32_t *d_g, const int32_t *d_a, int32_t num_layers,
                                        int32_t mode);
kfac_status_t kfac_precondition(const int32_t *d_g, const int32_t *d_a, int32_t num_layers,
                                const float *const *grad, const int32_t *ld_W,
                                const float *const *Q_G, const int32_t *ld_QG, const float *const *v_G,
                                const float *const *Q_A, const int32_t *ld_QA, const float *const *v_A,
                                float damping, int32_t mode, float *const *out,
                                void *ws, size_t ws_bytes, kfac_stream_t stream);

/* ---- Eq. 18 (R12): KL-clip.
 *   s = sum_l |<precond_l, grad_l>_F|,  nu = s > 0 ? min(1, sqrt(kappa / (lr^2 s))) : 1,
 *   precond_l *= nu  (in place).
 * precond[l], grad[l]: device rows[l] x ld[l] (columns >= cols[l] are padding: never read into
 * the sum, scaled along with the row).  Any number of layers.  nu_out: device float (nullable);
 * s_out: device double (nullable).  Fixed reduction order (fp64 partial sums, per-layer sums in
 * layer order), so identical inputs give bitwise identical nu and outputs.
 * Workspace: per-CTA fp64 partials, per-layer dot products, nu. */
size_t kfac_kl_clip_workspace_size(const int32_t *rows, const int32_t *cols, int32_t num_layers);
kfac_status_t kfac_kl_clip(float *const *precond, const float *const *grad,
                           const int32_t *rows, const int32_t *cols, const int32_t *ld,
                           int32_t num_layers, float lr, float kappa,
                           float *nu_out, double *s_out,
                           void *ws, size_t ws_bytes, kfac_stream_t stream);

/* ---- Alg. 1 "Assign factors ... to unique workers".  Host only,
 * deterministic, identical on every rank (no communication).
 * dims[f], layer_of[f]: host, factor f's dimension and layer (paper order
 * [A_0, G_0, A_1, G_1, ...]).  owner[f]: host output rank in [0, world_size). */
kfac_status_t kfac_assign(const int32_t *dims, const int32_t *layer_of, int32_t num_factors,
                          int32_t num_layers, int32_t world_size, int32_t policy, int32_t *owner);

const char *kfac_status_string(kfac_status_t status);
const char *kfac_last_error(void);
/* Number of CUDA kernels this library has launched in this process (all threads). */
uint64_t kfac_launch_count(void);
int32_t kfac_version(void);

/* ---- Instrumentation (bench.py's roofline).  kfac_profile_start(k) arms per-launch timing of one
 * kernel class k (KFAC_PROF_*): every launch of that class records a CUDA event pair on the
 * stream it is launched on and adds its algorithmic bytes and flops.
 * kfac_profile_stop synchronises those events and returns the summed device time (ms), the
 * launch count and the algorithmic bytes/flops, then disarms.  Host only; at most one class at
 * a time; not for use inside CUDA-graph capture.  Returns KFAC_ERR_INVALID_VALUE for an unknown
 * class or null outputs. */
#define KFAC_PROF_TRD_PANEL 1   /* Householder tridiagonalisation panel (trd_panel)        */
#define KFAC_PROF_GEMM64 2      /* fp64-accumulating GEMMs of the eigensolver (gemm64_*)    */
#define KFAC_PROF_SYRK_TC 3     /* tcgen05 factor SYRK (syrk_tc_kernel)                     */
#define KFAC_PROF_GEMM_TC 4     /* tcgen05 preconditioning GEMMs (gemm_tc_kernel)           */
kfac_status_t kfac_profile_start(int32_t kernel_class);
kfac_status_t kfac_profile_stop(double *ms, int64_t *launches, double *bytes, double *flops);

#ifdef __cplusplus
}
#endif
#endif /* KFAC_H */
