// eigen_trd.cuh -- per-factor job of the dense symmetric eigensolver (eigen_trd.cu) and the
// interface of its two-stage tridiagonalisation (eigen_sbr.cu).  Internal to libkfac.
#pragma once

#include "internal.cuh"

#include <vector>

namespace kfac {

struct TrdJob {
    const float *F;
    float *Q, *evals;
    int *info;
    float *A;          // n x ldw working matrix (full symmetric storage, pads zero)
    float *Vb;         // n x ldw reflectors: column k = v_k (v_k[k+1] = 1, zero above)
    double *Vd;        // fp64 reflectors for the back-transformation GEMMs: column k = v_k with
                       // v_k[k + off] = 1, zero above (one-stage: copy of Vb; two-stage: stage 1)
    float *VW, *WV;    // n x 64 panel buffers: [V | W] and [W | V] of the current panel
    double *VWd, *WVd; // fp64 copies of the same (float) values: operands of the trailing update
    double *Z0, *Z1;   // n x ldw eigenvectors of T (D&C ping-pong), fp64
    double *Qnd, *Tmp; // n x ldw D&C scratch (permuted/rotated columns, GEMM output)
    double *Sb;        // n x ldw D&C secular eigenvectors S
    double *Yb, *Y2b;  // kBt x ldw back-transformation scratch
    double *Gb, *Tb;   // kBt x kBt Gram matrix V^T V and WY factor T
    double *Wt;        // kBt x kBt scratch for the recursive T
    double *d, *e, *tau;       // tridiagonal T and reflector scalars
    double *x, *y;             // corrected column / mat-vec result (sytrd)
    double *D;                 // current eigenvalues of the D&C subproblems
    double *dval, *zval;       // merge: sorted (d, z) -- non-deflated first, deflated last
    double *rtau, *wz;         // merge: root offsets, z-hat
    double *vnorm;             // merge: eigenvector column norms
    double *rot_c, *rot_s;     // merge: Givens rotations
    int *col, *posof, *rorg, *rot_p, *rot_j, *srcpos;
    int *ctyp;                 // merge: column type (1 upper, 2 mixed, 3 lower), then GEMM position
    int *mstate;               // per merge at slot a: {k, nrot, k, k1 + k2, 0, k, k, k1}
                               // (two GEMM dynamic {N, K, K start} triples: upper and lower rows)
    double *mscal;             // per merge: {rho2, tol}
    double *part;              // kMaxGroupCtas x kPart
    double *DP;                // symv direct partials  [n][ldp]  (row, 128-column chunk)
    double *TP;                // symv transposed partials [n][ldtp] (column, 64-row block)
    // ---- two-stage reduction (eigen_sbr.cu; null for one-stage factors) ----
    double *Ad;                // n x ldw fp64 working matrix of stage 1 (lower triangle live)
    double *Xs;                // n x 16: X' = A22 V T of the current panel
    double *VWs, *WVs;         // n x 32: [V | W] and [W | V], operands of the rank-32 update
    double *Ts, *Ms;           // 16 x 16: panel WY factor T, and M = T^T V^T X'
    double *Ps;                // per 64-row tile: partial V^T X' (16 x 16)
    double *Rq;                // stage-2 reflectors, [k][s][16] = (v_1 .. v_15, tau) of step (s, k)
    int ldp, ldtp;
    unsigned *bar;
    int n, ldF, ldQ, ldw;
    int levels;                // D&C merge levels (n <= kLeaf -> 0)
    int off;                   // row offset of reflector k's unit entry: 1 (one-stage), 16 (two-stage)
};

// Eigenvectors of T after the last merge level: level l writes Z0 (l even) / Z1 (l odd).
__host__ __device__ inline double *final_z(const TrdJob &J) { return (J.levels & 1) ? J.Z1 : J.Z0; }

// ------------------------------------------------------------------------------------------------
// Two-stage tridiagonalisation for the large factors (eigen_sbr.cu):
//   stage 1  F -> B = Q1^T F Q1, B symmetric with lower bandwidth kSbrBw (panels of kSbrBw columns:
//            Householder QR of the panel below the band, two-sided WY update of the trailing matrix
//            as fp64 DMMA products);
//   stage 2  B -> T = Q2^T B Q2 tridiagonal by bulge chasing (one thread-block cluster per factor,
//            the band resident in distributed shared memory, one warp per sweep segment);
//   Q2 Z     the stage-2 reflectors applied to the eigenvectors of T (before the Q1 blocks, which
//            the one-stage back-transformation applies with reflector offset kSbrBw).
namespace sbr {
constexpr int kSbrBw = 16;               // band width b
constexpr int kSbrMinN = 1024;           // smaller factors stay on the one-stage reduction
constexpr int kSbrMaxN = 5632;           // the band must fit 8 CTAs' shared memory (stage 2)

inline bool eligible(int n) { return n >= kSbrMinN && n <= kSbrMaxN; }
// Reduction of each factor of a call (1 = two-stage), from the dims and the eigen flags only.
std::vector<char> route(const int32_t *dims, int count, uint32_t flags);

// Workspace the two-stage fields of one factor need (bytes, 256-aligned slices).
size_t extra_bytes(int n, int ldw);
// Carve those fields out of the workspace, starting at offset `cur` (offsets, rebased by the caller).
void plan_fields(TrdJob &J, size_t &cur);
void rebase_fields(TrdJob &J, char *base);

// Stage 1 + stage 2 for the factors `ids` (indices into jobs / djobs): on return J.d, J.e hold T,
// J.Vd / J.tau the stage-1 reflectors (offset kSbrBw) and J.Rq the stage-2 reflectors.
kfac_status_t reduce(const TrdJob *djobs, const std::vector<TrdJob> &jobs, const std::vector<int> &ids,
                     cudaStream_t s);
// The two halves of reduce: stage 1 (dense -> band, fills the GPU) and stage 2 (bulge chase, one
// cluster of chase_ctas-many CTAs in all, latency-bound).
kfac_status_t stage1(const TrdJob *djobs, const std::vector<TrdJob> &jobs, const std::vector<int> &ids,
                     cudaStream_t s);
kfac_status_t chase(const TrdJob *djobs, const std::vector<TrdJob> &jobs, const std::vector<int> &ids,
                    cudaStream_t s);
int chase_ctas(const std::vector<TrdJob> &jobs, const std::vector<int> &ids);
// final_z(J) <- Q2 final_z(J) for the factors `ids`.
kfac_status_t apply_q2(const TrdJob *djobs, const std::vector<TrdJob> &jobs, const std::vector<int> &ids,
                       cudaStream_t s);
}  // namespace sbr

}  // namespace kfac
