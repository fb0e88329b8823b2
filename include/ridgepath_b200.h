/*
 * ridgepath_b200.h -- C ABI of the B200-native piCholesky cross-validation path.
 *
 * Drop-in boundary for the hot path of the reference package `ridgepath`
 * (/root/reference/pkg/src/ridgepath), `cvsearch.grid_search_pichol`
 * (cvsearch.py:206-243). The reference has no FFI: its boundary is its Python
 * API, which `paper_1404_0466_b200/{ridge,linalg,trivec,pichol,cvsearch}.py`
 * mirrors and which calls the entry points below through ctypes
 * (paper_1404_0466_b200/_lib.py). Each entry point names the reference
 * routine it replaces.
 *
 * Conventions
 *  - All matrices are FP64, caller-owned DEVICE memory; no allocation happens
 *    inside an entry point except where a *_workspace_size query says so.
 *  - Column-major d x d matrices (like the reference's F-ordered factors,
 *    linalg.py:101) unless stated otherwise; row-major n x d designs (numpy
 *    C-order X).
 *  - `stream` is a cudaStream_t passed as void*; every call is stream-ordered
 *    and asynchronous. Calls on distinct streams/devices are thread-safe.
 *  - Return: 0 = OK, < 0 = invalid argument (maps to UsageError /
 *    DimensionMismatch), > 0 = cudaError_t. rp_last_error() gives the message.
 *  - Numerical failures are reported in device `info` / `flags` arrays, like
 *    LAPACK info: the host maps them to NotPositiveDefinite
 *    (linalg.py:99-100) and SingularInterpolant (ridge.py:88-89).
 *
 * Packed-factor layout ("tile" layout): the order-d
 * lower triangle is cut into 64 x 64 tiles (I, J), I >= J, d padded up to
 * dp = 64 * ceil(d / 64). Tile (I, J) is stored at tile index I(I+1)/2 + J;
 * a tile holds P = r + 1 coefficient planes of 64 x 64, column-major with a
 * padded leading dimension of 68 (TP = 64*68 doubles per plane): plane p of
 * tile t at (t*P + p)*TP, element (i, j) at j*68 + i. A 16-column slab of a
 * tile is one contiguous block (the forward substitution's bulk copies) and a
 * 16-row slab is one 2-D TMA box (the backward substitution reads the
 * transposed operand from the same copy). Entries above the diagonal of a
 * diagonal tile and the padding are 0; padded diagonal entries are 1 in
 * plane 0 (the identity) so solves stay well defined. Per fold:
 * rp_theta_size(d, r) doubles.
 */
#ifndef RIDGEPATH_B200_H
#define RIDGEPATH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RP_METRIC_RMSE 0     /* cvsearch.RMSE (cvsearch.py:29) */
#define RP_METRIC_MISCLASS 1 /* cvsearch.MISCLASS (cvsearch.py:30) */

int rp_version(void);
const char* rp_last_error(void);
/* Number of kernels this library has launched in the process (evidence for bench.py). */
long long rp_launch_count(void);
/* Number of tensor-core (Ozaki) products whose device-side range guard tripped, so that the gated
 * FP64 DMMA fallback computed them, since the library was loaded (synchronizes the device). */
long long rp_ozaki_fallbacks(void);

/* Number of 64 x 64 tiles of the packed lower triangle of order d, and the
 * size in doubles of one fold's coefficient buffer. */
int64_t rp_tile_count(int d);
int64_t rp_theta_size(int d, int r);

/* (1) Hessian blocks.  Replaces ridge.assemble (ridge.py:50-60): H = X^T X
 * (:58-59) and g = X^T y (:60), evaluated per contiguous row block so that
 * H_f = sum_{b != f} G_b (contiguous FoldPlan, cvsearch.py:145-147).
 *   X: nblocks * rows_per_block rows, row-major, leading dim ldx (>= d)
 *   Y: same rows, row-major (rows x m), leading dim ldy (>= m); may be NULL when m == 0
 *   G: nblocks x (d x d column-major); the lower triangle is written (and the
 *      upper parts of the tiles that straddle the diagonal)
 *   C: nblocks x (d x m column-major)  (X_b^T Y_b)
 *   work: rp_gram_workspace_size(d, rows_per_block, nblocks) bytes (16-byte
 *      aligned), or NULL. With a workspace and d % 128 == 0, G is computed on
 *      the int8 tensor cores (tcgen05, CTA pairs) by the Ozaki scheme with 7
 *      balanced base-256 digits per value -- FP64-level accuracy (~1e-15
 *      relative to sqrt(G_ii G_jj)), NaN/inf propagated -- unless a column of X
 *      fails the device-side range guard (max |x| > 1024 rms(x): the truncation
 *      error would exceed FP64's by ~500x), in which case the same call computes G
 *      by FP64 DMMA (a gated kernel, no host synchronization); otherwise by FP64
 *      DMMA. C is computed by the same FP64 kernel on either path.   */
size_t rp_gram_workspace_size(int d, int64_t rows_per_block, int nblocks);
int rp_gram_blocks(const double* X, int64_t ldx, int64_t rows_per_block, int nblocks, int d,
                   const double* Y, int64_t ldy, int m, double* G, double* C, void* work, void* stream);

/* Per-block column sums of squares: yy[b][o] = sum_rows Y_b[row][o]^2 (the y^T y term of the
 * Gram-form hold-out error). */
int rp_col_sumsq(const double* Y, int64_t ldy, int64_t rows_per_block, int nblocks, int m, double* yy,
                 void* stream);

/* Fill the upper triangle of nmat column-major d x d matrices from the lower. */
int rp_symmetrize(double* G, int d, int64_t stride, int nmat, void* stream);

/* Per-fold shifted systems for the sampled-lambda factorizations (any nf, s: chunked per launch)
 * (pichol.py:105-107, `H + lam * eye`; H = X_tr^T X_tr of ridge.py:58 as a sum of fold blocks):
 *   A[f][s] = sum_{b != folds[f]} G_b + lams[s] * I  (b = 0..nblocks-1 in order; lower triangle,
 *                                                     d x d col-major)
 *   rhs[f]  = sum_{b != folds[f]} C_b                 (dp x m row-major, rows >= d zero)
 * A: nf*s*d*d. rhs: nf*dp*m. The sum of fold f does not depend on whether block f is among
 * the nblocks, so a fold can be assembled from the other folds' blocks before its own block
 * exists (folds_host[f] >= nblocks or -1: nothing is left out). */
int rp_fold_systems(const double* G, const double* C, int nblocks, int d, int m, const int* folds_host,
                    int nf, const double* lams_host, int s, double* A, double* rhs, void* stream);

/* (2) Batched blocked Cholesky, lower, in place.  Replaces linalg.cholesky's
 * dpotrf (linalg.py:98) for the s sampled lambdas of every local fold.
 * info[b] = 0 on success, j+1 when the leading minor of order j+1 is not
 * positive definite (LAPACK convention).  work: rp_potrf_workspace_size bytes
 * (16-byte aligned). Outer panels of 768 columns, 128-column blocks factored
 * left-looking on FP64 DMMA; the trailing updates A22 -= L21 L21^T run on the
 * int8 tensor cores by the Ozaki scheme (FP64-level accuracy, same range guard
 * and gated FP64 fallback as rp_gram_blocks) when d % 128 == 0. */
size_t rp_potrf_workspace_size(int d, int batch);

/* Path selection for A/B runs and tests (process-wide; workspace sizes follow it):
 *   "chol_ozaki" 0: Cholesky trailing updates on FP64 DMMA (default 1: int8 tensor cores)
 *   "gram_dmma"  1: Gram blocks on FP64 DMMA even with a workspace (default 0)
 *   "holdout_ozaki" 0: Gram-form hold-out on FP64 DMMA (default 1: int8 tensor cores)
 *   "profile"    1: time selected kernels with CUDA events (bench roofline)
 *   "solve_lam"  n: force the fused solve's lambda chunk (0 = planner)
 *   "solve_cluster" 2/4/8: fused solve on clusters of that many CTAs sharing each coefficient slab
 *                (TMA multicast; 0/1 = off, the default: measured slower)                     */
int rp_set_option(const char* name, int value);

/* Sum of the recorded durations (ms) of kernel `name` ("oz_syrk", "eval_solve",
 * "holdout_gemm"; NULL = all) since the last call; synchronizes the device. */
double rp_profile_ms(const char* name);
int rp_potrf_batched(double* A, int d, int64_t stride, int batch, int* info, void* work, void* stream);

/* (3)+(4) Polynomial fit of the packed factors.  Replaces trivec.bulk_gather
 * (trivec.py:165-191) + the normal-equation solve of pichol.fit
 * (pichol.py:122-125): theta_p = sum_s P[p][s] * L_s per packed entry, where the
 * host computed P = (V^T V)^{-1} V^T exactly as the reference (same V, same
 * COND_LIMIT rescale).  Also the Frobenius residual ||T - V theta||_F per fold.
 *   L: nf x s factors (d x d col-major, lower), P: (r+1) x s row-major,
 *   V: s x (r+1) row-major (host), theta: nf x tile-layout, resid: nf (device).
 *   Any s > r >= 0 (s <= 32 and r <= 4 keep P and V in kernel parameters; otherwise
 *   they are copied into the workspace).                                      */
int rp_fit_tiles(const double* L, int d, int s, int nf, int r, const double* P_host,
                 const double* V_host, double* theta, double* resid, void* work, void* stream);
size_t rp_fit_workspace_size(int d, int nf, int s, int r);

/* (5) Fused evaluate + solve.  Replaces, for all q lambdas at once,
 * pichol.eval_vector (pichol.py:143-151) + trivec.unvectorize
 * (trivec.py:150-162) + the singular check (ridge.py:88-89) +
 * linalg.solve_chol (linalg.py:104-128): W[f][:, j*m:(j+1)*m] solves
 * L_f(t_j) L_f(t_j)^T W = rhs[f], with L_f(t) = sum_p theta_p t^p evaluated
 * tile by tile in registers, never materialized.
 *   theta: nf x rp_theta_size(d, r) doubles; rhs: nf x (dp x m) row-major
 *   tvals: q values t_j = t_scale*lambda_j + t_shift (device)
 *   W: nf x (dp x ldw) row-major, ldw >= q*m, ldw even
 *   flags: nf x q ints, set to 1 where min |L_ii(t_j)| < 1e-12
 *   work: rp_eval_solve_workspace_size(d, r, nf, m, q) bytes (per-chunk solve rows).
 *   Degrees up to 4 run fused; a higher degree evaluates each lambda's factor into a
 *   one-plane tile buffer in the workspace (same Horner arithmetic) and solves it. */
size_t rp_eval_solve_workspace_size(int d, int r, int nf, int m, int q);
/* The launch plan rp_eval_solve uses for this shape on the current device (introspection for
 * benchmarks and tests; needs a GPU): plan[0] = lambdas per CTA of the main launch, plan[1] = its
 * chunks (CTAs) per fold, plan[2] = lambdas per job of the tail launch that covers each fold's last
 * lambdas on the SMs the main launch leaves idle (0: no tail launch), plan[3] = its CTAs. */
int rp_eval_solve_plan(int d, int r, int nf, int m, int q, int* plan);
int rp_eval_solve(const double* theta, int d, int r, int nf, const double* rhs, int m, const double* tvals,
                  int q, double* W, int64_t ldw, int* flags, void* work, void* stream);

/* Debug / single-lambda API (pichol.eval, pichol.py:154-164): dense d x d
 * column-major L(t) from one fold's tile-layout theta. */
int rp_eval_materialize(const double* theta, int d, int r, double t, double* L, void* stream);

/* Layout conversion between the tile layout and a reference VecLayout
 * permutation (trivec.py:65-120; perm[j] = column-major flat index of the
 * j-th packed entry). export: out[p][j] = theta_p at perm[j]; import: inverse. */
int rp_theta_export(const double* theta, int d, int r, const int64_t* perm, int64_t D, double* out,
                    void* stream);
int rp_theta_import(const double* vec, int d, int r, const int64_t* perm, int64_t D, double* theta,
                    void* stream);

/* (6) Hold-out error.  Replaces cvsearch.holdout_error (cvsearch.py:106-123)
 * for every (fold, lambda, output):
 *   direct: pred = X_val W (DMMA GEMM) fused with (pred - y)^2 or sign-mismatch
 *           row reduction (RMSE or MISCLASS)
 *   gram:   RMSE only, n_val*MSE = y^T y - 2 w^T C_f + w^T G_f w with G_f, C_f
 *           the fold's own Gram blocks. Only G_f's lower triangle is read
 *           (w^T G w = 2 w^T T w, T = strict_lower(G) + diag(G)/2) when G_f and W
 *           are 16-byte aligned with even sizes; otherwise G_f's upper triangle is
 *           filled in place first and the full product is used. T W runs on the int8
 *           tensor cores (Ozaki) unless "holdout_ozaki" is 0 or the operands fail the
 *           range guard (then FP64 DMMA). Columns whose Gram-form value would lose
 *           more than 20 bits to cancellation (y^T y + |2 w^T c| + w^T G w > 2^20 sse,
 *           a near-exact fit) are recomputed from the direct residual when Xval is
 *           given (Xval rows of fold f at Xval + f*fold_stride_rows*ldx, Y likewise).
 * Xval rows of fold f start at Xval + f*fold_stride_rows*ldx (same for Yval).
 * curves: nf x q x m.  work: rp_holdout_workspace_size bytes (16-byte aligned). */
size_t rp_holdout_workspace_size(int64_t n_val, int d, int q, int m, int nf);
int rp_holdout_direct(const double* Xval, int64_t ldx, int64_t fold_stride_rows, int64_t n_val, int d,
                      const double* Yval, int64_t ldy, int m, const double* W, int64_t ldw,
                      int64_t w_fold_stride, int q, int nf, int metric, double* curves, void* work,
                      void* stream);
int rp_holdout_gram(double* Gf, int64_t g_stride, const double* Cf, int64_t c_stride, const double* yy,
                    int64_t n_val, int d, int m, const double* W, int64_t ldw, int64_t w_fold_stride, int q,
                    int nf, const double* Xval, int64_t ldx, int64_t fold_stride_rows, const double* Yval,
                    int64_t ldy, double* curves, void* work, void* stream);

/* Fold mean + selection (cvsearch._merge, cvsearch.py:154-175): mean[j][o] =
 * (sum_f curves[f][j][o]) / k in fold order; best[o] = first argmin over j
 * (NaN-propagating like np.argmin).  curves: k x q x m. */
int rp_select(const double* curves, int k, int q, int m, double* mean, int* best, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RIDGEPATH_B200_H */
