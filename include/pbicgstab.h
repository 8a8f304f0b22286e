/*
 * pbicgstab.h -- C ABI of the B200-native preconditioned pipelined BiCGStab
 * (p-BiCGStab) library, arXiv 1809.01948 (S. Cools).
 *
 * The library solves A x = b for a sparse N x N matrix A with
 * Algorithm 2 "Preconditioned pipelined BiCGStab", Jacobi
 * preconditioner M = diag(A) (BASELINE; reading A3), periodic residual
 * replacement (eq:rr P:596-601, placed after line 20 P:602-603, period policy
 * P:607) and the true-vs-recursive residual gap history (eq:res_gap P:112-116).
 * All arithmetic is fp64 on the GPU (sm_100a); every step of the iteration runs
 * in this library's own CUDA kernels.  There is no CPU fallback: on a machine
 * without a usable CUDA device every call that needs the device returns
 * PBICG_ECUDA.
 *
 * Conventions shared by every entry point
 *  - Every call returns pbicg_status; 0 = PBICG_OK.  No exception crosses the ABI.
 *    On error, pbicgstab_last_error(handle) (or NULL for create errors) returns a
 *    thread-local / handle-owned message.
 *  - Pointers are BORROWED for the duration of the call only, unless stated.
 *  - "_dev" pointers are CUDA device pointers of the calling process's current
 *    device; "host" pointers are ordinary host memory.
 *  - Vector layout: natural x-fastest row order, row = x + nx*(y + ny*z), fp64.
 *  - A handle is not thread-safe; use one handle per thread/stream.
 */
#ifndef PBICGSTAB_H
#define PBICGSTAB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pbicg_ctx* pbicg_handle;

typedef enum {
  PBICG_OK = 0,
  PBICG_EINVAL = 1, /* bad argument (sizes, NULL, zero diagonal, bad option key) */
  PBICG_ECUDA = 2,  /* CUDA runtime error or no CUDA device */
  PBICG_ENCCL = 3,  /* NCCL error (multi-GPU) */
  PBICG_ENOMEM = 4, /* device or host allocation failed */
  PBICG_ESTATE = 5  /* handle in a failed state, or feature not available in this build */
} pbicg_status;

/* Outcome of a solve (reading A9). */
typedef enum {
  PBICG_CONVERGED = 0, /* ||r_i|| <= tol * ||b|| with r_i the recursive residual (A7) */
  PBICG_MAXIT = 1,     /* maxit iterations done without convergence */
  PBICG_BREAKDOWN = 2  /* non-finite or zero scalar denominator (A9); x = last finite iterate */
} pbicg_outcome;

/* Preconditioner M (reading A3 / A33 / A34):
 *   PBICG_PREC_JACOBI        M = diag(A), applied as fl(dinv_j v_j), dinv_j = 1/a_jj
 *   PBICG_PREC_BJ(b)         block Jacobi ("block preconditioners"; SURVEY
 *                            NEXT-4), b in {2,4,8,16,32}: M = the b x b diagonal blocks
 *                            of A over rows [kb, (k+1)b) (global numbering), each
 *                            inverted once by Gauss-Jordan elimination without
 *                            pivoting; (M^-1 v)_i = sum_k inv_ik v_{kb+k}, ascending k.
 *                            CSR: b in {2,4,8,16,32}, every rank's row_begin and
 *                            n_local multiples of b, all three methods.  Stencils:
 *                            b in {2,4,8}, nx % b == 0, full-line TMA tiles (nx <=
 *                            1024 in 2D, ~850 in 3D), all three methods (classic
 *                            BiCGStab's derived operands are derived, then
 *                            transformed once per staged element).  A zero pivot
 *                            is EINVAL.  Costs b-1 extra doubles per row read in
 *                            each kernel that applies M^-1.
 *   PBICG_PREC_ILU0          ILU(0): the incomplete LU factorisation with the sparsity
 *                            pattern of A (zero fill-in; Saad's IKJ variant restricted to
 *                            the pattern, pivots applied as reciprocals), M = L U;
 *                            M^-1 v by forward then backward substitution, every row in
 *                            ascending column order (reading A34).  Factorised once on
 *                            the host at create; applied by the library's wavefront
 *                            kernels (stencils: pipelined line wavefront; CSR: level-
 *                            ordered rows).  Multi-rank: each rank factorises its own
 *                            diagonal block (couplings to other ranks dropped from M).
 *                            All three methods; no automated replacement (EINVAL).
 *   PBICG_PREC_ICC0          ICC(0) (Table 1 "Precond."): for a
 *                            symmetric A (stencil: coef[1]==coef[2], coef[3]==coef[4],
 *                            coef[5]==coef[6]; CSR: each rank's diagonal block symmetric,
 *                            else EINVAL) the incomplete Cholesky factorisation with zero
 *                            fill-in, in root-free form: the same M and the same
 *                            arithmetic as PBICG_PREC_ILU0. */
typedef enum {
  PBICG_PREC_JACOBI = 1,
  PBICG_PREC_ILU0 = 2,
  PBICG_PREC_ICC0 = 3,
  PBICG_PREC_BLOCK_JACOBI = 0x100
} pbicg_prec;
#define PBICG_PREC_BJ(b) ((pbicg_prec)(PBICG_PREC_BLOCK_JACOBI | (b)))

/* Matrix-free constant-coefficient stencil (Table 1 shapes).
 *   dim = 2: 5-point on an nx x ny grid (nz ignored, treated as 1)
 *   dim = 3: 7-point on an nx x ny x nz grid
 *   coef = {centre, -x, +x, -y, +y, -z, +z}: row `row` has coef[1] at column
 *   row-1, coef[2] at row+1, coef[3] at row-nx, coef[4] at row+nx, coef[5] at
 *   row-nx*ny, coef[6] at row+nx*ny.  Legs leaving the grid are dropped
 *   (homogeneous Dirichlet, reading A5).  Each row is summed in ascending column
 *   order: -z, -y, -x, centre, +x, +y, +z.  coef[0] must be nonzero (Jacobi). */
typedef struct {
  int32_t dim;
  int64_t nx, ny, nz;
  double coef[7];
} pbicg_stencil;

/* General sparse matrix, this rank's rows in CSR (host arrays, copied).
 *   rows [row_begin, row_begin + n_local) of an n_global x n_global matrix;
 *   row_ptr[n_local+1] offsets into col/val (row_ptr[0] may be nonzero);
 *   col = GLOBAL column ids, sorted ascending within each row; every row must
 *   contain its diagonal entry with a nonzero value (Jacobi).  Rows are summed
 *   in the stored (ascending) order.  Multi-GPU: columns must lie within the
 *   neighbouring ranks' rows [row_begin - H, row_begin + n_local + H) with
 *   H = PBICG_CSR_HALO (nearest-neighbour halo only), else PBICG_EINVAL. */
typedef struct {
  int64_t n_global, row_begin, n_local;
  const int64_t* row_ptr;
  const int32_t* col;
  const double* val;
} pbicg_csr;

#define PBICG_CSR_HALO 4096

/* Multi-GPU description (one process per GPU).  NULL => single GPU.
 * nccl_id_halo / nccl_id_red: 128-byte ncclUniqueId blobs from
 * pbicgstab_get_unique_id() on rank 0, broadcast to all ranks by the caller.
 * nccl_id_red may be NULL (one communicator; the reductions then block the compute
 * stream: option "overlap" is forced to 0).  The reduction communicator is created
 * with ncclCommInitRankConfig and maxCTAs = 2 (tiny payloads), its side stream with
 * the highest stream priority.  nranks == 1 WITH an nccl_id_halo creates a one-rank
 * NCCL job that runs the multi-rank schedule (rank-row all-reduce, empty halo
 * groups, finalize kernels, peer-memory transport) -- bitwise equal to the plain
 * single-GPU path; nranks == 1 with a NULL id is the plain single-GPU path.
 * Stencils are split into contiguous z-slabs (3D) / y-slabs (2D) chosen by the
 * library (pbicgstab_local_rows reports them); CSR uses the caller's rows. */
typedef struct {
  int32_t nranks, rank;
  const void* nccl_id_halo;
  const void* nccl_id_red;
} pbicg_dist;

/* Create a solver for a stencil operator.  `cuda_stream` is the cudaStream_t every
 * kernel and copy of this handle is enqueued on; NULL => the handle creates (and
 * owns) a private cudaStreamNonBlocking stream, and every entry point that reads
 * caller memory first orders that stream after the legacy default stream (event
 * record on stream 0 + wait), so data written there before the call is visible.
 * Create-time uploads run on the handle's stream and finish before create returns.
 * Allocates the device workspace (14 fp64 vectors of n_local rows plus ghost
 * planes).  Errors: EINVAL (dim not 2/3, nx/ny/nz < 1, coef[0] == 0,
 * nranks/rank inconsistent), ECUDA, ENOMEM, ENCCL. */
pbicg_status pbicgstab_create_stencil(const pbicg_stencil* op, pbicg_prec prec,
                                      const pbicg_dist* dist, void* cuda_stream,
                                      pbicg_handle* out);

/* Create a solver for a CSR operator (copied to the device as a column-major
 * padded ELL matrix in the same per-row order).  Errors as above, plus EINVAL
 * for unsorted/out-of-range columns or a missing/zero diagonal. */
pbicg_status pbicgstab_create_csr(const pbicg_csr* op, pbicg_prec prec, const pbicg_dist* dist,
                                  void* cuda_stream, pbicg_handle* out);

/* Rank emulation on ONE device (testing the multi-rank path without several
 * GPUs): creates `nranks` handles out[0..nranks-1] that partition the operator
 * exactly as nranks processes would (slabs / the given CSR row blocks), share
 * one stream, and exchange halos and dot-product rows with device-to-device
 * copies instead of NCCL (loopback transport).  Kernels of different ranks never
 * wait on each other: everything is ordered on the one stream.
 * _csr_loopback takes ops[nranks] with contiguous ordered row blocks. */
pbicg_status pbicgstab_create_stencil_loopback(const pbicg_stencil* op, pbicg_prec prec,
                                               int32_t nranks, void* cuda_stream,
                                               pbicg_handle* out);
pbicg_status pbicgstab_create_csr_loopback(const pbicg_csr* ops, pbicg_prec prec, int32_t nranks,
                                           void* cuda_stream, pbicg_handle* out);
/* y = A x on a loopback group: x_dev[r], y_dev[r] are rank r's rows. */
pbicg_status pbicgstab_apply_loopback(pbicg_handle* hs, int32_t nranks, const double* const* x_dev,
                                      double* const* y_dev);
/* pbicgstab_solve over a loopback group (per-rank b, x0, x pointers; one
 * history, identical for every rank). */
pbicg_status pbicgstab_solve_loopback(pbicg_handle* hs, int32_t nranks,
                                      const double* const* b_dev, const double* const* x0_dev,
                                      double tol, int32_t maxit, int32_t rr_period,
                                      double* const* x_dev_out, double* rnorm_hist,
                                      double* gap_hist, int32_t* iters_out, int32_t* outcome_out);

/* Host-only (no device needed): the slab a stencil handle of `rank` out of
 * `nranks` will own -- contiguous z-slabs (3D) / y-slabs (2D) of floor or ceil
 * (outer/nranks) planes, lower ranks taking the remainder.  Rows
 * [row_begin, row_begin + n_local).  EINVAL if nranks exceeds the slab count. */
pbicg_status pbicgstab_stencil_partition(const pbicg_stencil* op, int32_t nranks, int32_t rank,
                                         int64_t* row_begin, int64_t* n_local);

/* Global rows owned by this rank: [row_begin, row_begin + n_local). */
pbicg_status pbicgstab_local_rows(pbicg_handle h, int64_t* row_begin, int64_t* n_local);

/* Options (int64 values):
 *   "bench"      1 => run exactly maxit iterations, no exit on convergence (A23)
 *   "graphs"     1 (default) => replay chunks of iterations as CUDA graphs
 *   "timing"     1 => record CUDA events around every kernel (disables graphs);
 *                read with pbicgstab_kernel_time
 *   "overlap"    1 (default) => multi-GPU: each global reduction runs on a side
 *                stream behind the halo exchange / SpMV the next phase needs;
 *                0 => blocking on the compute stream
 *   "tile"       1 (default) => stencil sweeps use the TMA-staged 2.5D kernels
 *                (full-line tiles; x-segmented tiles for even nx > 1024 and 3D nx >
 *                ~850; odd nx beyond those keeps the line kernels); 0 => plain line
 *                kernels (same results; not with block Jacobi)
 *   "csr_tma"    1 (default) => CSR with the Jacobi preconditioner: sweeps A and C
 *                stream their vectors through shared memory with bulk copies
 *                (c_sweep_tma); 0 => per-row global loads (same results)
 *   "pdl"        1 => launch the tile kernels with programmatic dependent launch:
 *                the next sweep's CTAs are scheduled as the previous sweep's CTAs
 *                retire (griddepcontrol); same results.  Default 0: measured +1-15%
 *                without CUDA graphs, within +-2% with them
 *   "schedule"   0 (default) auto (stencil: fused, CSR: split); 1 fused 2-sweep
 *                (stencil only: t, v recomputed inside the sweeps, 24 passes); 2 split
 *                4-phase (the paper's pipeline: stored t, v, stand-alone SpMVs the
 *                reductions hide behind, 32 passes; stencil: Jacobi, method 0,
 *                rr_auto off)
 *   "method"     0 (default) p-BiCGStab, Alg. 2; 1 classic preconditioned
 *                BiCGStab, Alg. 1; 2 preconditioned pipelined CG (the
 *                paper's p-CG comparison, reconstructed: DESIGN.md A19).
 *                Methods 1 and 2 need rr_period = 0; on a stencil also the TMA tile
 *                kernels (nx <= 1024; EINVAL otherwise); every preconditioner
 *   "transport"  multi-rank reductions: 0 (default) NCCL all-reduce of the zero-padded
 *                rank rows (loopback: device copies); 1 peer memory -- the last CTA of
 *                each reducing kernel stores its rank's Dot2 pairs into every rank's
 *                receive buffer over NVLink (CUDA IPC mappings exchanged once with an
 *                NCCL all-gather) and raises a flag; the finalize kernel waits for the
 *                P flags.  No collective launch per reduction.  Stencil, fused
 *                schedule: sweeps A and C also store their boundary planes of z_i and
 *                w_{i+1} into the neighbours' ghost planes (published by the same
 *                flags), so no halo exchange is enqueued for them.  Collective option for
 *                NCCL ranks (all call it with the same value); <= 8 ranks
 *   "rr_auto"    1 => automated residual replacement: the run-time bound
 *                f^r_i on the residual gap (eq:DDr_bound) is propagated on the device
 *                and iteration i replaces when f_{i-1} <= sqrt(eps)||r_{i-1}|| and
 *                f_i > sqrt(eps)||r_i|| (eq:criterion).  Needs method 0, the tile
 *                kernels on a stencil (not odd nx > 1024) and rr_period = 0 in
 *                pbicgstab_solve
 * Errors: EINVAL for an unknown key or bad value. */
pbicg_status pbicgstab_set_option(pbicg_handle h, const char* key, int64_t value);

/* y = A x for this rank's rows (x_dev, y_dev: n_local doubles on the device).
 * Same arithmetic as the solver's SpMV (ascending column order, no FMA).  Used
 * to form b = A x* for synthetic problems.  Collective for nranks > 1. */
pbicg_status pbicgstab_apply(pbicg_handle h, const double* x_dev, double* y_dev);

/* Solve A x = b with p-BiCGStab (Alg. 2).  Collective: every rank calls it with
 * identical scalar arguments.  Host-synchronous: returns after the histories are
 * on the host.
 *   b_dev, x0_dev   device, n_local doubles (this rank's rows)
 *   tol             relative to ||b||_2: stop when ||r_i|| <= tol*||b|| (A7)
 *   maxit >= 0      iteration cap
 *   rr_period >= 0  residual replacement after line 20 of every iteration i with
 *                   (i+1) % rr_period == 0, until ||r_i|| < sqrt(eps)||r_0||
 *                   (A11, A12); 0 disables replacement
 *   x_dev_out       device, n_local doubles; may alias x0_dev
 *   rnorm_hist      host, >= maxit+1 doubles: ||r_i|| for i = 0..iters
 *   gap_hist        host, >= maxit+1 doubles, or NULL (no gap tracking):
 *                   ||(b - A x_i) - r_i|| for i = 0..iters (eq:res_gap P:113)
 *   iters_out       completed iterations;  outcome_out  pbicg_outcome
 * Entries beyond iters are left untouched. */
pbicg_status pbicgstab_solve(pbicg_handle h, const double* b_dev, const double* x0_dev,
                             double tol, int32_t maxit, int32_t rr_period, double* x_dev_out,
                             double* rnorm_hist, double* gap_hist, int32_t* iters_out,
                             int32_t* outcome_out);

/* Same as pbicgstab_solve with HOST b, x0 and x_out (n_local doubles each); the
 * host<->device copies happen inside the call (end-to-end entry point). */
pbicg_status pbicgstab_solve_host(pbicg_handle h, const double* b_host, const double* x0_host,
                                  double tol, int32_t maxit, int32_t rr_period,
                                  double* x_host_out, double* rnorm_hist, double* gap_hist,
                                  int32_t* iters_out, int32_t* outcome_out);

/* Per-kernel statistics since the last reset (reset = 1 clears them).
 *   name: "init", "sweepA", "sweepC", "spmvB", "spmvD", "rr1", "rr2", "gap",
 *   "apply", "fin" (multi-rank scalar finalisation), "cl1", "cl2", "cl3" (classic
 *   BiCGStab), "pcg" (p-CG), "prec" (stand-alone M^-1: block Jacobi, ILU(0)), or "all".
 *   launches: kernel launches issued (graph nodes count once per replay);
 *   ms: summed CUDA-event time (only with option "timing"; else NaN). */
pbicg_status pbicgstab_kernel_time(pbicg_handle h, const char* name, int64_t* launches,
                                   double* ms, int32_t reset);

/* Algorithmic HBM bytes one launch of kernel `name` must move for this handle's
 * operator; 0 if unknown. */
pbicg_status pbicgstab_kernel_bytes(pbicg_handle h, const char* name, double* bytes);

/* Replacement record of the last solve on h (rank 0's handle for a loopback
 * group).  fr_hist (host, >= iters+1 doubles, or NULL): f^r_i, i = 0..iters, with
 * option rr_auto (NaN otherwise).  rr_iters (host, cap ints, or NULL): the
 * iterations i whose line 20 was followed by a replacement (periodic or
 * automated), ascending; *n_rr = their number (may exceed cap).
 * ESTATE before the first solve. */
pbicg_status pbicgstab_rr_info(pbicg_handle h, double* fr_hist, int32_t* rr_iters, int32_t cap,
                               int32_t* n_rr);

/* Parity diagnostics: the scalars of the last p-BiCGStab solve on h
 * (rank 0's handle for a loopback group), per iteration i < min(iters, cap):
 * out[9i..9i+8] = alpha_i, beta_i, omega_i, rho_i = (r^0, r_i), then the raw Dot2
 * results (q_i, y_i), (y_i, y_i) (line 12) and (r^0, w_{i+1}), (r^0, s_i), (r^0, z_i)
 * (line 21, of the replaced vectors after a replacement) -- the layout of the oracle's
 * scalar trace, so the first iteration and dot where a run leaves the oracle, and by
 * how many ulps, can be named.  Rows of iterations that stopped
 * before omega_i was formed are unspecified.  EINVAL for methods 1 / 2, ESTATE
 * before the first solve. */
pbicg_status pbicgstab_scalar_trace(pbicg_handle h, double* out, int32_t cap);

/* ncclUniqueId blob (128 bytes) for multi-GPU creation; ESTATE without NCCL. */
pbicg_status pbicgstab_get_unique_id(void* out128);

/* Error message for the last failing call on h (h may be NULL: last create error
 * on this thread).  Owned by the library; valid until the next call. */
const char* pbicgstab_last_error(pbicg_handle h);

/* Release every resource of h.  NULL is a no-op. */
void pbicgstab_destroy(pbicg_handle h);

#ifdef __cplusplus
}
#endif
#endif /* PBICGSTAB_H */
