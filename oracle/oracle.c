/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct fp64 CPU
 * implementation of what the p-BiCGStab hot path computes, written from the paper
 * (arXiv 1809.01948, S. Cools, "Analyzing and improving maximal attainable accuracy
 * in the communication hiding pipelined BiCGStab method").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  It shares NO code with the CUDA path
 * (paper_1809_01948_b200/csrc) and includes none of its headers.
 *
 * Citation convention: "P:n" is line n of the paper's text, with the
 * algorithm / equation it falls in.  Readings of ambiguous passages are the
 * A-numbers of DESIGN.md section "Readings".
 *
 * Conventions (readings A4-A6):
 *   - every vector expression is evaluated left to right with the brackets as
 *     printed; build with -ffp-contract=off so no FMA contraction
 *     happens anywhere except the explicit fma() inside TwoProd;
 *   - SpMV sums a row's stored entries in ascending column order, starting from
 *     +0.0 (A5);
 *   - dot products are Dot2 (TwoProd + TwoSum compensated, rounded once) (A6);
 *     flag ORC_PLAIN_DOT switches to a plain sequential sum (diagnostic only);
 *   - Jacobi: dinv_j = 1.0 / a_jj, applied as fl(dinv_j * v_j) (A3).
 *
 * Parity status of each function: see the pins in tests/test_oracle_*.py and
 * DESIGN.md "Oracle pins".  pcg / pipecg: the paper gives no p-CG pseudocode
 * (P:465-472 defers to companion work); the reconstruction is pinned only by
 * exact rational equivalence with PCG (tests/test_oracle_rational.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_BENCH 1      /* run maxit iterations: no exit on convergence (A23) */
#define ORC_PLAIN_DOT 2  /* plain left-to-right dot instead of Dot2 (diagnostic) */
#define ORC_GAP 4        /* compute the residual gap history */
#define ORC_AUTO_RR 8    /* automated replacement: bound f^r_i (eq:DDr_bound) + eq:criterion */
#define ORC_ILU0 16      /* preconditioner ILU(0) (= ICC(0) for symmetric A), reading A34 */
#define ORC_SCW 9        /* doubles per iteration of orc_pbicgstab's scalar trace */

#define OUT_CONVERGED 0
#define OUT_MAXIT 1
#define OUT_BREAKDOWN 2

/* ------------------------------------------------------------------------- */
/* Dot2 (Ogita-Rump-Oishi): error-free TwoProd + TwoSum, one final rounding.  */
/* The paper only fixes the error bound |(v,w) - fl((v,w))| <= N|v||w|eps     */
/* (P:49); Dot2 is reading A6.                                               */
/* ------------------------------------------------------------------------- */
static void two_sum(double a, double b, double* s, double* e) {
  double ss = a + b;
  double z = ss - a;
  *e = (a - (ss - z)) + (b - z);
  *s = ss;
}

double orc_dot2(int64_t n, const double* x, const double* y) {
  double P = 0.0, S = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    double h = x[j] * y[j];
    double r = fma(x[j], y[j], -h); /* exact low part of the product */
    double q;
    two_sum(P, h, &P, &q);
    S = S + (q + r);
  }
  return P + S;
}

double orc_dot_plain(int64_t n, const double* x, const double* y) {
  double s = 0.0;
  for (int64_t j = 0; j < n; ++j) s = s + x[j] * y[j];
  return s;
}

static double dotf(int flags, int64_t n, const double* x, const double* y) {
  return (flags & ORC_PLAIN_DOT) ? orc_dot_plain(n, x, y) : orc_dot2(n, x, y);
}

/* ------------------------------------------------------------------------- */
/* Sparse matrix in CSR, columns ascending per row.                           */
/* ------------------------------------------------------------------------- */
/* y = A x: "fl(Av)" of P:48.  Row sum over stored entries in ascending column
 * order, starting from +0.0 (reading A5). */
void orc_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
              const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) acc = acc + va[p] * x[ci[p]];
    y[i] = acc;
  }
}

/* Jacobi preconditioner M = diag(A) (reading A3): dinv_j = 1 / a_jj.
 * Returns -1 if a diagonal entry is missing or zero. */
int orc_jacobi_dinv(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
                    double* dinv) {
  for (int64_t i = 0; i < n; ++i) {
    double d = 0.0;
    int found = 0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      if (ci[p] == i) { d = va[p]; found = 1; }
    if (!found || d == 0.0) return -1;
    dinv[i] = 1.0 / d;
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Preconditioner M^{-1} (reading A33).  flags bits 8-15 =  */
/* block size b: b <= 1 is Jacobi (A3), M^{-1} u = fl(dinv_j * u_j); b >= 2 is   */
/* block Jacobi with the b x b diagonal blocks of A over rows [kb, (k+1)b)      */
/* ("block preconditioners"): the blocks are inverted once by plain      */
/* Gauss-Jordan elimination without pivoting and applied as                    */
/* (M^{-1}u)_i = sum_k inv_ik u_{kb+k}, ascending k from +0.0.                  */
/* ------------------------------------------------------------------------- */
typedef struct {
  int64_t n;
  int b;
  double* inv; /* b = 1: dinv[n]; else row-major [n][b]: row i of its block's inverse */
  /* ILU(0) (b = 0): the factors on the pattern of the preconditioner matrix */
  const int64_t* rp;
  const int64_t* ci;
  double* lu;   /* strictly lower part: multipliers l_ik; upper part: u_ij; diagonal: u_ii */
} Prec;

/* ------------------------------------------------------------------------- */
/* ILU(0) / ICC(0) (Table 1 "Precond." ICC(0); "incomplete Cholesky  */
/* preconditioner with zero fill-in"; reading A34).  */
/* The incomplete factorisation with the sparsity pattern of A (no fill):        */
/* Saad's IKJ variant of Gaussian elimination restricted to the pattern --       */
/*   for i = 0..n-1:                                                             */
/*     for k < i with (i,k) in NZ, ascending:  a_ik := a_ik * uinv_k             */
/*       for j > k with (k,j) in NZ, ascending: if (i,j) in NZ:                  */
/*                                               a_ij := a_ij - a_ik * a_kj      */
/*     uinv_i := 1 / a_ii                                                        */
/* giving M = L U (L unit lower triangular with the multipliers l_ik, U upper    */
/* with u_ij); for symmetric A this M is the incomplete Cholesky (ICC(0)) M =     */
/* L~ L~^T in root-free form (L~ = L diag(u)^{1/2}).  The pivots are applied as   */
/* reciprocals (uinv, as the Jacobi dinv of A3).  M^{-1} v: forward              */
/* y_i = v_i - sum_{k<i} l_ik y_k, then backward x_i = (y_i - sum_{j>i} u_ij x_j) */
/* * uinv_i, every row summed in ascending column order (A5).  Returns -1 on a   */
/* missing or zero pivot. */
int orc_ilu0_factor(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
                    double* lu, double* uinv) {
  for (int64_t p = 0; p < rp[n]; ++p) lu[p] = va[p];
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t p = rp[i]; p < rp[i + 1] && ci[p] < i; ++p) {
      const int64_t k = ci[p];
      lu[p] = lu[p] * uinv[k];
      for (int64_t q = rp[k]; q < rp[k + 1]; ++q) {
        if (ci[q] <= k) continue;
        for (int64_t p2 = rp[i]; p2 < rp[i + 1]; ++p2)
          if (ci[p2] == ci[q]) { lu[p2] = lu[p2] - lu[p] * lu[q]; break; }
      }
    }
    double d = 0.0;
    int found = 0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      if (ci[p] == i) { d = lu[p]; found = 1; }
    if (!found || d == 0.0 || !isfinite(d)) return -1;
    uinv[i] = 1.0 / d;
  }
  return 0;
}

/* The matrix whose ILU(0) defines M (NULL: A itself).  Test infrastructure sets it
 * to the block-diagonal part of A over the ranks' row blocks for the multi-rank
 * reading of A34 (each rank factorises its own diagonal block). */
static int64_t g_pm_n = -1;
static const int64_t *g_pm_rp = 0, *g_pm_ci = 0;
static const double* g_pm_va = 0;
void orc_set_prec_matrix(int64_t n, const int64_t* rp, const int64_t* ci, const double* va) {
  g_pm_n = rp ? n : -1;
  g_pm_rp = rp;
  g_pm_ci = ci;
  g_pm_va = va;
}

#define ORC_BLOCK(flags) (((flags) >> 8) & 0xff)

/* Gauss-Jordan inverse of the dense b x b matrix a (row-major, destroyed) into e.
 * Returns -1 on a zero pivot. */
int orc_gauss_jordan(int b, double* a, double* e) {
  for (int r = 0; r < b; ++r)
    for (int c = 0; c < b; ++c) e[r * b + c] = (r == c) ? 1.0 : 0.0;
  for (int p = 0; p < b; ++p) {
    const double piv = a[p * b + p];
    if (piv == 0.0 || !isfinite(piv)) return -1;
    const double f = 1.0 / piv;
    for (int c = 0; c < b; ++c) {
      a[p * b + c] = a[p * b + c] * f;
      e[p * b + c] = e[p * b + c] * f;
    }
    for (int r = 0; r < b; ++r) {
      if (r == p) continue;
      const double g = a[r * b + p];
      for (int c = 0; c < b; ++c) {
        a[r * b + c] = a[r * b + c] - g * a[p * b + c];
        e[r * b + c] = e[r * b + c] - g * e[p * b + c];
      }
    }
  }
  return 0;
}

static int prec_make(int32_t flags, int64_t n, const int64_t* rp, const int64_t* ci,
                     const double* va, Prec* P) {
  const int b = ORC_BLOCK(flags) > 1 ? ORC_BLOCK(flags) : 1;
  P->n = n;
  P->b = b;
  P->lu = 0;
  if (flags & ORC_ILU0) {
    if (g_pm_rp && g_pm_n == n) { rp = g_pm_rp; ci = g_pm_ci; va = g_pm_va; }
    P->b = 0;
    P->rp = rp;
    P->ci = ci;
    P->inv = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    P->lu = (double*)calloc((size_t)(rp[n] > 0 ? rp[n] : 1), sizeof(double));
    if (orc_ilu0_factor(n, rp, ci, va, P->lu, P->inv) != 0) {
      free(P->lu); free(P->inv); P->lu = 0; return -1;
    }
    return 0;
  }
  P->inv = (double*)calloc((size_t)(n > 0 ? n : 1) * (size_t)b, sizeof(double));
  if (b == 1) {
    if (orc_jacobi_dinv(n, rp, ci, va, P->inv) != 0) { free(P->inv); return -1; }
    return 0;
  }
  if (n % b != 0) { free(P->inv); return -1; }
  double* a = (double*)calloc((size_t)b * b, sizeof(double));
  double* e = (double*)calloc((size_t)b * b, sizeof(double));
  for (int64_t k0 = 0; k0 < n; k0 += b) {
    for (int q = 0; q < b * b; ++q) a[q] = 0.0;
    for (int r = 0; r < b; ++r)
      for (int64_t p = rp[k0 + r]; p < rp[k0 + r + 1]; ++p)
        if (ci[p] >= k0 && ci[p] < k0 + b) a[r * b + (ci[p] - k0)] = va[p];
    if (orc_gauss_jordan(b, a, e) != 0) { free(a); free(e); free(P->inv); return -1; }
    for (int r = 0; r < b; ++r)
      for (int c = 0; c < b; ++c) P->inv[(size_t)(k0 + r) * b + c] = e[r * b + c];
  }
  free(a);
  free(e);
  return 0;
}

/* v := M^{-1} u */
static void pprec(const Prec* P, const double* u, double* v) {
  const int b = P->b;
  if (b == 0) { /* ILU(0): forward then backward substitution (A34) */
    for (int64_t i = 0; i < P->n; ++i) {
      double acc = u[i];
      for (int64_t p = P->rp[i]; p < P->rp[i + 1] && P->ci[p] < i; ++p)
        acc = acc - P->lu[p] * v[P->ci[p]];
      v[i] = acc;
    }
    for (int64_t i = P->n - 1; i >= 0; --i) {
      double acc = v[i];
      for (int64_t p = P->rp[i]; p < P->rp[i + 1]; ++p)
        if (P->ci[p] > i) acc = acc - P->lu[p] * v[P->ci[p]];
      v[i] = acc * P->inv[i];
    }
    return;
  }
  if (b == 1) {
    for (int64_t j = 0; j < P->n; ++j) v[j] = P->inv[j] * u[j];
    return;
  }
  for (int64_t j = 0; j < P->n; ++j) {
    const int64_t k0 = j - j % b;
    double acc = 0.0;
    for (int k = 0; k < b; ++k) acc = acc + P->inv[(size_t)j * b + k] * u[k0 + k];
    v[j] = acc;
  }
}

/* ||M^{-1}||_2 <= max over blocks of sqrt(||B^-1||_1 ||B^-1||_inf) (b = 1: max |dinv|),
 * with row / column sums in ascending order (reading A29 for M^{-1}). */
static double prec_norm_bound(const Prec* P) {
  const int b = P->b;
  double mx = 0.0;
  if (b == 1) {
    for (int64_t j = 0; j < P->n; ++j)
      if (fabs(P->inv[j]) > mx) mx = fabs(P->inv[j]);
    return mx;
  }
  for (int64_t k0 = 0; k0 < P->n; k0 += b) {
    double rmax = 0.0, cmax = 0.0;
    for (int r = 0; r < b; ++r) {
      double rs = 0.0;
      for (int c = 0; c < b; ++c) rs = rs + fabs(P->inv[(size_t)(k0 + r) * b + c]);
      if (rs > rmax) rmax = rs;
    }
    for (int c = 0; c < b; ++c) {
      double cs = 0.0;
      for (int r = 0; r < b; ++r) cs = cs + fabs(P->inv[(size_t)(k0 + r) * b + c]);
      if (cs > cmax) cmax = cs;
    }
    const double nb = sqrt(cmax * rmax);
    if (nb > mx) mx = nb;
  }
  return mx;
}

static void prec_free(Prec* P) {
  free(P->inv);
  if (P->lu) free(P->lu);
}

/* v := M^{-1} u for tests (flags as the solvers'); -1 if M cannot be formed. */
int orc_prec_apply(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
                   int32_t flags, const double* u, double* v) {
  Prec P;
  if (prec_make(flags, n, rp, ci, va, &P) != 0) return -1;
  pprec(&P, u, v);
  prec_free(&P);
  return 0;
}

/* Constant-coefficient 5-point (dim=2) / 7-point (dim=3) stencil written out
 * as CSR, natural x-fastest ordering row = x + nx*(y + ny*z), Dirichlet legs
 * dropped (Table 1 P:645-704 shapes; reading A5).  coef = {centre, -x, +x,
 * -y, +y, -z, +z}.  Entries of a row are emitted in ascending column order:
 * -z, -y, -x, centre, +x, +y, +z.  rp has n+1 entries; ci/va need 7n room.
 * Returns nnz. */
int64_t orc_stencil_csr(int dim, int64_t nx, int64_t ny, int64_t nz, const double* coef,
                        int64_t* rp, int64_t* ci, double* va) {
  if (dim == 2) nz = 1;
  int64_t n = nx * ny * nz, nnz = 0;
  for (int64_t zz = 0; zz < nz; ++zz)
    for (int64_t yy = 0; yy < ny; ++yy)
      for (int64_t xx = 0; xx < nx; ++xx) {
        int64_t row = xx + nx * (yy + ny * zz);
        rp[row] = nnz;
        if (dim == 3 && zz > 0) { ci[nnz] = row - nx * ny; va[nnz++] = coef[5]; }
        if (yy > 0) { ci[nnz] = row - nx; va[nnz++] = coef[3]; }
        if (xx > 0) { ci[nnz] = row - 1; va[nnz++] = coef[1]; }
        ci[nnz] = row; va[nnz++] = coef[0];
        if (xx < nx - 1) { ci[nnz] = row + 1; va[nnz++] = coef[2]; }
        if (yy < ny - 1) { ci[nnz] = row + nx; va[nnz++] = coef[4]; }
        if (dim == 3 && zz < nz - 1) { ci[nnz] = row + nx * ny; va[nnz++] = coef[6]; }
      }
  rp[n] = nnz;
  return nnz;
}

/* ||A||_2 <= sqrt(||A||_1 ||A||_inf) (Hoelder): the upper bound the run-time
 * gap bound uses for ||A|| (reading A29).  Row sums in ascending column order,
 * column sums in ascending row order, |a_ij| summed from +0.0. */
double orc_anorm_bound(int64_t n, const int64_t* rp, const int64_t* ci, const double* va) {
  double* col = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  double rmax = 0.0, cmax = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double rs = 0.0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      rs = rs + fabs(va[p]);
      col[ci[p]] = col[ci[p]] + fabs(va[p]);
    }
    if (rs > rmax) rmax = rs;
  }
  for (int64_t j = 0; j < n; ++j)
    if (col[j] > cmax) cmax = col[j];
  free(col);
  return sqrt(cmax * rmax);
}

/* ------------------------------------------------------------------------- */
/* Workspace helper                                                          */
/* ------------------------------------------------------------------------- */
static double* vec(int64_t n) { return (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }

/* gap = || (b - A x) - r ||  (eq:res_gap; reading A13). */
static double res_gap(int flags, int64_t n, const int64_t* rp, const int64_t* ci,
                      const double* va, const double* b, const double* x, const double* r,
                      double* tmp) {
  orc_spmv(n, rp, ci, va, x, tmp);
  for (int64_t j = 0; j < n; ++j) tmp[j] = (b[j] - tmp[j]) - r[j];
  return sqrt(dotf(flags, n, tmp, tmp));
}

/* Number of vectors recorded per trace slot by orc_pbicgstab. */
#define NTRACE 15
/* trace slot layout (slot i = iteration i, slot maxit = final state):
 *  0 x_i  1 r_i  2 k_i  3 w_i  4 m_i  5 t_i        (state entering iteration i)
 *  6 g_i  7 s_i  8 l_i  9 z_i 10 q_i 11 u_i 12 y_i 13 n_i 14 v_i  (lines 5-14)  */

/* ------------------------------------------------------------------------- */
/* Preconditioned pipelined BiCGStab: Algorithm 2, step by step,   */
/* with periodic residual replacement (eq:rr P:596-601, placed after line 20  */
/* P:602-603, period policy P:607 / P:764) and the residual-gap history       */
/* (eq:res_gap P:113).                                                        */
/*                                                                            */
/* Readings: A1 (previous-iteration vectors = 0, omega_{-1} = 0), A2 (r^_0 =   */
/* r_0), A7 (stop when ||r_i|| <= tol*||b||), A8 ((r,r) added to reduction 2),*/
/* A9 (breakdown guards), A10-A12 (replacement placement/schedule/sqrt(eps)  */
/* stop, latched), A26 (n_i, v_i are not replaced).                           */
/* sc_trace (optional): per iteration i, ORC_SCW = 9 doubles: alpha_i, beta_i,  */
/* omega_i, rho_i, then the raw dots (q,y), (y,y) of line 12 and (r0,w), (r0,s), */
/* (r0,z) of line 21 (after a replacement: of the replaced vectors).           */
/* ------------------------------------------------------------------------- */
/* Automated residual replacement, flag ORC_AUTO_RR.  The run-time
 * bound f^r_i on ||Delta^r_i|| (eq:DDr_bound P:613-616) is propagated by the
 * triangle inequality over the one-step gap recurrences eq:Dr, eq:Ds
 * (P:276-280), eq:Dw, eq:Dz, with every local error
 * replaced by its bound eq:errbounds1-4:
 *   Dz_i     = |b_i| Dz_{i-1} + ||A|| e^l_i + e^z_i
 *   Ds_i     = Dw_i + |b_i| Ds_{i-1} + |b_i w_{i-1}| Dz_{i-1} + ||A|| e^g_i + e^s_i
 *   Dw_{i+1} = Dw_i + |a_i| Dz_i + ||A|| e^k_{i+1} + e^w_{i+1} + ||A|| e^u_i + e^y_i
 *   f_{i+1}  = f_i + |a_i| Ds_i + |w_i| Dw_i + |w_i a_i| Dz_i
 *              + ||A|| e^x_{i+1} + e^r_{i+1} + |w_i| ||A|| e^u_i + e^q_i + |w_i| e^y_i
 * Initial values: f_0 = ((mu sqrt N + 1)||A|| ||x_0||
 * + ||b||) eps, Dw_0 = mu sqrt N ||A|| ||k_0|| eps, Ds_{-1} = Dz_{-1} = 0 (g, l, z
 * at i = -1 are exact zeros, A1).  After a replacement in iteration i the gaps
 * are those of the explicit recomputation (reading A31): f_{i+1} = ((mu sqrt N
 * + 1)||A|| ||x_{i+1}|| + ||b||) eps, Ds_i = mu sqrt N ||A|| ||g_i|| eps, Dw_{i+1} =
 * mu sqrt N ||A|| ||k_{i+1}|| eps, Dz_i = mu sqrt N ||A|| ||l_i|| eps.
 * Criterion eq:criterion, tau = sqrt(eps): replace in iteration i
 * (after line 20, A10) iff f_{i-1} <= tau ||r_{i-1}|| and f_i > tau ||r_i||
 * (decided at the end of iteration i-1; i >= 1).  eps = 2^-53 (A12); ||A|| =
 * orc_anorm_bound (A29); ||M^-1|| = max |dinv_j|; mu = max nnz per row of A,
 * mu~ = 1 (Jacobi, A25).  Norms are 2-norms sqrt((v,v)) with Dot2 (A6).
 * Every vector whose norm enters is stored by this transcription, so the norms
 * are taken directly from the vectors of the current and previous iteration. */
typedef struct {
  double f, f_prev, Dw, Ds, Dz; /* f_i, f_{i-1}, Dw_i, Ds_{i-1}, Dz_{i-1} */
  double nA, muN, mutN;         /* ||A||, mu sqrt N, mu~ sqrt N ||M^-1|| */
  double eps, tau;
} autorr;

static double nrm2(int64_t n, const double* v) { return sqrt(orc_dot2(n, v, v)); }

int orc_pbicgstab(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
                  const double* b, const double* x0, double tol, int32_t maxit,
                  int32_t rr_period, int32_t flags, double* x, double* rhist,
                  double* gaphist, int32_t* iters_out, int32_t* outcome_out,
                  double* sc_trace, double* vec_trace, double* bound_trace,
                  int32_t* rr_list, int32_t* n_rr) {
  if (n < 0 || maxit < 0 || rr_period < 0) return -2;
  /* the run-time bound needs mu~ and ||M^-1|| (A29); not defined here for ILU(0) */
  if ((flags & ORC_AUTO_RR) && (flags & ORC_ILU0)) return -3;
  Prec P;
  if (prec_make(flags, n, rp, ci, va, &P) != 0) return -1;
  double *r = vec(n), *rh = vec(n), *k = vec(n), *w = vec(n), *m = vec(n), *t = vec(n);
  double *g = vec(n), *s = vec(n), *l = vec(n), *z = vec(n), *nn = vec(n), *v = vec(n);
  double *q = vec(n), *u = vec(n), *y = vec(n), *tmp = vec(n);
  int fgap = (flags & ORC_GAP) && gaphist;
  const double sqrt_eps = sqrt(ldexp(1.0, -53)); /* reading A12: eps = 2^-53 */

  memcpy(x, x0, (size_t)n * sizeof(double));
  /* line 2: r0 := b - A x0; k0 := M^-1 r0; w0 := A k0; m0 := M^-1 w0 */
  orc_spmv(n, rp, ci, va, x, tmp);
  for (int64_t j = 0; j < n; ++j) r[j] = b[j] - tmp[j];
  memcpy(rh, r, (size_t)n * sizeof(double)); /* A2: shadow residual r^ := r0 */
  pprec(&P, r, k);
  orc_spmv(n, rp, ci, va, k, w);
  pprec(&P, w, m);
  /* line 3: t0 := A m0; alpha0 := (r0,r0)/(r0,w0); beta0 := 0 */
  orc_spmv(n, rp, ci, va, m, t);
  double rho = dotf(flags, n, rh, r);
  double alpha = rho / dotf(flags, n, rh, w);
  double beta = 0.0, omega = 0.0; /* A1: omega_{-1} := 0; g,s,l,z,n,v := 0 (calloc) */
  double nb = sqrt(dotf(flags, n, b, b));
  rhist[0] = sqrt(dotf(flags, n, r, r));
  if (fgap) gaphist[0] = res_gap(flags, n, rp, ci, va, b, x, r, tmp);
  double h0 = rhist[0];
  /* automated replacement state */
  const int fauto = (flags & ORC_AUTO_RR) != 0;
  autorr ar;
  memset(&ar, 0, sizeof(ar));
  int rr_next = 0, nrr = 0;
  if (fauto) {
    int64_t mu = 0;
    const double mi = prec_norm_bound(&P); /* ||M^-1|| (A29) */
    for (int64_t j = 0; j < n; ++j)
      if (rp[j + 1] - rp[j] > mu) mu = rp[j + 1] - rp[j];
    ar.eps = ldexp(1.0, -53);
    ar.tau = sqrt(ar.eps);
    ar.nA = orc_anorm_bound(n, rp, ci, va);
    ar.muN = (double)mu * sqrt((double)n);
    ar.mutN = (double)P.b * sqrt((double)n) * mi; /* mu~ = b nonzeros per row of M^-1 */
    ar.f = ((ar.muN + 1.0) * ar.nA * nrm2(n, x) + nb) * ar.eps;
    ar.f_prev = ar.f;
    ar.Dw = ar.muN * ar.nA * nrm2(n, k) * ar.eps;
    ar.Ds = 0.0;
    ar.Dz = 0.0;
    if (bound_trace) {
      bound_trace[0] = ar.f;
      bound_trace[1] = ar.Dw;
      bound_trace[2] = NAN;
      bound_trace[3] = NAN;
    }
  }
  int rr_off = 0; /* A12: replacements stop for good once ||r_i|| < sqrt(eps)||r_0|| */
  if (h0 < sqrt_eps * h0) rr_off = 1;
  int32_t iters = 0, outcome = OUT_MAXIT;
  int done = 0;
  if (rhist[0] <= tol * nb && !(flags & ORC_BENCH)) { outcome = OUT_CONVERGED; done = 1; }
  else if (!isfinite(alpha)) { outcome = OUT_BREAKDOWN; done = 1; }

  for (int32_t i = 0; i < maxit && !done; ++i) {
    if (vec_trace) {
      double* T = vec_trace + (size_t)i * NTRACE * (size_t)n;
      const double* src[6] = {x, r, k, w, m, t};
      for (int a = 0; a < 6; ++a) memcpy(T + (size_t)a * n, src[a], (size_t)n * sizeof(double));
    }
    if (sc_trace) { sc_trace[ORC_SCW * i + 0] = alpha; sc_trace[ORC_SCW * i + 1] = beta; sc_trace[ORC_SCW * i + 3] = rho; }
    /* norms of the previous iteration's g, s, l, z, n, v (zero at i = 0, A1;
     * after a replacement s, l, z are the replaced vectors, n, v are not, A26)
     * and of this iteration's x, k, w, m, t, for the bound f^r */
    double nGp = 0, nSp = 0, nLp = 0, nZp = 0, nNp = 0, nVp = 0;
    double nX = 0, nK = 0, nW = 0, nM = 0, nT = 0;
    const double om_prev = omega;
    if (fauto) {
      nGp = nrm2(n, g); nSp = nrm2(n, s); nLp = nrm2(n, l); nZp = nrm2(n, z);
      nNp = nrm2(n, nn); nVp = nrm2(n, v);
      nX = nrm2(n, x); nK = nrm2(n, k); nW = nrm2(n, w); nM = nrm2(n, m); nT = nrm2(n, t);
    }
    for (int64_t j = 0; j < n; ++j) {
      /* lines 5-8, n_{i-1} and v_{i-1} as stored (A26) */
      g[j] = k[j] + beta * (g[j] - omega * l[j]);
      s[j] = w[j] + beta * (s[j] - omega * z[j]);
      l[j] = m[j] + beta * (l[j] - omega * nn[j]);
      z[j] = t[j] + beta * (z[j] - omega * v[j]);
    }
    for (int64_t j = 0; j < n; ++j) {
      /* lines 9-11 */
      q[j] = r[j] - alpha * s[j];
      u[j] = k[j] - alpha * l[j];
      y[j] = w[j] - alpha * z[j];
    }
    /* line 12: reduction (q,y), (y,y) */
    double qy = dotf(flags, n, q, y);
    double yy = dotf(flags, n, y, y);
    /* lines 13-14: n := M^-1 z; v := A n */
    pprec(&P, z, nn);
    orc_spmv(n, rp, ci, va, nn, v);
    if (vec_trace) {
      double* T = vec_trace + (size_t)i * NTRACE * (size_t)n;
      const double* src[9] = {g, s, l, z, q, u, y, nn, v};
      for (int a = 0; a < 9; ++a)
        memcpy(T + (size_t)(6 + a) * n, src[a], (size_t)n * sizeof(double));
    }
    /* line 16: omega := (q,y)/(y,y); A9: (y,y) = 0 => omega := 0 */
    omega = (yy == 0.0) ? 0.0 : qy / yy;
    if (sc_trace) {
      sc_trace[ORC_SCW * i + 2] = omega;
      sc_trace[ORC_SCW * i + 4] = qy;
      sc_trace[ORC_SCW * i + 5] = yy;
    }
    if (!isfinite(omega)) { outcome = OUT_BREAKDOWN; iters = i; done = 1; break; }
    /* bound recursion of iteration i, before x, r, k, w move on */
    double nG = 0, nS = 0, nL = 0, nZ = 0, nQ = 0, nU = 0, nY = 0, nN = 0, nV = 0;
    double Dz_i = 0, Ds_i = 0, Dw_1 = 0, f_1 = 0;
    if (fauto) {
      nG = nrm2(n, g); nS = nrm2(n, s); nL = nrm2(n, l); nZ = nrm2(n, z);
      nQ = nrm2(n, q); nU = nrm2(n, u); nY = nrm2(n, y); nN = nrm2(n, nn); nV = nrm2(n, v);
      const double R = rhist[i];
      const double ab = fabs(beta), abw = fabs(beta * om_prev);
      const double aa = fabs(alpha), aw = fabs(omega), awa = fabs(omega * alpha);
      const double nA = ar.nA, muN = ar.muN, mutN = ar.mutN, e = ar.eps;
      /* eq:errbounds1-4 without the common factor eps */
      const double eg = nK + 3.0 * ab * nGp + 4.0 * abw * nLp;
      const double es = nW + 3.0 * ab * nSp + 4.0 * abw * nZp;
      const double el = nM + mutN * nW + 3.0 * ab * nLp + 4.0 * abw * nNp + mutN * abw * nZp;
      const double ez = nT + muN * nA * nM + mutN * nA * nW + 3.0 * ab * nZp + 4.0 * abw * nVp +
                        muN * nA * abw * nNp + mutN * nA * abw * nZp;
      const double eq = R + 2.0 * aa * nS;
      const double eu = nK + 2.0 * aa * nL;
      const double ey = nW + 2.0 * aa * nZ;
      const double ex = 2.0 * nX + 3.0 * aa * nG + 2.0 * aw * nU;
      const double er = nQ + 2.0 * aw * nY;
      const double ek = nU + 3.0 * aw * nM + mutN * aw * nW + 4.0 * awa * nN + mutN * awa * nZ;
      const double ew = nY + 3.0 * aw * nT + muN * nA * aw * nM + mutN * nA * aw * nW +
                        4.0 * awa * nV + muN * nA * awa * nN + mutN * nA * awa * nZ;
      /* eq:Dz, eq:Ds, eq:Dw, eq:Dr by the triangle inequality */
      Dz_i = ab * ar.Dz + nA * el * e + ez * e;
      Ds_i = ar.Dw + ab * ar.Ds + abw * ar.Dz + nA * eg * e + es * e;
      Dw_1 = ar.Dw + aa * Dz_i + nA * ek * e + ew * e + nA * eu * e + ey * e;
      f_1 = ar.f + aa * Ds_i + aw * ar.Dw + awa * Dz_i + nA * ex * e + er * e +
            aw * nA * eu * e + eq * e + aw * ey * e;
    }
    /* lines 17-20 */
    for (int64_t j = 0; j < n; ++j) {
      x[j] = (x[j] + alpha * g[j]) + omega * u[j];
      r[j] = q[j] - omega * y[j];
      k[j] = u[j] - omega * (m[j] - alpha * nn[j]);
      w[j] = y[j] - omega * (t[j] - alpha * v[j]);
    }
    /* residual replacement after line 20, eq:rr:
     * r := b - A x; k := M^-1 r; w := A k; s := A g; l := M^-1 s; z := A l.
     * Schedule (A11): loop index i replaces when (i+1) mod P_rr == 0. */
    const int fire = fauto ? rr_next
                           : (rr_period > 0 && (i + 1) % rr_period == 0 && !rr_off);
    if (fire) {
      orc_spmv(n, rp, ci, va, x, tmp);
      for (int64_t j = 0; j < n; ++j) r[j] = b[j] - tmp[j];
      pprec(&P, r, k);
      orc_spmv(n, rp, ci, va, k, w);
      orc_spmv(n, rp, ci, va, g, s);
      pprec(&P, s, l);
      orc_spmv(n, rp, ci, va, l, z);
      if (fauto) {
        /* gaps of the explicit recomputation (reading A31) */
        f_1 = ((ar.muN + 1.0) * ar.nA * nrm2(n, x) + nb) * ar.eps;
        Ds_i = ar.muN * ar.nA * nG * ar.eps;
        Dw_1 = ar.muN * ar.nA * nrm2(n, k) * ar.eps;
        Dz_i = ar.muN * ar.nA * nrm2(n, l) * ar.eps;
      }
      if (rr_list) rr_list[nrr] = i; /* record (periodic or automated) */
      nrr++;
    }
    /* line 21: reduction (r0,r), (r0,w), (r0,s), (r0,z); + (r,r) (A8) */
    double rho1 = dotf(flags, n, rh, r);
    double dw = dotf(flags, n, rh, w);
    double ds = dotf(flags, n, rh, s);
    double dz = dotf(flags, n, rh, z);
    rhist[i + 1] = sqrt(dotf(flags, n, r, r));
    if (sc_trace) {
      sc_trace[ORC_SCW * i + 6] = dw;
      sc_trace[ORC_SCW * i + 7] = ds;
      sc_trace[ORC_SCW * i + 8] = dz;
    }
    /* lines 22-23: m := M^-1 w; t := A m */
    pprec(&P, w, m);
    orc_spmv(n, rp, ci, va, m, t);
    if (fgap) gaphist[i + 1] = res_gap(flags, n, rp, ci, va, b, x, r, tmp);
    iters = i + 1;
    if (fauto) {
      /* eq:criterion for iteration i+1 */
      rr_next = (ar.f <= ar.tau * rhist[i]) && (f_1 > ar.tau * rhist[i + 1]);
      ar.f_prev = ar.f;
      ar.f = f_1;
      ar.Dw = Dw_1;
      ar.Ds = Ds_i;
      ar.Dz = Dz_i;
      if (bound_trace) {
        bound_trace[4 * (i + 1) + 0] = f_1;
        bound_trace[4 * (i + 1) + 1] = Dw_1;
        bound_trace[4 * i + 2] = Ds_i;
        bound_trace[4 * i + 3] = Dz_i;
        bound_trace[4 * (i + 1) + 2] = NAN;
        bound_trace[4 * (i + 1) + 3] = NAN;
      }
    }
    if (rhist[i + 1] < sqrt_eps * h0) rr_off = 1;
    if (rhist[i + 1] <= tol * nb && !(flags & ORC_BENCH)) { outcome = OUT_CONVERGED; done = 1; break; }
    /* lines 25-26 */
    double beta1 = ((alpha / omega) * rho1) / rho;
    double den = (dw + beta1 * ds) - (beta1 * omega) * dz;
    double alpha1 = rho1 / den;
    beta = beta1;
    alpha = alpha1;
    rho = rho1;
    if (!isfinite(beta) || !isfinite(alpha) || den == 0.0 || rho1 == 0.0) {
      outcome = OUT_BREAKDOWN; done = 1; break;
    }
  }
  if (vec_trace && !done) {
    double* T = vec_trace + (size_t)maxit * NTRACE * (size_t)n;
    const double* src[6] = {x, r, k, w, m, t};
    for (int a = 0; a < 6; ++a) memcpy(T + (size_t)a * n, src[a], (size_t)n * sizeof(double));
  }
  *iters_out = iters;
  *outcome_out = outcome;
  if (n_rr) *n_rr = nrr;
  prec_free(&P); free(r); free(rh); free(k); free(w); free(m); free(t); free(g); free(s);
  free(l); free(z); free(nn); free(v); free(q); free(u); free(y); free(tmp);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Classic preconditioned BiCGStab: Algorithm 1, step by step.       */
/* Same conventions; rhist[i] = ||r_i||, stop when ||r_i|| <= tol ||b|| (A7). */
/* sc_trace: alpha_i, beta_i, omega_i, rho_i per iteration.                   */
/* ------------------------------------------------------------------------- */
int orc_bicgstab(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
                 const double* b, const double* x0, double tol, int32_t maxit, int32_t flags,
                 double* x, double* rhist, double* gaphist, int32_t* iters_out,
                 int32_t* outcome_out, double* sc_trace) {
  if (n < 0 || maxit < 0) return -2;
  Prec P;
  if (prec_make(flags, n, rp, ci, va, &P) != 0) return -1;
  double *r = vec(n), *rh = vec(n), *p = vec(n), *g = vec(n), *s = vec(n), *q = vec(n);
  double *u = vec(n), *y = vec(n), *tmp = vec(n);
  int fgap = (flags & ORC_GAP) && gaphist;
  memcpy(x, x0, (size_t)n * sizeof(double));
  /* line 2: r0 := b - A x0; p0 := r0 */
  orc_spmv(n, rp, ci, va, x, tmp);
  for (int64_t j = 0; j < n; ++j) r[j] = b[j] - tmp[j];
  memcpy(rh, r, (size_t)n * sizeof(double));
  memcpy(p, r, (size_t)n * sizeof(double));
  double rho = dotf(flags, n, rh, r);
  double nb = sqrt(dotf(flags, n, b, b));
  rhist[0] = sqrt(dotf(flags, n, r, r));
  if (fgap) gaphist[0] = res_gap(flags, n, rp, ci, va, b, x, r, tmp);
  int32_t iters = 0, outcome = OUT_MAXIT;
  int done = 0;
  if (rhist[0] <= tol * nb && !(flags & ORC_BENCH)) { outcome = OUT_CONVERGED; done = 1; }
  for (int32_t i = 0; i < maxit && !done; ++i) {
    pprec(&P, p, g);                   /* line 4 */
    orc_spmv(n, rp, ci, va, g, s);         /* line 5 */
    double rs = dotf(flags, n, rh, s);     /* line 6 */
    double alpha = rho / rs;               /* line 7 */
    for (int64_t j = 0; j < n; ++j) q[j] = r[j] - alpha * s[j]; /* line 8 */
    pprec(&P, q, u);                   /* line 9 */
    orc_spmv(n, rp, ci, va, u, y);         /* line 10 */
    double qy = dotf(flags, n, q, y);      /* line 11 */
    double yy = dotf(flags, n, y, y);
    double omega = (yy == 0.0) ? 0.0 : qy / yy; /* line 12, guard A9 */
    if (sc_trace) { sc_trace[4 * i] = alpha; sc_trace[4 * i + 2] = omega; sc_trace[4 * i + 3] = rho; }
    if (!isfinite(alpha) || !isfinite(omega)) { outcome = OUT_BREAKDOWN; iters = i; done = 1; break; }
    for (int64_t j = 0; j < n; ++j) {
      x[j] = (x[j] + alpha * g[j]) + omega * u[j]; /* line 13, eq:auxrec0 */
      r[j] = q[j] - omega * y[j];                   /* line 14 */
    }
    double rho1 = dotf(flags, n, rh, r);   /* line 15 */
    rhist[i + 1] = sqrt(dotf(flags, n, r, r));
    if (fgap) gaphist[i + 1] = res_gap(flags, n, rp, ci, va, b, x, r, tmp);
    iters = i + 1;
    if (rhist[i + 1] <= tol * nb && !(flags & ORC_BENCH)) { outcome = OUT_CONVERGED; done = 1; break; }
    double beta = ((alpha / omega) * rho1) / rho; /* line 16 */
    if (sc_trace) sc_trace[4 * i + 1] = beta;
    for (int64_t j = 0; j < n; ++j) p[j] = r[j] + beta * (p[j] - omega * s[j]); /* line 17 */
    rho = rho1;
    if (!isfinite(beta) || rho1 == 0.0) { outcome = OUT_BREAKDOWN; done = 1; break; }
  }
  *iters_out = iters;
  *outcome_out = outcome;
  prec_free(&P); free(r); free(rh); free(p); free(g); free(s); free(q); free(u); free(y); free(tmp);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Preconditioned CG (Hestenes-Stiefel form) -- comparison solver for cfg1.   */
/* Not an algorithm printed in the paper (cited at P:30); standard PCG.       */
/* ------------------------------------------------------------------------- */
int orc_pcg(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
            const double* b, const double* x0, double tol, int32_t maxit, int32_t flags,
            double* x, double* rhist, double* gaphist, int32_t* iters_out,
            int32_t* outcome_out) {
  Prec P;
  if (prec_make(flags, n, rp, ci, va, &P) != 0) return -1;
  double *r = vec(n), *u = vec(n), *p = vec(n), *s = vec(n), *tmp = vec(n);
  int fgap = (flags & ORC_GAP) && gaphist;
  memcpy(x, x0, (size_t)n * sizeof(double));
  orc_spmv(n, rp, ci, va, x, tmp);
  for (int64_t j = 0; j < n; ++j) r[j] = b[j] - tmp[j];
  pprec(&P, r, u);
  memcpy(p, u, (size_t)n * sizeof(double));
  double gam = dotf(flags, n, r, u);
  double nb = sqrt(dotf(flags, n, b, b));
  rhist[0] = sqrt(dotf(flags, n, r, r));
  if (fgap) gaphist[0] = res_gap(flags, n, rp, ci, va, b, x, r, tmp);
  int32_t iters = 0, outcome = OUT_MAXIT;
  int done = (rhist[0] <= tol * nb && !(flags & ORC_BENCH));
  if (done) outcome = OUT_CONVERGED;
  for (int32_t i = 0; i < maxit && !done; ++i) {
    orc_spmv(n, rp, ci, va, p, s);
    double alpha = gam / dotf(flags, n, p, s);
    for (int64_t j = 0; j < n; ++j) { x[j] = x[j] + alpha * p[j]; r[j] = r[j] - alpha * s[j]; }
    pprec(&P, r, u);
    double gam1 = dotf(flags, n, r, u);
    rhist[i + 1] = sqrt(dotf(flags, n, r, r));
    if (fgap) gaphist[i + 1] = res_gap(flags, n, rp, ci, va, b, x, r, tmp);
    iters = i + 1;
    if (rhist[i + 1] <= tol * nb && !(flags & ORC_BENCH)) { outcome = OUT_CONVERGED; break; }
    double beta = gam1 / gam;
    for (int64_t j = 0; j < n; ++j) p[j] = u[j] + beta * p[j];
    gam = gam1;
    if (!isfinite(alpha) || !isfinite(beta)) { outcome = OUT_BREAKDOWN; break; }
  }
  *iters_out = iters;
  *outcome_out = outcome;
  prec_free(&P); free(r); free(u); free(p); free(s); free(tmp);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Preconditioned pipelined CG (Ghysels-Vanroose form).  The paper compares   */
/* against p-CG (Figs. 1-2) but prints no pseudocode (reading      */
/* A19); this reconstruction is pinned only by exact rational equivalence     */
/* with PCG.  One reduction {(r,u),(w,u)} per iteration, overlapped with      */
/* m := M^-1 w, n := A m.                                                     */
/* ------------------------------------------------------------------------- */
int orc_pipecg(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
               const double* b, const double* x0, double tol, int32_t maxit, int32_t flags,
               double* x, double* rhist, double* gaphist, int32_t* iters_out,
               int32_t* outcome_out) {
  Prec P;
  if (prec_make(flags, n, rp, ci, va, &P) != 0) return -1;
  double *r = vec(n), *u = vec(n), *w = vec(n), *m = vec(n), *nn = vec(n);
  double *z = vec(n), *q = vec(n), *s = vec(n), *p = vec(n), *tmp = vec(n);
  int fgap = (flags & ORC_GAP) && gaphist;
  memcpy(x, x0, (size_t)n * sizeof(double));
  orc_spmv(n, rp, ci, va, x, tmp);
  for (int64_t j = 0; j < n; ++j) r[j] = b[j] - tmp[j];
  pprec(&P, r, u);
  orc_spmv(n, rp, ci, va, u, w);
  double nb = sqrt(dotf(flags, n, b, b));
  rhist[0] = sqrt(dotf(flags, n, r, r));
  if (fgap) gaphist[0] = res_gap(flags, n, rp, ci, va, b, x, r, tmp);
  int32_t iters = 0, outcome = OUT_MAXIT;
  int done = (rhist[0] <= tol * nb && !(flags & ORC_BENCH));
  if (done) outcome = OUT_CONVERGED;
  double gam_old = 0.0, alpha_old = 0.0;
  for (int32_t i = 0; i < maxit && !done; ++i) {
    double gam = dotf(flags, n, r, u);
    double del = dotf(flags, n, w, u);
    pprec(&P, w, m);
    orc_spmv(n, rp, ci, va, m, nn);
    double beta, alpha;
    if (i == 0) { beta = 0.0; alpha = gam / del; }
    else { beta = gam / gam_old; alpha = gam / (del - (beta * gam) / alpha_old); }
    if (!isfinite(alpha) || !isfinite(beta)) { outcome = OUT_BREAKDOWN; iters = i; break; }
    for (int64_t j = 0; j < n; ++j) {
      z[j] = nn[j] + beta * z[j];
      q[j] = m[j] + beta * q[j];
      s[j] = w[j] + beta * s[j];
      p[j] = u[j] + beta * p[j];
      x[j] = x[j] + alpha * p[j];
      r[j] = r[j] - alpha * s[j];
      u[j] = u[j] - alpha * q[j];
      w[j] = w[j] - alpha * z[j];
    }
    gam_old = gam;
    alpha_old = alpha;
    rhist[i + 1] = sqrt(dotf(flags, n, r, r));
    if (fgap) gaphist[i + 1] = res_gap(flags, n, rp, ci, va, b, x, r, tmp);
    iters = i + 1;
    if (rhist[i + 1] <= tol * nb && !(flags & ORC_BENCH)) { outcome = OUT_CONVERGED; break; }
  }
  *iters_out = iters;
  *outcome_out = outcome;
  prec_free(&P); free(r); free(u); free(w); free(m); free(nn); free(z); free(q); free(s); free(p);
  free(tmp);
  return 0;
}
