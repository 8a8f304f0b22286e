// state.cuh -- device-resident solver state shared by all kernels of a handle.
//
// The scalars of Alg. 2 (alpha_i, beta_i, omega_i, rho_i = (r0, r_i); P:169,
// P:182), the stopping / replacement control and the
// iteration counter live on the device; the host never synchronises inside the
// iteration.  Each kernel reads them in its prologue; the last CTA of the
// kernel that produces a new scalar writes it (after every other CTA of that
// kernel has finished, so no CTA can still be reading the old value).
#pragma once
#include <cstdint>

#define OUT_CONVERGED 0
#define OUT_MAXIT 1
#define OUT_BREAKDOWN 2

struct Scal {
  double alpha, beta, omega, rho;  // alpha_i, beta_i, omega (latest), (r0, r_i)
  double h0, nb, tol, tol_abs;     // ||r_0||, ||b||, tol, fl(tol*||b||)
  double sqrt_eps;                 // sqrt(2^-53) (reading A12)
  double tmp0, tmp1;               // init scratch
  int32_t iter;                    // index i of the iteration being executed
  int32_t done, outcome, iters;
  int32_t rr_fire;                 // replacement decided for this iteration
  int32_t use_rr;                  // previous iteration replaced z (reading A26)
  int32_t rr_off;                  // ||r_i|| < sqrt(eps)||r_0|| seen: no more replacements
  int32_t gap_iter;                // last iteration whose gap was written
  int32_t bench, rr_period, pad0, pad1;
  unsigned int counter[8];         // last-CTA tickets, one per kernel kind
};

enum TicketSlot { T_INIT1 = 0, T_INIT2, T_SWEEPA, T_SWEEPC, T_RR2, T_GAP, T_APPLY, T_MISC };

struct Hist {
  double* rnorm;  // [maxit+1]
  double* gap;    // [maxit+1]
};

// Line 21-26 bookkeeping done by one thread once the five dots of
// reduction #2 are known: history, sqrt(eps) latch (A12), stop test (A7),
// beta_{i+1}, alpha_{i+1} (left to right as printed, A4), breakdown (A9).
__device__ __forceinline__ void finalize_iteration(Scal* s, Hist h, double rho1, double dw,
                                                   double ds, double dz, double rr) {
  const int i = s->iter;
  const double hn = sqrt(rr);
  h.rnorm[i + 1] = hn;
  s->iters = i + 1;
  s->iter = i + 1;
  if (hn < s->sqrt_eps * s->h0) s->rr_off = 1;
  s->rr_fire = 0;
  if (hn <= s->tol_abs && !s->bench) {
    s->done = 1;
    s->outcome = OUT_CONVERGED;
    return;
  }
  const double alpha = s->alpha, omega = s->omega, rho = s->rho;
  const double beta1 = ((alpha / omega) * rho1) / rho;
  const double den = (dw + beta1 * ds) - (beta1 * omega) * dz;
  const double alpha1 = rho1 / den;
  s->beta = beta1;
  s->alpha = alpha1;
  s->rho = rho1;
  if (!isfinite(beta1) || !isfinite(alpha1) || den == 0.0 || rho1 == 0.0) {
    s->done = 1;
    s->outcome = OUT_BREAKDOWN;
  }
}

// Replacement decision for iteration i (A11: (i+1) mod P == 0; A12 latch).
__device__ __forceinline__ bool rr_scheduled(const Scal* s) {
  return s->rr_period > 0 && ((s->iter + 1) % s->rr_period) == 0 && !s->rr_off;
}
