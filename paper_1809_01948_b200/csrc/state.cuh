// state.cuh -- device-resident solver state shared by all kernels of a handle.
//
// The scalars of Alg. 2 (alpha_i, beta_i, omega_i, rho_i = (r0, r_i); P:169,
// P:182), the stopping / replacement control and the
// iteration counter live on the device; the host never synchronises inside the
// iteration.  Each kernel reads them in its prologue.  A new scalar is formed
//   * on one rank: by the last CTA of the kernel that produced the dots (after
//     every other CTA of that kernel has finished reading the old value);
//   * on P ranks: each rank's last CTA publishes its Dot2 partial pairs into its
//     row of red_send; the rows are exchanged (NCCL all-reduce of a zero-padded
//     [P][8] buffer = exact all-gather, or the loopback transport); a one-CTA
//     finalize kernel combines the rows in rank order and forms the scalar.
#pragma once
#include <cstdint>

#include "dd.cuh"

#define OUT_CONVERGED 0
#define OUT_MAXIT 1
#define OUT_BREAKDOWN 2
#define RED_K 8  // dot slots per rank in the reduction buffers

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
  int32_t bench, rr_period;
  int32_t method;                  // 0 p-BiCGStab (Alg. 2), 1 BiCGStab (Alg. 1), 2 p-CG
  double g_old, a_old;             // p-CG: gamma_{i-1}, alpha_{i-1}
  int32_t nranks, rank;
  Dd* red_send;                    // [nranks][RED_K]: only row `rank` is ever written
  Dd* red_recv;                    // [nranks][RED_K]: all rows after the exchange
  unsigned int counter[16];        // last-CTA tickets, one per kernel kind
};

enum TicketSlot { T_INIT1 = 0, T_INIT2, T_SWEEPA, T_SWEEPC, T_RR2, T_GAP, T_APPLY, T_MISC,
                  T_CL1, T_CL2, T_CL3, T_PC, T_PCI1, T_PCI2 };

// which scalar-forming step a reduction feeds
enum FinKind { F_INIT1 = 0, F_INIT2, F_SWEEPA, F_SWEEPC, F_RR2, F_GAP,
               F_CL1, F_CL2, F_CL3, F_PINIT2, F_PC };

struct Hist {
  double* rnorm;  // [maxit+1]
  double* gap;    // [maxit+1]
};

// Line 21-26 bookkeeping once the five dots of reduction #2 are
// known: history, sqrt(eps) latch (A12), stop test (A7), beta_{i+1},
// alpha_{i+1} (left to right as printed, A4), breakdown (A9).
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

// The scalar-forming steps, given the combined dot totals (one thread).
template <int F>
__device__ __forceinline__ void fin_step(Scal* sc, Hist h, const Dd* tot) {
  if (F == F_INIT1) {
    sc->tmp0 = dd_round(tot[0]);  // (r0, r0) = (r^0, r0) = rho_0
    sc->tmp1 = dd_round(tot[1]);  // (b, b)
    if (sc->method != 0) {
      // Alg. 1 lines 2-3 / p-CG init: rho_0 := (r^0, r0) = (r0, r0) (r^0 := r0,
      // A2); ||r0||, ||b||, stop test (A7); beta, omega := 0 (line 17 with p_{-1} = 0)
      sc->rho = sc->tmp0;
      sc->alpha = 0.0;
      sc->beta = 0.0;
      sc->omega = 0.0;
      sc->h0 = sqrt(sc->tmp0);
      sc->nb = sqrt(sc->tmp1);
      sc->tol_abs = sc->tol * sc->nb;
      h.rnorm[0] = sc->h0;
      if (sc->h0 <= sc->tol_abs && !sc->bench) {
        sc->done = 1;
        sc->outcome = OUT_CONVERGED;
      }
    }
  } else if (F == F_CL1) {
    // Alg. 1 lines 6-7: alpha_i := rho_i / (r^0, s_i)
    sc->alpha = sc->rho / dd_round(tot[0]);
  } else if (F == F_CL2) {
    // Alg. 1 lines 11-12: omega_i := (q_i, y_i) / (y_i, y_i), guard A9
    const double qy = dd_round(tot[0]), yy = dd_round(tot[1]);
    const double om = (yy == 0.0) ? 0.0 : qy / yy;
    sc->omega = om;
    if (!isfinite(sc->alpha) || !isfinite(om)) {
      sc->done = 1;
      sc->outcome = OUT_BREAKDOWN;
      sc->iters = sc->iter;
    }
  } else if (F == F_CL3) {
    // Alg. 1 lines 15-16: rho_{i+1} := (r^0, r_{i+1}); ||r_{i+1}||; stop
    // test (A7); beta_i := (alpha_i / omega_i) (rho_{i+1} / rho_i), left to right (A4)
    const int i = sc->iter;
    const double rho1 = dd_round(tot[0]);
    const double hn = sqrt(dd_round(tot[1]));
    h.rnorm[i + 1] = hn;
    sc->iters = i + 1;
    sc->iter = i + 1;
    if (hn <= sc->tol_abs && !sc->bench) {
      sc->done = 1;
      sc->outcome = OUT_CONVERGED;
      return;
    }
    const double beta = ((sc->alpha / sc->omega) * rho1) / sc->rho;
    sc->beta = beta;
    sc->rho = rho1;
    if (!isfinite(beta) || rho1 == 0.0) {
      sc->done = 1;
      sc->outcome = OUT_BREAKDOWN;
    }
  } else if (F == F_PINIT2) {
    // p-CG iteration 0 scalars (reading A19): gamma_0 := (r0, u0), delta_0 := (w0, u0),
    // beta_0 := 0, alpha_0 := gamma_0 / delta_0
    if (sc->done) return;  // converged at i = 0
    const double gam = dd_round(tot[0]), del = dd_round(tot[1]);
    const double alpha = gam / del;
    sc->alpha = alpha;
    sc->beta = 0.0;
    sc->g_old = gam;
    sc->a_old = alpha;
    if (!isfinite(alpha)) {
      sc->done = 1;
      sc->outcome = OUT_BREAKDOWN;
      sc->iters = 0;
    }
  } else if (F == F_PC) {
    // p-CG end of iteration i: ||r_{i+1}||, stop test, then the scalars of iteration
    // i+1 from its single reduction {(r,u), (w,u)}: beta := gamma / gamma_old;
    // alpha := gamma / (delta - (beta gamma) / alpha_old)   (reading A19)
    const int i = sc->iter;
    const double gam = dd_round(tot[0]), del = dd_round(tot[1]);
    const double hn = sqrt(dd_round(tot[2]));
    h.rnorm[i + 1] = hn;
    sc->iters = i + 1;
    sc->iter = i + 1;
    if (hn <= sc->tol_abs && !sc->bench) {
      sc->done = 1;
      sc->outcome = OUT_CONVERGED;
      return;
    }
    const double beta = gam / sc->g_old;
    const double alpha = gam / (del - (beta * gam) / sc->a_old);
    sc->alpha = alpha;
    sc->beta = beta;
    sc->g_old = gam;
    sc->a_old = alpha;
    if (!isfinite(alpha) || !isfinite(beta)) {
      sc->done = 1;
      sc->outcome = OUT_BREAKDOWN;
    }
  } else if (F == F_INIT2) {
    // line 3: alpha0 := (r0,r0)/(r0,w0); beta0 := 0; omega_{-1} := 0 (A1)
    const double rho = sc->tmp0;
    sc->rho = rho;
    sc->alpha = rho / dd_round(tot[0]);
    sc->beta = 0.0;
    sc->omega = 0.0;
    sc->h0 = sqrt(rho);
    sc->nb = sqrt(sc->tmp1);
    sc->tol_abs = sc->tol * sc->nb;
    h.rnorm[0] = sc->h0;
    if (sc->h0 <= sc->tol_abs && !sc->bench) {
      sc->done = 1;
      sc->outcome = OUT_CONVERGED;
    } else if (!isfinite(sc->alpha)) {
      sc->done = 1;
      sc->outcome = OUT_BREAKDOWN;
    }
  } else if (F == F_SWEEPA) {
    // line 16: omega := (q,y)/(y,y), guard A9
    const double qy = dd_round(tot[0]), yy = dd_round(tot[1]);
    const double omn = (yy == 0.0) ? 0.0 : qy / yy;
    sc->omega = omn;
    sc->use_rr = 0;
    if (!isfinite(omn)) {
      sc->done = 1;
      sc->outcome = OUT_BREAKDOWN;
      sc->iters = sc->iter;
    }
  } else if (F == F_SWEEPC) {
    if (rr_scheduled(sc)) {
      sc->rr_fire = 1;  // the line-21 dots are recomputed after the replacement
    } else {
      finalize_iteration(sc, h, dd_round(tot[0]), dd_round(tot[1]), dd_round(tot[2]),
                         dd_round(tot[3]), dd_round(tot[4]));
    }
  } else if (F == F_RR2) {
    finalize_iteration(sc, h, dd_round(tot[0]), dd_round(tot[1]), dd_round(tot[2]),
                       dd_round(tot[3]), dd_round(tot[4]));
    sc->use_rr = 1;
  } else if (F == F_GAP) {
    h.gap[sc->iter] = sqrt(dd_round(tot[0]));
    sc->gap_iter = sc->iter;
  }
}

// Tail of every reducing kernel (thread 0 of the last CTA): finish on one rank,
// publish the rank's partial pairs on several.
template <int F, int K>
__device__ __forceinline__ void publish(Scal* sc, Hist h, const Dd (&tot)[K]) {
  if (sc->nranks > 1) {
    Dd* row = sc->red_send + (size_t)sc->rank * RED_K;
#pragma unroll
    for (int k = 0; k < K; ++k) row[k] = tot[k];
  } else {
    fin_step<F>(sc, h, tot);
  }
}

// One-CTA finalize after the exchange: combine the rank rows in rank order.
template <int F, int K>
__global__ void k_fin(Scal* __restrict__ sc, Hist h) {
  if (threadIdx.x != 0) return;
  if (F == F_GAP) {
    if (sc->gap_iter >= sc->iter) return;
  } else if (F == F_RR2) {
    if (sc->done || !sc->rr_fire) return;
  } else if (F != F_INIT1 && F != F_INIT2) {
    if (sc->done) return;
  }
  Dd tot[K];
#pragma unroll
  for (int k = 0; k < K; ++k) tot[k] = dd_zero();
  for (int r = 0; r < sc->nranks; ++r) {
#pragma unroll
    for (int k = 0; k < K; ++k) tot[k] = dd_add(tot[k], sc->red_recv[(size_t)r * RED_K + k]);
  }
  fin_step<F>(sc, h, tot);
}
