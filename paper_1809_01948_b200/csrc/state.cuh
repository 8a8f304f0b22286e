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
#define RED_K 16  // dot slots per rank in the reduction buffers
#define P2P_MAXR 8
#define SC_W 9      // doubles per iteration of the scalar trace (Hist.sc)  // ranks of the peer-memory transport (one NVSwitch domain of B200s)

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
  int32_t spd_par;                 // split stencil schedule: buffer parity of the w SpMV_D reads
  double g_old, a_old;             // p-CG: gamma_{i-1}, alpha_{i-1}
  // automated residual replacement (oracle.c orc_pbicgstab, ORC_AUTO_RR)
  int32_t auto_rr;                 // option rr_auto
  int32_t rr_next;                 // eq:criterion decided for the next iteration
  int32_t n_rr;                    // replacements so far (Hist.rrl)
  double ar_nA, ar_muN, ar_mutN;   // ||A|| bound (A29), mu sqrt N, mu~ sqrt N ||M^-1||
  double ar_eps, ar_tau;           // 2^-53, sqrt(eps)
  double ar_f, ar_Dw, ar_Ds, ar_Dz; // f_i, Dw_i, Ds_{i-1}, Dz_{i-1}
  double ar_omp;                   // omega_{i-1} (0 at i = 0, A1)
  double nA_[10];                  // sweep A norms: k, w, m, t, g, s, l, z, q, y (iteration i)
  double nC_[4];                   // sweep C norms: x_i, u_i, n_i, v_i
  double nR_[4];                   // rr1 norms: x_{i+1}, k_{i+1}, s_i, l_i (replaced)
  double nP_[6];                   // previous iteration: g, s, l, z, n, v
  double nX0, nK0;                 // init: ||x_0||, ||k_0||
  int32_t nranks, rank;
  int32_t dist;                    // rank-row exchange + finalize kernel (nranks > 1, or an
                                   // NCCL communicator of one rank)
  Dd* red_send;                    // [nranks][RED_K]: only row `rank` is ever written
  Dd* red_recv;                    // [nranks][RED_K]: all rows after the exchange
  // peer-memory transport (option "transport" 1): the last CTA of a reducing kernel
  // stores its rank's pairs into row `rank` of EVERY rank's p2p_recv[q] (NVLink
  // stores; double-buffered by epoch parity) and raises p2p_flag[q][rank] = epoch;
  // the finalize kernel waits for all P flags -- no collective launch at all
  int32_t p2p;
  unsigned long long* p2p_epoch;   // own counter (device, persists across solves)
  Dd* p2p_recv[P2P_MAXR];          // rank q's receive buffer [2][nranks][RED_K]
  unsigned long long* p2p_flag[P2P_MAXR];  // rank q's flags [nranks]
  unsigned int counter[16];        // last-CTA tickets, one per kernel kind
};

enum TicketSlot { T_INIT1 = 0, T_INIT2, T_SWEEPA, T_SWEEPC, T_RR2, T_GAP, T_APPLY, T_MISC,
                  T_CL1, T_CL2, T_CL3, T_PC, T_PCI1, T_PCI2, T_RR1 };

// which scalar-forming step a reduction feeds
enum FinKind { F_INIT1 = 0, F_INIT2, F_SWEEPA, F_SWEEPC, F_RR2, F_GAP,
               F_CL1, F_CL2, F_CL3, F_PINIT2, F_PC, F_RR1 };

struct Hist {
  double* rnorm;  // [maxit+1]
  double* gap;    // [maxit+1]
  double* fr;     // [maxit+1] run-time gap bound f^r_i (automated replacement)
  int32_t* rrl;   // [maxit] iterations i that replaced r_{i+1}
  double* sc;     // [maxit][SC_W] p-BiCGStab scalars of iteration i: alpha_i, beta_i,
                  // omega_i, rho_i, (q,y)_i, (y,y)_i, (r0,w), (r0,s), (r0,z) of line 21
                  // (the oracle's sc_trace layout; parity diagnostics)
};

// The scalar state the end-of-iteration bookkeeping reads (fin_step F_SWEEPA /
// F_SWEEPC / F_RR2), loaded in one batch of independent loads.  Every field is
// written only by the scalar-forming step of an earlier kernel, so a copy taken
// after a kernel's PDL wait is the state its own publish starts from; the tile
// sweeps take it in their prologue (off the critical path) and the last CTA's
// bookkeeping then issues only stores -- no chain of dependent global-memory
// round trips behind the grid reduction (scripts/timeline.py: C's publish 1.5-3.2 us).
struct Snap {
  double alpha, beta, omega, rho, sqrt_eps, h0, tol_abs;
  int32_t iter, bench, auto_rr, rr_next, rr_period, rr_off, n_rr, dist, p2p;
};

__device__ __forceinline__ void snap_load(Snap& p, const Scal* s) {
  p.alpha = s->alpha; p.beta = s->beta; p.omega = s->omega; p.rho = s->rho;
  p.sqrt_eps = s->sqrt_eps; p.h0 = s->h0; p.tol_abs = s->tol_abs;
  p.iter = s->iter; p.bench = s->bench; p.auto_rr = s->auto_rr; p.rr_next = s->rr_next;
  p.rr_period = s->rr_period; p.rr_off = s->rr_off; p.n_rr = s->n_rr;
  p.dist = s->dist; p.p2p = s->p2p;
}

// ---------------------------------------------------------------------------
// Automated replacement bookkeeping, one thread, same formulas and
// operation order as oracle.c; the norms are the kernels' Dot2 sums of squares
// (reading A30), so f^r and the decisions are the oracle's bitwise.
__device__ __forceinline__ void auto_step(Scal* s, Hist h, double R1) {
  const int i = s->iter;
  const double R = h.rnorm[i];
  const double nK = s->nA_[0], nW = s->nA_[1], nM = s->nA_[2], nT = s->nA_[3];
  const double nG = s->nA_[4], nS = s->nA_[5], nL = s->nA_[6], nZ = s->nA_[7];
  const double nQ = s->nA_[8], nY = s->nA_[9];
  const double nX = s->nC_[0], nU = s->nC_[1], nN = s->nC_[2], nV = s->nC_[3];
  const double nGp = s->nP_[0], nSp = s->nP_[1], nLp = s->nP_[2], nZp = s->nP_[3];
  const double nNp = s->nP_[4], nVp = s->nP_[5];
  const double alpha = s->alpha, beta = s->beta, omega = s->omega, om_prev = s->ar_omp;
  const double ab = fabs(beta), abw = fabs(beta * om_prev);
  const double aa = fabs(alpha), aw = fabs(omega), awa = fabs(omega * alpha);
  const double nA = s->ar_nA, muN = s->ar_muN, mutN = s->ar_mutN, e = s->ar_eps;
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
  const double Dz_i = ab * s->ar_Dz + nA * el * e + ez * e;
  const double Ds_i = s->ar_Dw + ab * s->ar_Ds + abw * s->ar_Dz + nA * eg * e + es * e;
  const double Dw_1 = s->ar_Dw + aa * Dz_i + nA * ek * e + ew * e + nA * eu * e + ey * e;
  const double f_1 = s->ar_f + aa * Ds_i + aw * s->ar_Dw + awa * Dz_i + nA * ex * e + er * e +
                     aw * nA * eu * e + eq * e + aw * ey * e;
  s->rr_next = (s->ar_f <= s->ar_tau * R) && (f_1 > s->ar_tau * R1);  // eq:criterion
  s->ar_f = f_1;
  s->ar_Dw = Dw_1;
  s->ar_Ds = Ds_i;
  s->ar_Dz = Dz_i;
  h.fr[i + 1] = f_1;
  s->nP_[0] = nG; s->nP_[1] = nS; s->nP_[2] = nL; s->nP_[3] = nZ;
  s->nP_[4] = nN; s->nP_[5] = nV;
}

// after a replacement in iteration i: the gaps of the explicit recomputation
// (reading A31); nZr = ||z_i|| replaced (rr2)
__device__ __forceinline__ void auto_reset(Scal* s, Hist h, double R1, double nZr) {
  const int i = s->iter;
  const double R = h.rnorm[i];
  const double nA = s->ar_nA, muN = s->ar_muN, e = s->ar_eps;
  const double f_1 = ((muN + 1.0) * nA * s->nR_[0] + s->nb) * e;
  const double Ds_i = muN * nA * s->nA_[4] * e;
  const double Dw_1 = muN * nA * s->nR_[1] * e;
  const double Dz_i = muN * nA * s->nR_[3] * e;
  s->rr_next = (s->ar_f <= s->ar_tau * R) && (f_1 > s->ar_tau * R1);
  s->ar_f = f_1;
  s->ar_Dw = Dw_1;
  s->ar_Ds = Ds_i;
  s->ar_Dz = Dz_i;
  h.fr[i + 1] = f_1;
  s->nP_[0] = s->nA_[4]; s->nP_[1] = s->nR_[2]; s->nP_[2] = s->nR_[3]; s->nP_[3] = nZr;
  s->nP_[4] = s->nC_[2]; s->nP_[5] = s->nC_[3];
}

// Line 21-26 bookkeeping once the five dots of reduction #2 are
// known: history, sqrt(eps) latch (A12), stop test (A7), beta_{i+1},
// alpha_{i+1} (left to right as printed, A4), breakdown (A9).
// p: the state before this step (Snap).
__device__ __forceinline__ void finalize_iteration(Scal* s, Hist h, const Snap& p, double rho1,
                                                   double dw, double ds, double dz, double rr) {
  const int i = p.iter;
  const double hn = sqrt(rr);
  h.rnorm[i + 1] = hn;
  {
    double* t = h.sc + SC_W * (size_t)i;
    t[6] = dw;
    t[7] = ds;
    t[8] = dz;
  }
  s->iters = i + 1;
  s->iter = i + 1;
  if (hn < p.sqrt_eps * p.h0) s->rr_off = 1;
  s->rr_fire = 0;
  if (hn <= p.tol_abs && !p.bench) {
    s->done = 1;
    s->outcome = OUT_CONVERGED;
    return;
  }
  const double alpha = p.alpha, omega = p.omega, rho = p.rho;
  const double beta1 = ((alpha / omega) * rho1) / rho;
  const double den = (dw + beta1 * ds) - (beta1 * omega) * dz;
  const double alpha1 = rho1 / den;
  s->beta = beta1;
  s->alpha = alpha1;
  s->rho = rho1;
  s->ar_omp = omega;  // omega_i is omega_{(i+1)-1} of the next auto_step
  if (!isfinite(beta1) || !isfinite(alpha1) || den == 0.0 || rho1 == 0.0) {
    s->done = 1;
    s->outcome = OUT_BREAKDOWN;
  }
}

// Replacement decision for iteration i (A11: (i+1) mod P == 0; A12 latch).
__device__ __forceinline__ bool rr_scheduled(const Snap& s) {
  if (s.auto_rr) return s.rr_next != 0;  // eq:criterion
  return s.rr_period > 0 && ((s.iter + 1) % s.rr_period) == 0 && !s.rr_off;
}

// The scalar-forming steps, given the combined dot totals (one thread).
template <int F>
__device__ __forceinline__ void fin_step(Scal* sc, Hist h, const Dd* tot, const Snap& p) {
  if (F == F_INIT1) {
    sc->tmp0 = dd_round(tot[0]);  // (r0, r0) = (r^0, r0) = rho_0
    sc->tmp1 = dd_round(tot[1]);  // (b, b)
    if (sc->auto_rr) {            // ||x_0||, ||k_0|| for f_0, Dw_0
      sc->nX0 = sqrt(dd_round(tot[2]));
      sc->nK0 = sqrt(dd_round(tot[3]));
    }
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
    if (sc->auto_rr) {  // initial gap bounds; Ds_{-1} = Dz_{-1} = 0 (A1)
      sc->ar_f = ((sc->ar_muN + 1.0) * sc->ar_nA * sc->nX0 + sc->nb) * sc->ar_eps;
      sc->ar_Dw = sc->ar_muN * sc->ar_nA * sc->nK0 * sc->ar_eps;
      sc->ar_Ds = 0.0;
      sc->ar_Dz = 0.0;
      sc->ar_omp = 0.0;
      for (int k = 0; k < 6; ++k) sc->nP_[k] = 0.0;
      sc->rr_next = 0;
      h.fr[0] = sc->ar_f;
    }
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
    {
      double* t = h.sc + SC_W * (size_t)p.iter;
      t[0] = p.alpha;
      t[1] = p.beta;
      t[2] = omn;
      t[3] = p.rho;
      t[4] = qy;
      t[5] = yy;
    }
    if (p.auto_rr)
      for (int k = 0; k < 10; ++k) sc->nA_[k] = sqrt(dd_round(tot[2 + k]));
    if (!isfinite(omn)) {
      sc->done = 1;
      sc->outcome = OUT_BREAKDOWN;
      sc->iters = p.iter;
    }
  } else if (F == F_SWEEPC) {
    if (p.auto_rr)
      for (int k = 0; k < 4; ++k) sc->nC_[k] = sqrt(dd_round(tot[5 + k]));
    if (rr_scheduled(p)) {
      sc->rr_fire = 1;  // the line-21 dots are recomputed after the replacement
      h.rrl[p.n_rr] = p.iter;
      sc->n_rr = p.n_rr + 1;
    } else {
      if (p.auto_rr) auto_step(sc, h, sqrt(dd_round(tot[4])));
      finalize_iteration(sc, h, p, dd_round(tot[0]), dd_round(tot[1]), dd_round(tot[2]),
                         dd_round(tot[3]), dd_round(tot[4]));
    }
  } else if (F == F_RR1) {  // norms of the replaced x_{i+1}, k_{i+1}, s_i, l_i
    for (int k = 0; k < 4; ++k) sc->nR_[k] = sqrt(dd_round(tot[k]));
  } else if (F == F_RR2) {
    if (p.auto_rr) auto_reset(sc, h, sqrt(dd_round(tot[4])), sqrt(dd_round(tot[5])));
    finalize_iteration(sc, h, p, dd_round(tot[0]), dd_round(tot[1]), dd_round(tot[2]),
                       dd_round(tot[3]), dd_round(tot[4]));
    sc->use_rr = 1;
  } else if (F == F_GAP) {
    h.gap[sc->iter] = sqrt(dd_round(tot[0]));
    sc->gap_iter = sc->iter;
  }
}

// Tail of every reducing kernel (thread 0 of the last CTA): finish on one rank,
// publish the rank's partial pairs on several.
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// pre: the kernel's prologue copy of the state (Snap), or null to load it here
template <int F, int K>
__device__ __forceinline__ void publish(Scal* sc, Hist h, const Dd (&tot)[K],
                                        const Snap* pre = nullptr) {
  Snap p;
  if (pre) p = *pre;
  else snap_load(p, sc);
  if (p.dist && p.p2p) {
    // every rank performs the same reductions in the same order: the epoch numbers
    // them identically on all ranks
    const unsigned long long e = *sc->p2p_epoch + 1;
    *sc->p2p_epoch = e;
    const int P = sc->nranks;
    const size_t off = ((size_t)(e & 1) * P + sc->rank) * RED_K;
    for (int q = 0; q < P; ++q) {
#pragma unroll
      for (int k = 0; k < K; ++k) sc->p2p_recv[q][off + k] = tot[k];
    }
    __threadfence_system();
    for (int q = 0; q < P; ++q) st_release_sys(sc->p2p_flag[q] + sc->rank, e);
  } else if (p.dist) {
    Dd* row = sc->red_send + (size_t)sc->rank * RED_K;
#pragma unroll
    for (int k = 0; k < K; ++k) row[k] = tot[k];
  } else {
    fin_step<F>(sc, h, tot, p);
  }
}

// One-CTA finalize after the exchange: combine the rank rows in rank order.
template <int F, int K>
__global__ void k_fin(Scal* __restrict__ sc, Hist h) {
  if (threadIdx.x != 0) return;
  if (F == F_GAP) {
    if (sc->gap_iter >= sc->iter) return;
  } else if (F == F_RR2 || F == F_RR1) {
    if (sc->done || !sc->rr_fire) return;
  } else if (F != F_INIT1 && F != F_INIT2) {
    if (sc->done) return;
  }
  const Dd* rows = sc->red_recv;
  if (sc->p2p) {  // wait for every rank's pairs of this epoch (written by their kernels)
    const unsigned long long e = *sc->p2p_epoch;
    const unsigned long long* flag = sc->p2p_flag[sc->rank];
    for (int r = 0; r < sc->nranks; ++r)
      while (ld_acquire_sys(flag + r) < e) __nanosleep(32);
    rows = sc->p2p_recv[sc->rank] + (size_t)(e & 1) * sc->nranks * RED_K;
  }
  Dd tot[K];
#pragma unroll
  for (int k = 0; k < K; ++k) tot[k] = dd_zero();
  for (int r = 0; r < sc->nranks; ++r) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const Dd* q = rows + (size_t)r * RED_K + k;
      Dd v;
      v.hi = __ldcv(&q->hi);  // peers wrote it over NVLink: bypass L1
      v.lo = __ldcv(&q->lo);
      tot[k] = dd_add(tot[k], v);
    }
  }
  Snap p;
  snap_load(p, sc);
  fin_step<F>(sc, h, tot, p);
}
