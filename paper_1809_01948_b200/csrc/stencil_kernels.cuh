// stencil_kernels.cuh -- matrix-free 5/7-point stencil path, fused 2-sweep
// schedule of Algorithm 2.
//
// B200 design: with a constant-coefficient stencil and
// Jacobi (pointwise dinv), the SpMV outputs t_i = A M^-1 w_i and
// v_i = A M^-1 z_i are recomputed on the fly from w and z inside the two AXPY
// sweeps instead of being stored, so one iteration is two streaming kernels:
//   sweepA : lines 5-12  (g, s, l, z; q, y in registers; Dot2 (q,y), (y,y))
//   sweepC : lines 16-21 (x, r, k, w; u, q, y recomputed; 5 Dot2 dots)
// Every value is produced with the same operations, in the same order, as the
// oracle's "compute and store" schedule, so results are bitwise identical.
// The reductions of lines 12 and 21 are the grid-level last-CTA reductions of
// dd.cuh; the scalars (omega; beta, alpha) are formed by that last CTA.
//
// Vectors have H ghost elements before and after the n_local rows (H = nx*ny in
// 3D, nx in 2D) so every neighbour address is inside the allocation; Dirichlet
// legs are dropped with selects (reading A5).  z and w are double-buffered
// because the sweeps read them with a stencil while writing the new values.
#pragma once
#include "dd.cuh"
#include "state.cuh"

struct Geo {
  int64_t nx, ny;    // x extent; y extent (3D)
  int64_t nol;       // local outer count: z-planes (3D) / y-lines (2D)
  int64_t o0, nog;   // global index of the first local outer plane/line; global count
  int64_t pxy;       // outer stride: nx*ny (3D) / nx (2D)
  int64_t nlines;    // x-lines owned: ny*nol (3D) / nol (2D)
  double c[7];       // {centre, -x, +x, -y, +y, -z, +z}
  double dinv;       // fl(1 / c[0])  (A3)
};

struct Vecs {
  double *x, *r, *rh, *k, *g, *s, *l, *b;
  double *w0, *w1, *z0, *z1, *zrr;
  double *nv, *mv;  // CSR path: n = M^-1 z and m = M^-1 w, inputs of the window SpMVs
  double *tv, *vv;  // stencil split schedule: stored t_i = A M^-1 w_i, v_i = A M^-1 z_i
  // peer-memory transport (option transport 1), fused schedule: where sweep A stores its
  // first / last plane of z (hz[b]: buffer z_b) and sweep C of w (hw[b]: buffer w_b) in
  // the lower ([0]: its upper ghost plane) and upper ([1]: its lower ghost plane)
  // neighbours' memory; nullptr = no neighbour / no fused halo
  double* hz[2][2];
  double* hw[2][2];
  // tile replacement step: per-CTA block totals of the three line-21 dots RR1 forms
  // ((r^, r), (r^, s), (r, r) of the replaced r, s), read back by RR2's grid reduction
  Dd* stash;
};

template <int DIM>
__device__ __forceinline__ void line_bnd(const Geo& g, int64_t line, bool& ym, bool& yp, bool& zm,
                                         bool& zp) {
  if (DIM == 3) {
    const int64_t y = line % g.ny;
    const int64_t oz = g.o0 + line / g.ny;
    ym = y > 0;
    yp = y < g.ny - 1;
    zm = oz > 0;
    zp = oz < g.nog - 1;
  } else {
    const int64_t oy = g.o0 + line;
    ym = oy > 0;
    yp = oy < g.nog - 1;
    zm = zp = false;
  }
}

// fl(A v)_j (PREC=false) or fl(A M^-1 v)_j (PREC=true), legs in ascending
// column order -z, -y, -x, c, +x, +y, +z, starting from +0.0 (A5).
template <int DIM, bool PREC>
__device__ __forceinline__ double apply_row(const double* __restrict__ v, int64_t j, double vc,
                                            const Geo& g, bool xm, bool xp, bool ym, bool yp,
                                            bool zm, bool zp) {
  double vzm = 0.0, vzp = 0.0;
  if (DIM == 3) {
    vzm = __ldg(v + j - g.pxy);
    vzp = __ldg(v + j + g.pxy);
  }
  const double vym = __ldg(v + j - g.nx), vyp = __ldg(v + j + g.nx);
  const double vxm = __ldg(v + j - 1), vxp = __ldg(v + j + 1);
  if (PREC) {
    vzm = g.dinv * vzm;
    vzp = g.dinv * vzp;
  }
  const double pym = PREC ? g.dinv * vym : vym, pyp = PREC ? g.dinv * vyp : vyp;
  const double pxm = PREC ? g.dinv * vxm : vxm, pxp = PREC ? g.dinv * vxp : vxp;
  const double pc = PREC ? g.dinv * vc : vc;
  double acc = 0.0;
  if (DIM == 3) acc = zm ? acc + g.c[5] * vzm : acc;
  acc = ym ? acc + g.c[3] * pym : acc;
  acc = xm ? acc + g.c[1] * pxm : acc;
  acc = acc + g.c[0] * pc;
  acc = xp ? acc + g.c[2] * pxp : acc;
  acc = yp ? acc + g.c[4] * pyp : acc;
  if (DIM == 3) acc = zp ? acc + g.c[6] * vzp : acc;
  return acc;
}

#define STENCIL_LOOP_BEGIN                                                  \
  for (int64_t line = blockIdx.x; line < g.nlines; line += gridDim.x) {     \
    bool ym, yp, zm, zp;                                                    \
    line_bnd<DIM>(g, line, ym, yp, zm, zp);                                 \
    const int64_t base = line * g.nx;                                       \
    for (int64_t xx = threadIdx.x; xx < g.nx; xx += blockDim.x) {           \
      const int64_t j = base + xx;                                          \
      const bool xm = xx > 0, xp = xx < g.nx - 1;
#define STENCIL_LOOP_END \
  }                      \
  }

#define NBR xm, xp, ym, yp, zm, zp

// ---------------------------------------------------------------------------
// init1 (Alg. 2 line 2): r0 := b - A x0; r^ := r0 (A2); k0 := M^-1 r0;
// dots (r0,r0) and (b,b).
template <int DIM>
__global__ void __launch_bounds__(256) k_init1(Geo g, Vecs V, Scal* __restrict__ sc,
                                               Dd* __restrict__ part, Hist h) {
  Dd acc[2] = {dd_zero(), dd_zero()};
  STENCIL_LOOP_BEGIN
  const double xc = V.x[j];
  const double ax = apply_row<DIM, false>(V.x, j, xc, g, NBR);
  const double bj = V.b[j];
  const double rj = bj - ax;
  V.r[j] = rj;
  V.rh[j] = rj;
  V.k[j] = g.dinv * rj;
  dd_fma(acc[0], rj, rj);
  dd_fma(acc[1], bj, bj);
  STENCIL_LOOP_END
  Dd tot[2];
  if (dd_grid_reduce<2>(acc, part, &sc->counter[T_INIT1], tot) && threadIdx.x == 0)
    publish<F_INIT1>(sc, h, tot);
}

// init2 (lines 2-3): w0 := A k0 = A M^-1 r0; (r0, w0);
// alpha0 := (r0,r0)/(r0,w0); beta0 := 0; omega_{-1} := 0 (A1).
template <int DIM>
__global__ void __launch_bounds__(256) k_init2(Geo g, Vecs V, Scal* __restrict__ sc,
                                               Dd* __restrict__ part, Hist h) {
  Dd acc[1] = {dd_zero()};
  STENCIL_LOOP_BEGIN
  const double rc = V.r[j];
  const double wj = apply_row<DIM, true>(V.r, j, rc, g, NBR);
  V.w0[j] = wj;
  dd_fma(acc[0], V.rh[j], wj);
  STENCIL_LOOP_END
  Dd tot[1];
  if (dd_grid_reduce<1>(acc, part, &sc->counter[T_INIT2], tot) && threadIdx.x == 0)
    publish<F_INIT2>(sc, h, tot);
}

// ---------------------------------------------------------------------------
// sweepA = Alg. 2 lines 5-12 with lines 13-14 of the previous
// iteration (n_{i-1}, v_{i-1}) and line 22-23 (m_i, t_i) recomputed from z_{i-1}
// and w_i on the fly.  After a replacement, n_{i-1}, v_{i-1} come from the
// pre-replacement z (reading A26) while the s and z recurrences use the
// replaced z.
template <int DIM>
__global__ void __launch_bounds__(256) k_sweepA(Geo g, Vecs V, Scal* __restrict__ sc,
                                                Dd* __restrict__ part, Hist h) {
  if (sc->done) return;
  const int it = sc->iter;
  const double al = sc->alpha, be = sc->beta, om = sc->omega;
  const bool rr = sc->use_rr != 0;
  const double* __restrict__ w = (it & 1) ? V.w1 : V.w0;
  const double* __restrict__ zn = (it & 1) ? V.z0 : V.z1;  // z_{i-1} (pre-replacement)
  const double* __restrict__ zo = rr ? V.zrr : zn;          // z_{i-1} as replaced
  double* __restrict__ zw = (it & 1) ? V.z1 : V.z0;         // z_i
  Dd acc[2] = {dd_zero(), dd_zero()};
  STENCIL_LOOP_BEGIN
  const double wc = w[j];
  const double znc = zn[j];
  const double zoc = rr ? zo[j] : znc;
  const double m = g.dinv * wc;                                 // m_i = M^-1 w_i
  const double t = apply_row<DIM, true>(w, j, wc, g, NBR);      // t_i = A m_i
  const double n = g.dinv * znc;                                // n_{i-1}
  const double v = apply_row<DIM, true>(zn, j, znc, g, NBR);    // v_{i-1}
  const double lj = V.l[j];
  const double gn = V.k[j] + be * (V.g[j] - om * lj);           // line 5
  const double sn = wc + be * (V.s[j] - om * zoc);              // line 6
  const double ln = m + be * (lj - om * n);                     // line 7
  const double zz = t + be * (zoc - om * v);                    // line 8
  const double q = V.r[j] - al * sn;                            // line 9
  const double y = wc - al * zz;                                // line 11
  dd_fma(acc[0], q, y);                                         // line 12
  dd_fma(acc[1], y, y);
  V.g[j] = gn;
  V.s[j] = sn;
  V.l[j] = ln;
  zw[j] = zz;
  STENCIL_LOOP_END
  Dd tot[2];
  if (dd_grid_reduce<2>(acc, part, &sc->counter[T_SWEEPA], tot) && threadIdx.x == 0)
    publish<F_SWEEPA>(sc, h, tot);
}

// sweepC = Alg. 2 lines 17-21: x, r, k, w; u, q, y recomputed
// (bitwise equal to sweepA's), m_i, n_i, t_i, v_i on the fly; Dot2
// (r0,r_{i+1}), (r0,w_{i+1}), (r0,s_i), (r0,z_i) and (r_{i+1},r_{i+1}) (A8).
template <int DIM>
__global__ void __launch_bounds__(256) k_sweepC(Geo g, Vecs V, Scal* __restrict__ sc,
                                                Dd* __restrict__ part, Hist h) {
  if (sc->done) return;
  const int it = sc->iter;
  const double al = sc->alpha, om = sc->omega;
  const double* __restrict__ w = (it & 1) ? V.w1 : V.w0;  // w_i
  double* __restrict__ ww = (it & 1) ? V.w0 : V.w1;       // w_{i+1}
  const double* __restrict__ z = (it & 1) ? V.z1 : V.z0;  // z_i
  Dd acc[5] = {dd_zero(), dd_zero(), dd_zero(), dd_zero(), dd_zero()};
  STENCIL_LOOP_BEGIN
  const double wc = w[j], zc = z[j];
  const double m = g.dinv * wc;                              // m_i
  const double t = apply_row<DIM, true>(w, j, wc, g, NBR);   // t_i
  const double n = g.dinv * zc;                              // n_i (line 13)
  const double v = apply_row<DIM, true>(z, j, zc, g, NBR);   // v_i (line 14)
  const double sj = V.s[j];
  const double u = V.k[j] - al * V.l[j];                     // line 10
  const double q = V.r[j] - al * sj;                         // line 9
  const double y = wc - al * zc;                             // line 11
  const double xn = (V.x[j] + al * V.g[j]) + om * u;         // line 17
  const double rn = q - om * y;                              // line 18
  const double kn = u - om * (m - al * n);                   // line 19
  const double wn = y - om * (t - al * v);                   // line 20
  const double rhj = V.rh[j];
  dd_fma(acc[0], rhj, rn);                                   // line 21
  dd_fma(acc[1], rhj, wn);
  dd_fma(acc[2], rhj, sj);
  dd_fma(acc[3], rhj, zc);
  dd_fma(acc[4], rn, rn);
  V.x[j] = xn;
  V.r[j] = rn;
  V.k[j] = kn;
  ww[j] = wn;
  STENCIL_LOOP_END
  Dd tot[5];
  if (dd_grid_reduce<5>(acc, part, &sc->counter[T_SWEEPC], tot) && threadIdx.x == 0)
    publish<F_SWEEPC>(sc, h, tot);
}

// ---------------------------------------------------------------------------
// Residual replacement eq:rr after line 20:
// rr1: r := b - A x; k := M^-1 r; s := A g; l := M^-1 s
template <int DIM>
__global__ void __launch_bounds__(256) k_rr1(Geo g, Vecs V, Scal* __restrict__ sc) {
  if (sc->done || !sc->rr_fire) return;
  STENCIL_LOOP_BEGIN
  const double xc = V.x[j], gc = V.g[j];
  const double ax = apply_row<DIM, false>(V.x, j, xc, g, NBR);
  const double rj = V.b[j] - ax;
  const double sj = apply_row<DIM, false>(V.g, j, gc, g, NBR);
  V.r[j] = rj;
  V.k[j] = g.dinv * rj;
  V.s[j] = sj;
  V.l[j] = g.dinv * sj;
  STENCIL_LOOP_END
}

// rr2: w := A k = A M^-1 r; z := A l = A M^-1 s (into zrr: the pre-replacement
// z_i stays for n_i, v_i, A26); then the line-21 dots on the replaced vectors.
template <int DIM>
__global__ void __launch_bounds__(256) k_rr2(Geo g, Vecs V, Scal* __restrict__ sc,
                                             Dd* __restrict__ part, Hist h) {
  if (sc->done || !sc->rr_fire) return;
  const int it = sc->iter;
  double* __restrict__ ww = (it & 1) ? V.w0 : V.w1;  // w_{i+1}
  Dd acc[5] = {dd_zero(), dd_zero(), dd_zero(), dd_zero(), dd_zero()};
  STENCIL_LOOP_BEGIN
  const double rc = V.r[j], sc_ = V.s[j];
  const double wn = apply_row<DIM, true>(V.r, j, rc, g, NBR);
  const double zr = apply_row<DIM, true>(V.s, j, sc_, g, NBR);
  ww[j] = wn;
  V.zrr[j] = zr;
  const double rhj = V.rh[j];
  dd_fma(acc[0], rhj, rc);
  dd_fma(acc[1], rhj, wn);
  dd_fma(acc[2], rhj, sc_);
  dd_fma(acc[3], rhj, zr);
  dd_fma(acc[4], rc, rc);
  STENCIL_LOOP_END
  Dd tot[5];
  if (dd_grid_reduce<5>(acc, part, &sc->counter[T_RR2], tot) && threadIdx.x == 0)
    publish<F_RR2>(sc, h, tot);
}

// ---------------------------------------------------------------------------
// Gap tracking (eq:res_gap P:113, reading A13): ||(b - A x_i) - r_i|| for the
// latest completed iteration i = iter, once per iteration.
template <int DIM>
__global__ void __launch_bounds__(256) k_gap(Geo g, Vecs V, Scal* __restrict__ sc,
                                             Dd* __restrict__ part, Hist h) {
  if (sc->gap_iter >= sc->iter) return;
  Dd acc[1] = {dd_zero()};
  STENCIL_LOOP_BEGIN
  const double xc = V.x[j];
  const double ax = apply_row<DIM, false>(V.x, j, xc, g, NBR);
  const double d = (V.b[j] - ax) - V.r[j];
  dd_fma(acc[0], d, d);
  STENCIL_LOOP_END
  Dd tot[1];
  if (dd_grid_reduce<1>(acc, part, &sc->counter[T_GAP], tot) && threadIdx.x == 0)
    publish<F_GAP>(sc, h, tot);
}

// y = A x (pbicgstab_apply): same leg order as the solver.
template <int DIM>
__global__ void __launch_bounds__(256) k_apply(Geo g, const double* __restrict__ xin,
                                               double* __restrict__ yout) {
  STENCIL_LOOP_BEGIN
  const double xc = xin[j];
  yout[j] = apply_row<DIM, false>(xin, j, xc, g, NBR);
  STENCIL_LOOP_END
}

// ---------------------------------------------------------------------------
// Split 4-phase schedule on a stencil (option schedule 2; the paper's own
// pipeline): the SpMVs of lines 13-14 and 22-23 are separate tile kernels
// (TM_SPB / TM_SPD) that the two global reductions hide behind on P ranks; these
// two point-wise sweeps read the stored t_i, v_{i-1} / v_i.  Same operations in the
// same order as the fused sweeps (tile_sweeps.cuh row_update), so bitwise equal.
// Buffers follow the fused convention: w_i in {w0, w1}[i & 1], z_i in {z0, z1}[i & 1].
template <int DIM>
__global__ void __launch_bounds__(256) k_sweepA2(Geo g, Vecs V, Scal* __restrict__ sc,
                                                 Dd* __restrict__ part, Hist h) {
  if (sc->done) return;
  const int it = sc->iter;
  const double al = sc->alpha, be = sc->beta, om = sc->omega;
  const bool rr = sc->use_rr != 0;
  const double* __restrict__ w = (it & 1) ? V.w1 : V.w0;   // w_i
  const double* __restrict__ zn = (it & 1) ? V.z0 : V.z1;  // z_{i-1} pre-replacement
  double* __restrict__ zw = (it & 1) ? V.z1 : V.z0;        // z_i
  const double dinv = g.dinv;
  const int64_t n = g.nlines * g.nx;
  Dd acc[2] = {dd_zero(), dd_zero()};
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double c0 = __ldcs(w + j), c1 = __ldcs(zn + j);
    const double zoc = rr ? __ldcs(V.zrr + j) : c1;
    const double t0 = __ldcs(V.tv + j), t1 = __ldcs(V.vv + j);  // t_i, v_{i-1}
    const double kj = __ldcs(V.k + j), gj = __ldcs(V.g + j), lj = __ldcs(V.l + j);
    const double sj = __ldcs(V.s + j), rj = __ldcs(V.r + j);
    const double m = dinv * c0, nn = dinv * c1;
    const double gn = kj + be * (gj - om * lj);                // line 5
    const double sn = c0 + be * (sj - om * zoc);               // line 6
    const double ln = m + be * (lj - om * nn);                 // line 7
    const double zz = t0 + be * (zoc - om * t1);               // line 8
    const double qq = rj - al * sn;                            // line 9
    const double yy = c0 - al * zz;                            // line 11
    dd_fma(acc[0], qq, yy);                                    // line 12
    dd_fma(acc[1], yy, yy);
    __stcs(V.g + j, gn);
    __stcs(V.s + j, sn);
    __stcs(V.l + j, ln);
    __stcs(zw + j, zz);
  }
  Dd tot[2];
  if (dd_grid_reduce<2>(acc, part, &sc->counter[T_SWEEPA], tot) && threadIdx.x == 0)
    publish<F_SWEEPA>(sc, h, tot);
}

template <int DIM>
__global__ void __launch_bounds__(256) k_sweepC2(Geo g, Vecs V, Scal* __restrict__ sc,
                                                 Dd* __restrict__ part, Hist h) {
  if (sc->done) return;
  const int it = sc->iter;
  const double al = sc->alpha, om = sc->omega;
  const double* __restrict__ w = (it & 1) ? V.w1 : V.w0;  // w_i
  double* __restrict__ ww = (it & 1) ? V.w0 : V.w1;       // w_{i+1}
  const double* __restrict__ z = (it & 1) ? V.z1 : V.z0;  // z_i
  const double dinv = g.dinv;
  const int64_t n = g.nlines * g.nx;
  Dd acc[5] = {dd_zero(), dd_zero(), dd_zero(), dd_zero(), dd_zero()};
  // SpMV_D may run before the finalize step advances iter (P ranks, overlap): tell it
  // where w_{i+1} is
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->spd_par = (it + 1) & 1;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double c0 = w[j], c1 = z[j];
    const double t0 = V.tv[j], t1 = V.vv[j];                  // t_i, v_i
    const double xj = V.x[j], gj = V.g[j], kj = V.k[j], lj = V.l[j], rj = V.r[j];
    const double sj = V.s[j], rhj = V.rh[j];
    const double m = dinv * c0, nn = dinv * c1;
    const double uu = kj - al * lj;                             // line 10
    const double qq = rj - al * sj;                             // line 9
    const double yy = c0 - al * c1;                             // line 11
    const double xn = (xj + al * gj) + om * uu;                 // line 17
    const double rn = qq - om * yy;                             // line 18
    const double kn = uu - om * (m - al * nn);                  // line 19
    const double wn = yy - om * (t0 - al * t1);                 // line 20
    dd_fma(acc[0], rhj, rn);                                    // line 21
    dd_fma(acc[1], rhj, wn);
    dd_fma(acc[2], rhj, sj);
    dd_fma(acc[3], rhj, c1);
    dd_fma(acc[4], rn, rn);
    V.x[j] = xn;
    V.r[j] = rn;
    V.k[j] = kn;
    ww[j] = wn;
  }
  Dd tot[5];
  if (dd_grid_reduce<5>(acc, part, &sc->counter[T_SWEEPC], tot) && threadIdx.x == 0)
    publish<F_SWEEPC>(sc, h, tot);
}
