// tile_sweeps.cuh -- the two fused sweeps of the stencil schedule as
// TMA-staged 2.5D z-marching kernels (the hot path on B200).
//
// Same arithmetic, same operation order as k_sweepA / k_sweepC
// (stencil_kernels.cuh) -- only the data movement differs:
//   * a CTA owns a tile of TY full x-lines of a plane (3D) or one x-line (2D)
//     and marches the outer dimension (z in 3D, y in 2D) over a chunk of planes;
//   * one elected thread streams every vector the step needs into shared memory
//     with cp.async.bulk (TMA bulk copies) one plane ahead, completion tracked by
//     mbarriers, so ~100 KB per SM is in flight while the CTA computes;
//   * the stencil operands w and z (z_{i-1} in sweepA) are staged as planes with
//     one halo line on each side (a 3-slot ring: z, z+1 resident, z+2 in flight);
//     the -z leg comes from registers (the previous step's centre values);
//   * one row pair per thread; 16-byte shared loads / global streaming stores
//     when nx is even; a warp-uniform interior path drops the boundary selects;
//   * outputs are written with streaming stores.
// Per row the kernels touch DRAM exactly once per vector (tile halos hit L2).
#pragma once
#include "dd.cuh"
#include "state.cuh"
#include "stencil_kernels.cuh"
#include "tma.cuh"

#define TNT 512      // threads per CTA
#define TNSTR_A 6    // sweepA streams: k, g, l, s, r (+ replaced z_{i-1})
#define TNSTR_C 7    // sweepC streams: x, g, k, l, r, s, r^

struct TileGeo {
  int64_t nx, ny;     // x extent; lines per plane (3D: ny, 2D: 1)
  int64_t nol, o0, nog;
  int64_t pxy;        // plane stride in rows
  int32_t TY, ncols, chunk, nchunks, units;
  int32_t st_stride;  // doubles per stream vector slot (even)
  int32_t sv_stride;  // doubles per stencil vector slot (even)
  int32_t halo;       // rows staged before the tile start (3D: nx + 2; 2D: 2)
  double c[7];
  double dinv;
};

__device__ __forceinline__ int align_off(const double* p) {
  return (int)(((uintptr_t)p & 15u) >> 3);
}

// stage `n` vectors' element range [e0, e0 + len) of plane p into dst slots
__device__ __forceinline__ void stage(double* dst, int stride, const double* const* src, int n,
                                      int64_t e0, int len, uint64_t* bar) {
  const double* s0 = src[0] + e0;
  const int off = align_off(s0);
  const uint32_t bytes = (uint32_t)(((off + len) * 8 + 15) & ~15);
  mbar_arrive_expect_tx(bar, bytes * (uint32_t)n);
  for (int v = 0; v < n; ++v)
    bulk_g2s(dst + (size_t)v * stride, src[v] + e0 - off, bytes, bar);
}

// two consecutive values from shared memory (16-byte load when VEC)
template <bool VEC>
__device__ __forceinline__ void ld2(const double* p, double& a, double& b) {
  if (VEC) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    a = v.x;
    b = v.y;
  } else {
    a = p[0];
    b = p[1];
  }
}

template <bool VEC>
__device__ __forceinline__ void st2(double* p, double a, double b, bool valid1) {
  if (VEC) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(a, b));
  } else {
    __stcs(p, a);
    if (valid1) __stcs(p + 1, b);
  }
}

// add one stencil leg: always (INTERIOR) or when its boundary bit is set (A5)
template <bool INTERIOR>
__device__ __forceinline__ double leg(unsigned b, unsigned bit, double acc, double term) {
  return (INTERIOR || (b & bit)) ? acc + term : acc;
}

// fl(A M^-1 v) for the row pair (r, r+1) of plane z.  W points at row r of
// plane z in shared memory, W1 at row r of plane z+1; m0/m1 are the plane z-1
// centre values.  Legs in ascending column order (A5); every leg is
// fl(c * fl(dinv * v)) added left to right from +0.0, exactly as the oracle's
// "n := M^-1 z; v := A n".  Products fl(dinv * v) shared by the two rows are
// formed once (same values).  bnd bits: 1 zm, 2 ym, 4 xm, 8 xp, 16 yp, 32 zp.
template <int DIM, bool VEC, bool INTERIOR>
__device__ __forceinline__ void stencil_pair(const TileGeo& g, int nx, const double* W,
                                             const double* W1, double zm0, double zm1,
                                             unsigned b0, unsigned b1, double& c0, double& c1,
                                             double& t0, double& t1) {
  const double d = g.dinv;
  ld2<VEC>(W, c0, c1);
  const double pm = d * W[-1], p0 = d * c0, p1 = d * c1, p2 = d * W[2];
  double ym0 = 0.0, ym1 = 0.0, yp0 = 0.0, yp1 = 0.0, zp0, zp1;
  if (DIM == 3) {
    ld2<VEC>(W - nx, ym0, ym1);
    ld2<VEC>(W + nx, yp0, yp1);
  }
  ld2<VEC>(W1, zp0, zp1);
  const double czm = g.c[DIM == 3 ? 5 : 3], czp = g.c[DIM == 3 ? 6 : 4];
  double a = 0.0;
  a = leg<INTERIOR>(b0, 1u, a, czm * (d * zm0));
  if (DIM == 3) a = leg<INTERIOR>(b0, 2u, a, g.c[3] * (d * ym0));
  a = leg<INTERIOR>(b0, 4u, a, g.c[1] * pm);
  a = a + g.c[0] * p0;
  a = leg<INTERIOR>(b0, 8u, a, g.c[2] * p1);
  if (DIM == 3) a = leg<INTERIOR>(b0, 16u, a, g.c[4] * (d * yp0));
  a = leg<INTERIOR>(b0, 32u, a, czp * (d * zp0));
  t0 = a;
  a = 0.0;
  a = leg<INTERIOR>(b1, 1u, a, czm * (d * zm1));
  if (DIM == 3) a = leg<INTERIOR>(b1, 2u, a, g.c[3] * (d * ym1));
  a = leg<INTERIOR>(b1, 4u, a, g.c[1] * p0);
  a = a + g.c[0] * p1;
  a = leg<INTERIOR>(b1, 8u, a, g.c[2] * p2);
  if (DIM == 3) a = leg<INTERIOR>(b1, 16u, a, g.c[4] * (d * yp1));
  a = leg<INTERIOR>(b1, 32u, a, czp * (d * zp1));
  t1 = a;
}

// Lines 5-12 (MODE 0) or 17-21 (MODE 1) for one row, given t = A M^-1 w and
// v = A M^-1 z at that row.  S = stream slot (row already applied), st = stride.
template <int MODE, int K>
__device__ __forceinline__ void row_update(const double* S, int st, bool rr, double wc, double zc,
                                           double t, double v, double al, double be, double om,
                                           double dinv, Dd (&acc)[K], double (&o)[4]) {
  if (MODE == 0) {
    const double kj = S[0], gj = S[st], lj = S[2 * st], sj = S[3 * st], rj = S[4 * st];
    const double zoc = rr ? S[5 * st] : zc;    // replaced z_{i-1} (A26)
    const double m = dinv * wc;                // m_i
    const double nn = dinv * zc;               // n_{i-1}
    o[0] = kj + be * (gj - om * lj);           // line 5: g
    o[1] = wc + be * (sj - om * zoc);          // line 6: s
    o[2] = m + be * (lj - om * nn);            // line 7: l
    o[3] = t + be * (zoc - om * v);            // line 8: z
    const double qq = rj - al * o[1];          // line 9
    const double yy = wc - al * o[3];          // line 11
    dd_fma(acc[0], qq, yy);                    // line 12
    dd_fma(acc[1 % K], yy, yy);
  } else {
    const double xj = S[0], gj = S[st], kj = S[2 * st], lj = S[3 * st], rj = S[4 * st];
    const double sj = S[5 * st], rhj = S[6 * st];
    const double m = dinv * wc;                // m_i
    const double nn = dinv * zc;               // n_i (line 13)
    const double uu = kj - al * lj;            // line 10
    const double qq = rj - al * sj;            // line 9
    const double yy = wc - al * zc;            // line 11
    o[0] = (xj + al * gj) + om * uu;           // line 17: x
    o[1] = qq - om * yy;                       // line 18: r
    o[2] = uu - om * (m - al * nn);            // line 19: k
    o[3] = yy - om * (t - al * v);             // line 20: w
    dd_fma(acc[0], rhj, o[1]);                 // line 21
    dd_fma(acc[1 % K], rhj, o[3]);
    dd_fma(acc[2 % K], rhj, sj);
    dd_fma(acc[3 % K], rhj, zc);
    dd_fma(acc[4 % K], o[1], o[1]);
  }
}

// MODE 0 = sweepA (lines 5-12), MODE 1 = sweepC (lines 17-21).  VEC: every
// staged range and every vector is 16-byte aligned (nx even) -> paired loads
// and stores.  One row pair per thread: TP <= 2 * TNT.
template <int DIM, int MODE, bool VEC>
__global__ void __launch_bounds__(TNT, 1) t_sweep(TileGeo g, Vecs V, Scal* __restrict__ sc,
                                                  Dd* __restrict__ part, Hist h) {
  constexpr int NSTR_MAX = MODE == 0 ? TNSTR_A : TNSTR_C;
  constexpr int K = MODE == 0 ? 2 : 5;
  if (sc->done) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);  // [0,1] streams, [2..4] stencil
  double* st = reinterpret_cast<double*>(smem_raw + 64);
  double* sv = st + 2 * NSTR_MAX * g.st_stride;
  const int tid = threadIdx.x;
  const int nx = (int)g.nx;
  const int sts = g.st_stride, svs = g.sv_stride;

  const int it = sc->iter;
  const double al = sc->alpha, be = sc->beta, om = sc->omega;
  const bool rr = MODE == 0 && sc->use_rr != 0;
  const double* svp[2];
  const double* stp[NSTR_MAX];
  int nstr;
  double* outp[4];
  if (MODE == 0) {
    svp[0] = (it & 1) ? V.w1 : V.w0;                 // w_i
    svp[1] = (it & 1) ? V.z0 : V.z1;                 // z_{i-1} pre-replacement
    stp[0] = V.k; stp[1] = V.g; stp[2] = V.l; stp[3] = V.s; stp[4] = V.r;
    stp[NSTR_MAX - 1] = V.zrr;                       // z_{i-1} replaced (A26)
    nstr = rr ? 6 : 5;
    outp[0] = V.g; outp[1] = V.s; outp[2] = V.l;
    outp[3] = (it & 1) ? V.z1 : V.z0;                // z_i
  } else {
    svp[0] = (it & 1) ? V.w1 : V.w0;                 // w_i
    svp[1] = (it & 1) ? V.z1 : V.z0;                 // z_i
    stp[0] = V.x; stp[1] = V.g; stp[2] = V.k; stp[3] = V.l; stp[4] = V.r; stp[5] = V.s;
    stp[NSTR_MAX - 1] = V.rh;
    nstr = 7;
    outp[0] = V.x; outp[1] = V.r; outp[2] = V.k;
    outp[3] = (it & 1) ? V.w0 : V.w1;                // w_{i+1}
  }
  if (tid == 0) {
    for (int i = 0; i < 5; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  uint32_t ph = 0;        // parity bits: bit s (streams 0,1), bit 2+s (stencil 0..2)
  int svc = 0, stc = 0;   // ring counters (slots filled so far)
  Dd acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = dd_zero();
  const int r = 2 * tid;  // this thread's row pair within the tile

  for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
    const int col = u % g.ncols, q = u / g.ncols;
    const int64_t y0 = (int64_t)col * g.TY;
    const int tyc = (int)((g.ny - y0) < g.TY ? (g.ny - y0) : g.TY);
    const int TP = tyc * nx;
    const int64_t z0 = (int64_t)q * g.chunk;
    const int64_t z1 = (z0 + g.chunk) < g.nol ? (z0 + g.chunk) : g.nol;
    const int nst = (int)(z1 - z0), nsv = nst + 2;
    const int64_t toff = DIM == 3 ? y0 * g.nx : 0;
    // per-row boundary bits (constant over the unit)
    const bool act = r < TP, valid1 = r + 1 < TP;
    unsigned b0 = 0, b1 = 0;
    {
      const int x0 = r % nx, x1 = (r + 1) % nx;
      const int64_t gy0 = y0 + r / nx, gy1 = y0 + (r + 1) / nx;
      if (x0 > 0) b0 |= 4u;
      if (x0 < nx - 1) b0 |= 8u;
      if (x1 > 0) b1 |= 4u;
      if (x1 < nx - 1) b1 |= 8u;
      if (DIM == 3) {
        if (gy0 > 0) b0 |= 2u;
        if (gy0 < g.ny - 1) b0 |= 16u;
        if (gy1 > 0) b1 |= 2u;
        if (gy1 < g.ny - 1) b1 |= 16u;
      }
    }
    const unsigned xy_all = DIM == 3 ? 30u : 12u;
    const bool xy_int = __all_sync(0xffffffffu, !act || ((b0 & xy_all) == xy_all &&
                                                         (b1 & xy_all) == xy_all));
    double mw0 = 0.0, mw1 = 0.0, mz0 = 0.0, mz1 = 0.0;  // plane z-1 centre values
    if (tid == 0) {
      for (int m = 0; m < 3 && m < nsv; ++m) {
        const int s = (svc + m) % 3;
        stage(sv + (size_t)s * 2 * svs, svs, svp, 2, (z0 - 1 + m) * g.pxy + toff - g.halo,
              TP + 2 * g.halo, &bar[2 + s]);
      }
      const int s = stc % 2;
      stage(st + (size_t)s * NSTR_MAX * sts, sts, stp, nstr, z0 * g.pxy + toff, TP, &bar[s]);
    }
    {  // plane z0-1 -> registers
      const int s = svc % 3;
      mbar_wait(&bar[2 + s], (ph >> (2 + s)) & 1u);
      ph ^= 1u << (2 + s);
      const double* b0p = sv + (size_t)s * 2 * svs +
                          align_off(svp[0] + (z0 - 1) * g.pxy + toff - g.halo) + g.halo + r;
      if (act) {
        ld2<VEC>(b0p, mw0, mw1);
        ld2<VEC>(b0p + svs, mz0, mz1);
      }
      const int s1 = (svc + 1) % 3;  // plane z0
      mbar_wait(&bar[2 + s1], (ph >> (2 + s1)) & 1u);
      ph ^= 1u << (2 + s1);
    }
    for (int n = 0; n < nst; ++n) {
      const int64_t z = z0 + n;
      __syncthreads();  // step n-1 done: its plane-(z-1) slot and stream slot are free
      if (tid == 0) {
        if (n + 3 < nsv) {  // plane z+2
          const int s = (svc + n + 3) % 3;
          stage(sv + (size_t)s * 2 * svs, svs, svp, 2, (z + 2) * g.pxy + toff - g.halo,
                TP + 2 * g.halo, &bar[2 + s]);
        }
        if (n + 1 < nst) {  // streams z+1
          const int s = (stc + n + 1) % 2;
          stage(st + (size_t)s * NSTR_MAX * sts, sts, stp, nstr, (z + 1) * g.pxy + toff, TP,
                &bar[s]);
        }
      }
      const int s_z = (svc + n + 1) % 3, s_z1 = (svc + n + 2) % 3, s_st = (stc + n) % 2;
      mbar_wait(&bar[2 + s_z1], (ph >> (2 + s_z1)) & 1u);
      ph ^= 1u << (2 + s_z1);
      mbar_wait(&bar[s_st], (ph >> s_st) & 1u);
      ph ^= 1u << s_st;
      if (!act) continue;
      const int oz = align_off(svp[0] + z * g.pxy + toff - g.halo) + g.halo;
      const int oz1 = align_off(svp[0] + (z + 1) * g.pxy + toff - g.halo) + g.halo;
      const int os = align_off(stp[0] + z * g.pxy + toff);
      const double* Wz = sv + (size_t)s_z * 2 * svs + oz + r;
      const double* Wz1 = sv + (size_t)s_z1 * 2 * svs + oz1 + r;
      const double* S0 = st + (size_t)s_st * NSTR_MAX * sts + os + r;
      const bool zin = (g.o0 + z) > 0 && (g.o0 + z) < g.nog - 1;
      const unsigned zb = ((g.o0 + z) > 0 ? 1u : 0u) | ((g.o0 + z) < g.nog - 1 ? 32u : 0u);
      double wc0, wc1, zc0, zc1, t0, t1, v0, v1;
      if (xy_int && zin) {
        stencil_pair<DIM, VEC, true>(g, nx, Wz, Wz1, mw0, mw1, 0u, 0u, wc0, wc1, t0, t1);
        stencil_pair<DIM, VEC, true>(g, nx, Wz + svs, Wz1 + svs, mz0, mz1, 0u, 0u, zc0, zc1, v0,
                                     v1);
      } else {
        stencil_pair<DIM, VEC, false>(g, nx, Wz, Wz1, mw0, mw1, b0 | zb, b1 | zb, wc0, wc1, t0,
                                      t1);
        stencil_pair<DIM, VEC, false>(g, nx, Wz + svs, Wz1 + svs, mz0, mz1, b0 | zb, b1 | zb,
                                      zc0, zc1, v0, v1);
      }
      mw0 = wc0;
      mw1 = wc1;
      mz0 = zc0;
      mz1 = zc1;
      double o0[4], o1[4];
      row_update<MODE, K>(S0, sts, rr, wc0, zc0, t0, v0, al, be, om, g.dinv, acc, o0);
      if (valid1) {
        row_update<MODE, K>(S0 + 1, sts, rr, wc1, zc1, t1, v1, al, be, om, g.dinv, acc, o1);
      } else {
        o1[0] = o1[1] = o1[2] = o1[3] = 0.0;
      }
      const int64_t gi = z * g.pxy + toff + r;
#pragma unroll
      for (int k = 0; k < 4; ++k) st2<VEC>(outp[k] + gi, o0[k], o1[k], valid1);
    }
    __syncthreads();  // unit done: every slot is free
    svc = (svc + nsv) % 3;
    stc = (stc + nst) % 2;
  }
  Dd tot[K];
  if (dd_grid_reduce<K>(acc, part, &sc->counter[MODE == 0 ? T_SWEEPA : T_SWEEPC], tot) &&
      tid == 0) {
    if (MODE == 0) publish<F_SWEEPA>(sc, h, tot);
    else publish<F_SWEEPC>(sc, h, tot);
  }
}

// host-side helper: shared-memory bytes of a t_sweep<., MODE> launch
inline size_t tile_smem_bytes(const TileGeo& g, int mode) {
  const int nstr = mode == 0 ? TNSTR_A : TNSTR_C;
  return 64 + sizeof(double) * ((size_t)2 * nstr * g.st_stride + (size_t)3 * 2 * g.sv_stride);
}
