// spmv_tile.cuh -- tall-tile kernels for the light steps of 3D Jacobi stencils:
//   * the split schedule's stand-alone SpMVs v_i = A M^-1 z_i (Alg. 2 lines 13-14,
//     P:185) and t_{i+1} = A M^-1 w_{i+1} (lines 22-23): TM_SPB / TM_SPD, four
//     row pairs per thread (option schedule 2 / the auto split schedule of small
//     multi-GPU slabs);
//   * the periodic residual replacement (eq:rr, then the line-21 dots on
//     the replaced vectors): TM_RR1 / TM_RR2 with the dot stash of
//     tile_sweeps.cuh (Stash), two row pairs per thread.
//
// Same data movement as the corresponding t_tile instances (a ring of TMA-staged
// planes with one halo line on each side, the -z leg from registers, streamed vectors
// one plane ahead) and the same arithmetic (stencil_pair: legs in ascending column
// order from +0.0; the modes' row updates and Dot2 accumulations expression for
// expression), but a taller tile: TY lines of nx with NP row pairs per thread.  These
// steps do 20-60 fp64 operations per row, so the template's per-plane-step costs (CTA
// barrier, ring bookkeeping, boundary tests, address arithmetic: ~100 issue slots per
// warp and plane for ONE row pair) bounded them at 67-75% of the HBM roofline under
// the power cap (profiles/r02e_spmv_tile.md, r02b_ncu_rr.md); with NP pairs per step
// they are spread over NP times the rows, and the y-halo lines staged per plane shrink
// from 2 per 2 lines to 2 per 2 NP lines.
#pragma once
#include "tile_sweeps.cuh"

// per mode: stencil operands (staged with halo lines), streamed vectors, outputs,
// dots, ring depths, row pairs per thread
template <int M> struct LtTraits;
template <> struct LtTraits<TM_SPB> { enum { NSV = 1, NST = 0, NOUT = 1, K = 0, SVR = 4, SD = 1, NP = 4 }; };
template <> struct LtTraits<TM_SPD> { enum { NSV = 1, NST = 0, NOUT = 1, K = 0, SVR = 4, SD = 1, NP = 4 }; };
#ifndef PBICG_RR_NP  // row pairs per thread of the replacement step (experiments: -D)
#define PBICG_RR_NP 2
#endif
template <> struct LtTraits<TM_RR1> { enum { NSV = 2, NST = 2, NOUT = 4, K = 3, SVR = 3, SD = 2, NP = PBICG_RR_NP }; };
template <> struct LtTraits<TM_RR2> { enum { NSV = 2, NST = 1, NOUT = 2, K = 5, SVR = 3, SD = 3, NP = PBICG_RR_NP }; };

struct SpmvGeo {
  int32_t TY, ncols, chunk, units, sv_stride, st_stride;
};

// MODE: TM_SPB (v_i from z_i), TM_SPD (t_{i+1} from w_{i+1}), TM_RR1, TM_RR2
template <int MODE>
__global__ void __launch_bounds__(TNT, 1) t_light3(TileGeo g, SpmvGeo q, Vecs V,
                                                   Scal* __restrict__ sc, Dd* __restrict__ part,
                                                   Hist h) {
  using T = LtTraits<MODE>;
  constexpr int NP = T::NP, NSV = T::NSV, NST = T::NST, SVR = T::SVR, SD = T::SD;
  constexpr int NOUT = T::NOUT, K = T::K > 0 ? T::K : 1;
  constexpr bool RR = MODE == TM_RR1 || MODE == TM_RR2;
  constexpr bool PREC = !RR;  // the SpMVs apply M^-1 per leg; RR1 / RR2 stage x, g / k, l
  static_assert(SVR + SD <= 8, "mbarriers in the 64-byte header");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Snap s_snap;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (MODE == TM_RR2 && threadIdx.x == 32) snap_load(s_snap, sc);
  if (sc->done) return;
  if (RR && !sc->rr_fire) return;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);  // [0, SVR) planes, [SVR, +SD) streams
  double* sv = reinterpret_cast<double*>(smem_raw + 64);
  double* st = sv + (size_t)SVR * NSV * q.sv_stride;
  const int tid = threadIdx.x;
  const int nx = (int)g.nx, svs = q.sv_stride, sts = q.st_stride, halo = (int)g.nx + 2;
  const int it = sc->iter;
  const double* svp[2] = {nullptr, nullptr};
  const double* stp[2] = {nullptr, nullptr};
  double* outp[4] = {nullptr, nullptr, nullptr, nullptr};
  if (MODE == TM_SPB) {
    svp[0] = (it & 1) ? V.z1 : V.z0;  // z_i as sweep A wrote it
    outp[0] = V.vv;
  } else if (MODE == TM_SPD) {
    svp[0] = sc->spd_par ? V.w1 : V.w0;  // w_{i+1}
    outp[0] = V.tv;
  } else if (MODE == TM_RR1) {  // r := b - A x, k := M^-1 r, s := A g, l := M^-1 s
    svp[0] = V.x; svp[1] = V.g;
    stp[0] = V.b; stp[1] = V.rh;
    outp[0] = V.r; outp[1] = V.k; outp[2] = V.s; outp[3] = V.l;
  } else {  // TM_RR2: w := A k, z := A l (k, l as RR1 stored them)
    svp[0] = V.k; svp[1] = V.l;
    stp[0] = V.rh;
    outp[0] = (it & 1) ? V.w0 : V.w1;  // w_{i+1}
    outp[1] = V.zrr;                   // replaced z_i (A26)
  }
  if (tid == 0) {
    for (int i = 0; i < SVR + SD; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  uint32_t ph = 0;
  int svc = 0, stc = 0;
  Dd acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = dd_zero();
  const double dinv = g.dinv;
  for (int u = blockIdx.x; u < q.units; u += gridDim.x) {
    const int col = u % q.ncols, qz = u / q.ncols;
    const int64_t y0 = (int64_t)col * q.TY;
    const int tyc = (int)((g.ny - y0) < q.TY ? (g.ny - y0) : q.TY);
    const int TP = tyc * nx;
    const int64_t z0 = (int64_t)qz * q.chunk;
    const int64_t z1 = (z0 + q.chunk) < g.nol ? (z0 + q.chunk) : g.nol;
    const int nst = (int)(z1 - z0), nsv = nst + 2;
    const int64_t toff = y0 * g.nx;
    // per pair p: row r = 2 tid + 2 TNT p of the tile, its boundary bits (constant over
    // the unit) and whether its warp is interior in x and y
    unsigned b0[NP], b1[NP];
    bool act[NP], act1[NP], xy_int[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int r = 2 * tid + 2 * TNT * p;
      act[p] = r < TP;
      act1[p] = r + 1 < TP;  // (nx even: always with act)
      const int x0 = r % nx, x1 = (r + 1) % nx;
      const int64_t gy0 = y0 + r / nx, gy1 = y0 + (r + 1) / nx;
      unsigned c0 = 0, c1 = 0;
      if (x0 > 0) c0 |= 4u;
      if (x0 < nx - 1) c0 |= 8u;
      if (x1 > 0) c1 |= 4u;
      if (x1 < nx - 1) c1 |= 8u;
      if (gy0 > 0) c0 |= 2u;
      if (gy0 < g.ny - 1) c0 |= 16u;
      if (gy1 > 0) c1 |= 2u;
      if (gy1 < g.ny - 1) c1 |= 16u;
      b0[p] = c0;
      b1[p] = c1;
      xy_int[p] = __all_sync(0xffffffffu, !act[p] || ((c0 & 30u) == 30u && (c1 & 30u) == 30u));
    }
    auto stage_sv = [&](int s, int64_t zp) {
      stage(sv + (size_t)s * NSV * svs, svs, svp, NSV, zp * g.pxy + toff - halo, TP + 2 * halo,
            &bar[s]);
    };
    auto stage_st = [&](int s, int64_t zp) {
      stage(st + (size_t)s * NST * sts, sts, stp, NST, zp * g.pxy + toff, TP, &bar[SVR + s]);
    };
    if (tid == 0) {
      for (int m = 0; m < SVR && m < nsv; ++m) stage_sv((svc + m) % SVR, z0 - 1 + m);
      if (NST > 0)
        for (int m = 0; m < SD - 1 && m < nst; ++m) stage_st((stc + m) % SD, z0 + m);
    }
    double m1[NP][NSV][2];
    {  // plane z0-1 -> registers; plane z0 resident
      const int s = svc % SVR;
      mbar_wait(&bar[s], (ph >> s) & 1u);
      ph ^= 1u << s;
      const double* bp = sv + (size_t)s * NSV * svs +
                         align_off(svp[0] + (z0 - 1) * g.pxy + toff - halo) + halo;
#pragma unroll
      for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int v = 0; v < NSV; ++v) {
          m1[p][v][0] = m1[p][v][1] = 0.0;
          if (act[p]) ld2<true>(bp + v * svs + 2 * tid + 2 * TNT * p, m1[p][v][0], m1[p][v][1]);
        }
      const int s1 = (svc + 1) % SVR;
      mbar_wait(&bar[s1], (ph >> s1) & 1u);
      ph ^= 1u << s1;
    }
    int k_new = svc % SVR, k_z = (svc + 1) % SVR, k_z1 = (svc + 2) % SVR;
    int k_st = stc % SD, k_stn = (stc + SD - 1) % SD;
    const int pstep = (int)(g.pxy & 1);
    const int ao0 = align_off(svp[0] + z0 * g.pxy + toff - halo);
    const int aos0 = NST > 0 ? align_off(stp[0] + z0 * g.pxy + toff) : 0;
    int64_t gz = z0 * g.pxy + toff;
    for (int n = 0; n < nst; ++n) {
      const int64_t z = z0 + n;
      if (n > 0) {
        k_new = k_new + 1 == SVR ? 0 : k_new + 1;
        k_z = k_z + 1 == SVR ? 0 : k_z + 1;
        k_z1 = k_z1 + 1 == SVR ? 0 : k_z1 + 1;
        k_st = k_st + 1 == SD ? 0 : k_st + 1;
        k_stn = k_stn + 1 == SD ? 0 : k_stn + 1;
        gz += g.pxy;
      }
      __syncthreads();  // step n-1 done: its plane-(z-1) slot and stream slot are free
      if (tid == 0) {
        if (n + SVR < nsv) stage_sv(k_new, z + SVR - 1);
        if (NST > 0 && n + SD - 1 < nst) stage_st(k_stn, z + SD - 1);
      }
      mbar_wait(&bar[k_z1], (ph >> k_z1) & 1u);
      ph ^= 1u << k_z1;
      if (NST > 0) {
        mbar_wait(&bar[SVR + k_st], (ph >> (SVR + k_st)) & 1u);
        ph ^= 1u << (SVR + k_st);
      }
      const int ov_z = (ao0 ^ (n & pstep)) + halo;
      const int ov_z1 = (ao0 ^ ((n + 1) & pstep)) + halo;
      const double* Wz = sv + (size_t)k_z * NSV * svs + ov_z;
      const double* Wz1 = sv + (size_t)k_z1 * NSV * svs + ov_z1;
      const double* S0 = st + (size_t)k_st * NST * sts + (aos0 ^ (n & pstep));
      const bool zin = (g.o0 + z) > 0 && (g.o0 + z) < g.nog - 1;
      const unsigned zb = ((g.o0 + z) > 0 ? 1u : 0u) | ((g.o0 + z) < g.nog - 1 ? 32u : 0u);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        if (!act[p]) continue;
        const int r = 2 * tid + 2 * TNT * p;
        double c[NSV][2], t[NSV][2];
#pragma unroll
        for (int v = 0; v < NSV; ++v) {
          if (xy_int[p] && zin)
            stencil_pair<3, true, 0u, PREC>(g, nx, Wz + v * svs + r, Wz1 + v * svs + r,
                                            m1[p][v][0], m1[p][v][1], 0u, 0u, c[v][0], c[v][1],
                                            t[v][0], t[v][1]);
          else if (zin)
            stencil_pair<3, true, 30u, PREC>(g, nx, Wz + v * svs + r, Wz1 + v * svs + r,
                                             m1[p][v][0], m1[p][v][1], b0[p], b1[p], c[v][0],
                                             c[v][1], t[v][0], t[v][1]);
          else
            stencil_pair<3, true, 63u, PREC>(g, nx, Wz + v * svs + r, Wz1 + v * svs + r,
                                             m1[p][v][0], m1[p][v][1], b0[p] | zb, b1[p] | zb,
                                             c[v][0], c[v][1], t[v][0], t[v][1]);
          m1[p][v][0] = c[v][0];
          m1[p][v][1] = c[v][1];
        }
        const int64_t gi = gz + r;
        double o0[NOUT], o1[NOUT];
        if (MODE == TM_SPB || MODE == TM_SPD) {
          o0[0] = t[0][0];
          o1[0] = t[0][1];
        } else if (MODE == TM_RR1) {  // tile_sweeps.cuh row_update<TM_RR1>, row by row
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (e == 1 && !act1[p]) break;
            double* o = e == 0 ? o0 : o1;
            const double bj = S0[r + e], rhj = S0[sts + r + e];
            const double rj = bj - t[0][e];    // r := b - A x
            o[0] = rj;
            o[1] = dinv * rj;                  // k := M^-1 r
            o[2] = t[1][e];                    // s := A g
            o[3] = dinv * t[1][e];             // l := M^-1 s
            dd_fma(acc[0], rhj, rj);           // (r^, r)
            dd_fma(acc[1 % K], rhj, t[1][e]);  // (r^, s)
            dd_fma(acc[2 % K], rj, rj);        // (r, r)
          }
        } else {  // TM_RR2
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (e == 1 && !act1[p]) break;
            double* o = e == 0 ? o0 : o1;
            const double rhj = S0[r + e];
            o[0] = t[0][e];                    // w := A k
            o[1 % NOUT] = t[1 % NSV][e];       // z := A l
            dd_fma(acc[1 % K], rhj, t[0][e]);  // (r^, w); slots 0, 2, 4 from RR1's stash
            dd_fma(acc[3 % K], rhj, t[1 % NSV][e]);
          }
        }
#pragma unroll
        for (int k = 0; k < NOUT; ++k)
          __stcs(reinterpret_cast<double2*>(outp[k] + gi), make_double2(o0[k], o1[k]));
      }
    }
    __syncthreads();  // unit done: every slot is free
    svc = (svc + nsv) % SVR;
    stc = (stc + nst) % SD;
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (MODE == TM_RR1) {  // each CTA's block totals of the three dots for RR2
    dd_block_reduce<K>(acc);
    if (tid == 0) {
#pragma unroll
      for (int j = 0; j < STASH_K; ++j) V.stash[(size_t)blockIdx.x * STASH_K + j] = acc[j];
    }
  } else if (MODE == TM_RR2) {  // dot slots 0, 2, 4 from the stash; reduction #2 (line 21)
    Dd tot[K];
    if (dd_grid_reduce<K, 0x15u>(acc, part, &sc->counter[T_RR2], tot, V.stash) && tid == 0)
      publish<F_RR2>(sc, h, tot, &s_snap);
  }
}

// host-side: shared-memory bytes of a t_light3<MODE> launch
template <int MODE>
inline size_t light_smem_bytes(const SpmvGeo& q) {
  using T = LtTraits<MODE>;
  return 64 + sizeof(double) * ((size_t)T::SVR * T::NSV * q.sv_stride +
                                (size_t)T::SD * T::NST * q.st_stride + 16);
}
