// spmv_tile.cuh -- the split schedule's stand-alone SpMVs on 3D stencils with the
// Jacobi preconditioner: v_i = A M^-1 z_i (Alg. 2 lines 13-14) and t_{i+1} =
// A M^-1 w_{i+1} (lines 22-23), option schedule 2 / the auto split schedule of
// small multi-GPU slabs.
//
// Same data movement as the TM_SPB / TM_SPD instances of t_tile (a ring of TMA-staged
// planes with one halo line on each side, the -z leg from registers) and the same
// arithmetic (stencil_pair: legs in ascending column order from +0.0, every leg
// fl(c * fl(dinv * v)) -- bitwise the template's results), but a taller tile: TY lines
// of nx with up to NP row pairs per thread.  A stand-alone SpMV does ~20 fp64 operations
// per row, so the template's per-plane-step costs (CTA barrier, ring bookkeeping,
// boundary tests, address arithmetic: ~100 issue slots per warp and plane for ONE row
// pair) bounded it at ~67% of the HBM roofline under the power cap (profiles/
// r02e_spmv_tile.md); with NP pairs per step they are spread over NP times the rows,
// and the y-halo lines staged per plane shrink from 2 per 2 lines to 2 per 2 NP lines.
#pragma once
#include "tile_sweeps.cuh"

#define SPT_SVR 4  // planes in the ring: z-1 .. z+2 (two in flight)

struct SpmvGeo {
  int32_t TY, ncols, chunk, units, sv_stride;
};

// MODE: TM_SPB (v_i from z_i) or TM_SPD (t_{i+1} from w_{i+1})
template <int MODE, int NP>
__global__ void __launch_bounds__(TNT, 1) t_spmv3(TileGeo g, SpmvGeo q, Vecs V,
                                                  const Scal* __restrict__ sc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (sc->done) return;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  double* sv = reinterpret_cast<double*>(smem_raw + 64);
  const int tid = threadIdx.x;
  const int nx = (int)g.nx, svs = q.sv_stride, halo = (int)g.nx + 2;
  const double* src = MODE == TM_SPB ? ((sc->iter & 1) ? V.z1 : V.z0)   // z_i as sweep A wrote it
                                     : (sc->spd_par ? V.w1 : V.w0);     // w_{i+1}
  double* const dst = MODE == TM_SPB ? V.vv : V.tv;
  if (tid == 0) {
    for (int i = 0; i < SPT_SVR; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  uint32_t ph = 0;
  int svc = 0;
  const double* srcs[1] = {src};
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
    bool act[NP], xy_int[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int r = 2 * tid + 2 * TNT * p;
      act[p] = r < TP;
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
      stage(sv + (size_t)s * svs, svs, srcs, 1, zp * g.pxy + toff - halo, TP + 2 * halo, &bar[s]);
    };
    if (tid == 0)
      for (int m = 0; m < SPT_SVR && m < nsv; ++m) stage_sv((svc + m) % SPT_SVR, z0 - 1 + m);
    double m1[NP][2];
    {  // plane z0-1 -> registers; plane z0 resident
      const int s = svc % SPT_SVR;
      mbar_wait(&bar[s], (ph >> s) & 1u);
      ph ^= 1u << s;
      const double* b = sv + (size_t)s * svs + align_off(src + (z0 - 1) * g.pxy + toff - halo) + halo;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        m1[p][0] = m1[p][1] = 0.0;
        if (act[p]) ld2<true>(b + 2 * tid + 2 * TNT * p, m1[p][0], m1[p][1]);
      }
      const int s1 = (svc + 1) % SPT_SVR;
      mbar_wait(&bar[s1], (ph >> s1) & 1u);
      ph ^= 1u << s1;
    }
    int k_new = svc % SPT_SVR, k_z = (svc + 1) % SPT_SVR, k_z1 = (svc + 2) % SPT_SVR;
    const int pstep = (int)(g.pxy & 1);
    const int ao0 = align_off(src + z0 * g.pxy + toff - halo);
    int64_t gz = z0 * g.pxy + toff;
    for (int n = 0; n < nst; ++n) {
      const int64_t z = z0 + n;
      if (n > 0) {
        k_new = k_new + 1 == SPT_SVR ? 0 : k_new + 1;
        k_z = k_z + 1 == SPT_SVR ? 0 : k_z + 1;
        k_z1 = k_z1 + 1 == SPT_SVR ? 0 : k_z1 + 1;
        gz += g.pxy;
      }
      __syncthreads();  // step n-1 done: its plane-(z-1) slot is free
      if (tid == 0 && n + SPT_SVR < nsv) stage_sv(k_new, z + SPT_SVR - 1);
      mbar_wait(&bar[k_z1], (ph >> k_z1) & 1u);
      ph ^= 1u << k_z1;
      const int ov_z = (ao0 ^ (n & pstep)) + halo;
      const int ov_z1 = (ao0 ^ ((n + 1) & pstep)) + halo;
      const double* Wz = sv + (size_t)k_z * svs + ov_z;
      const double* Wz1 = sv + (size_t)k_z1 * svs + ov_z1;
      const bool zin = (g.o0 + z) > 0 && (g.o0 + z) < g.nog - 1;
      const unsigned zb = ((g.o0 + z) > 0 ? 1u : 0u) | ((g.o0 + z) < g.nog - 1 ? 32u : 0u);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        if (!act[p]) continue;
        const int r = 2 * tid + 2 * TNT * p;
        double c0, c1, t0, t1;
        if (xy_int[p] && zin)
          stencil_pair<3, true, 0u, true>(g, nx, Wz + r, Wz1 + r, m1[p][0], m1[p][1], 0u, 0u, c0,
                                          c1, t0, t1);
        else if (zin)
          stencil_pair<3, true, 30u, true>(g, nx, Wz + r, Wz1 + r, m1[p][0], m1[p][1], b0[p],
                                           b1[p], c0, c1, t0, t1);
        else
          stencil_pair<3, true, 63u, true>(g, nx, Wz + r, Wz1 + r, m1[p][0], m1[p][1],
                                           b0[p] | zb, b1[p] | zb, c0, c1, t0, t1);
        m1[p][0] = c0;
        m1[p][1] = c1;
        __stcs(reinterpret_cast<double2*>(dst + gz + r), make_double2(t0, t1));
      }
    }
    __syncthreads();  // unit done: every slot is free
    svc = (svc + nsv) % SPT_SVR;
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// host-side: shared-memory bytes of a t_spmv3 launch
inline size_t spmv_smem_bytes(const SpmvGeo& q) {
  return 64 + sizeof(double) * ((size_t)SPT_SVR * q.sv_stride + 16);
}
