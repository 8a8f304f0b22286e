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
//   * outputs are written with streaming stores.
// Per row the kernels touch DRAM exactly once per vector (tile halos hit L2).
#pragma once
#include "dd.cuh"
#include "state.cuh"
#include "stencil_kernels.cuh"
#include "tma.cuh"

#define TNT 512      // threads per CTA
#define TKMAX 2      // row pairs per thread (TP <= 2 * TNT * TKMAX)
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

template <int DIM>
__device__ __forceinline__ double tile_stencil(const TileGeo& g, const double* sz, const double* sz1,
                                               int ci, double vzm, unsigned bnd) {
  // bnd bits: 0 zm, 1 ym, 2 xm, 3 xp, 4 yp, 5 zp; legs ascending column (A5)
  const double d = g.dinv;
  double acc = 0.0;
  acc = (bnd & 1u) ? acc + g.c[DIM == 3 ? 5 : 3] * (d * vzm) : acc;
  if (DIM == 3) acc = (bnd & 2u) ? acc + g.c[3] * (d * sz[ci - g.nx]) : acc;
  acc = (bnd & 4u) ? acc + g.c[1] * (d * sz[ci - 1]) : acc;
  acc = acc + g.c[0] * (d * sz[ci]);
  acc = (bnd & 8u) ? acc + g.c[2] * (d * sz[ci + 1]) : acc;
  if (DIM == 3) acc = (bnd & 16u) ? acc + g.c[4] * (d * sz[ci + g.nx]) : acc;
  acc = (bnd & 32u) ? acc + g.c[DIM == 3 ? 6 : 4] * (d * sz1[ci]) : acc;
  return acc;
}

// MODE 0 = sweepA (lines 5-12), MODE 1 = sweepC (lines 17-21)
template <int DIM, int MODE>
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

  const int it = sc->iter;
  const double al = sc->alpha, be = sc->beta, om = sc->omega;
  const bool rr = MODE == 0 && sc->use_rr != 0;
  // vector roles
  const double* svp[2];
  const double* stp[NSTR_MAX];
  int nstr;
  double* zout = nullptr;
  if (MODE == 0) {
    svp[0] = (it & 1) ? V.w1 : V.w0;                 // w_i
    svp[1] = (it & 1) ? V.z0 : V.z1;                 // z_{i-1} pre-replacement
    stp[0] = V.k; stp[1] = V.g; stp[2] = V.l; stp[3] = V.s; stp[4] = V.r;
    stp[NSTR_MAX - 1] = V.zrr;                       // z_{i-1} replaced (A26)
    nstr = rr ? 6 : 5;
    zout = (it & 1) ? V.z1 : V.z0;                   // z_i
  } else {
    svp[0] = (it & 1) ? V.w1 : V.w0;                 // w_i
    svp[1] = (it & 1) ? V.z1 : V.z0;                 // z_i
    stp[0] = V.x; stp[1] = V.g; stp[2] = V.k; stp[3] = V.l; stp[4] = V.r; stp[5] = V.s;
    stp[NSTR_MAX - 1] = V.rh;
    nstr = 7;
    zout = (it & 1) ? V.w0 : V.w1;                   // w_{i+1}
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

  for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
    const int col = u % g.ncols, q = u / g.ncols;
    const int64_t y0 = (int64_t)col * g.TY;
    const int tyc = (int)((g.ny - y0) < g.TY ? (g.ny - y0) : g.TY);
    const int TP = tyc * (int)g.nx;
    const int64_t z0 = (int64_t)q * g.chunk;
    const int64_t z1 = (z0 + g.chunk) < g.nol ? (z0 + g.chunk) : g.nol;
    const int nst = (int)(z1 - z0), nsv = nst + 2;
    const int64_t toff = DIM == 3 ? y0 * g.nx : 0;
    // per-row setup (constant over the unit)
    unsigned bnd[2 * TKMAX];
    int rowi[2 * TKMAX];
#pragma unroll
    for (int k = 0; k < 2 * TKMAX; ++k) {
      const int r = 2 * (tid + TNT * (k >> 1)) + (k & 1);
      rowi[k] = r;
      const int xx = r % (int)g.nx;
      const int64_t gy = y0 + r / (int)g.nx;
      unsigned b = 0;
      if (xx > 0) b |= 4u;
      if (xx < g.nx - 1) b |= 8u;
      if (DIM == 3) {
        if (gy > 0) b |= 2u;
        if (gy < g.ny - 1) b |= 16u;
      }
      bnd[k] = r < TP ? b : 0xffffffffu;  // all ones = inactive row
    }
    double m1[2][2 * TKMAX];  // -z neighbours (previous plane centre), per stencil vector
    // prologue: stencil planes z0-1, z0, z0+1; streams z0
    if (tid == 0) {
      for (int m = 0; m < 3 && m < nsv; ++m) {
        const int s = (svc + m) % 3;
        stage(sv + (size_t)s * 2 * g.sv_stride, g.sv_stride, svp, 2,
              (z0 - 1 + m) * g.pxy + toff - g.halo, TP + 2 * g.halo, &bar[2 + s]);
      }
      const int s = stc % 2;
      stage(st + (size_t)s * NSTR_MAX * g.st_stride, g.st_stride, stp, nstr, z0 * g.pxy + toff,
            TP, &bar[s]);
    }
    {  // plane z0-1 -> registers
      const int s = svc % 3;
      mbar_wait(&bar[2 + s], (ph >> (2 + s)) & 1u);
      ph ^= 1u << (2 + s);
      const double* b0 = sv + (size_t)s * 2 * g.sv_stride;
      const int o = align_off(svp[0] + (z0 - 1) * g.pxy + toff - g.halo) + g.halo;
#pragma unroll
      for (int k = 0; k < 2 * TKMAX; ++k) {
        if (bnd[k] != 0xffffffffu) {
          m1[0][k] = b0[o + rowi[k]];
          m1[1][k] = b0[g.sv_stride + o + rowi[k]];
        } else {
          m1[0][k] = m1[1][k] = 0.0;
        }
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
          stage(sv + (size_t)s * 2 * g.sv_stride, g.sv_stride, svp, 2,
                (z + 2) * g.pxy + toff - g.halo, TP + 2 * g.halo, &bar[2 + s]);
        }
        if (n + 1 < nst) {  // streams z+1
          const int s = (stc + n + 1) % 2;
          stage(st + (size_t)s * NSTR_MAX * g.st_stride, g.st_stride, stp, nstr,
                (z + 1) * g.pxy + toff, TP, &bar[s]);
        }
      }
      const int s_z = (svc + n + 1) % 3, s_z1 = (svc + n + 2) % 3, s_st = (stc + n) % 2;
      mbar_wait(&bar[2 + s_z1], (ph >> (2 + s_z1)) & 1u);
      ph ^= 1u << (2 + s_z1);
      mbar_wait(&bar[s_st], (ph >> s_st) & 1u);
      ph ^= 1u << s_st;
      const double* Wz = sv + (size_t)s_z * 2 * g.sv_stride;
      const double* Zz = Wz + g.sv_stride;
      const double* Wz1 = sv + (size_t)s_z1 * 2 * g.sv_stride;
      const double* Zz1 = Wz1 + g.sv_stride;
      const double* S0 = st + (size_t)s_st * NSTR_MAX * g.st_stride;
      const int oz = align_off(svp[0] + z * g.pxy + toff - g.halo) + g.halo;
      const int oz1 = align_off(svp[0] + (z + 1) * g.pxy + toff - g.halo) + g.halo;
      const int os = align_off(stp[0] + z * g.pxy + toff);
      const unsigned zb = ((g.o0 + z) > 0 ? 1u : 0u) | ((g.o0 + z) < g.nog - 1 ? 32u : 0u);
      const int64_t gbase = z * g.pxy + toff;
#pragma unroll
      for (int k = 0; k < 2 * TKMAX; ++k) {
        if (bnd[k] == 0xffffffffu) continue;
        const int r = rowi[k];
        const unsigned b = bnd[k] | zb;
        const int ci = oz + r, ci1 = oz1 + r, si = os + r;
        const double wc = Wz[ci], zc = Zz[ci];
        // same z+1 index shift: plane z+1 staged with its own alignment offset
        const double t = tile_stencil<DIM>(g, Wz, Wz1 + (ci1 - ci), ci, m1[0][k], b);
        const double v = tile_stencil<DIM>(g, Zz, Zz1 + (ci1 - ci), ci, m1[1][k], b);
        m1[0][k] = wc;
        m1[1][k] = zc;
        const int64_t gi = gbase + r;
        if (MODE == 0) {
          const double kj = S0[si], gj = S0[g.st_stride + si], lj = S0[2 * g.st_stride + si];
          const double sj = S0[3 * g.st_stride + si], rj = S0[4 * g.st_stride + si];
          const double zoc = rr ? S0[(NSTR_MAX - 1) * g.st_stride + si] : zc;
          const double m = g.dinv * wc;
          const double nn = g.dinv * zc;
          const double gn = kj + be * (gj - om * lj);    // line 5
          const double sn = wc + be * (sj - om * zoc);   // line 6
          const double ln = m + be * (lj - om * nn);     // line 7
          const double zz = t + be * (zoc - om * v);     // line 8
          const double qq = rj - al * sn;                // line 9
          const double yy = wc - al * zz;                // line 11
          dd_fma(acc[0], qq, yy);                        // line 12
          dd_fma(acc[1 % K], yy, yy);
          __stcs(V.g + gi, gn);
          __stcs(V.s + gi, sn);
          __stcs(V.l + gi, ln);
          __stcs(zout + gi, zz);
        } else {
          const double xj = S0[si], gj = S0[g.st_stride + si], kj = S0[2 * g.st_stride + si];
          const double lj = S0[3 * g.st_stride + si], rj = S0[4 * g.st_stride + si];
          const double sj = S0[5 * g.st_stride + si], rhj = S0[6 * g.st_stride + si];
          const double m = g.dinv * wc;
          const double nn = g.dinv * zc;
          const double uu = kj - al * lj;                // line 10
          const double qq = rj - al * sj;                // line 9
          const double yy = wc - al * zc;                // line 11
          const double xn = (xj + al * gj) + om * uu;    // line 17
          const double rn = qq - om * yy;                // line 18
          const double kn = uu - om * (m - al * nn);     // line 19
          const double wn = yy - om * (t - al * v);      // line 20
          dd_fma(acc[0], rhj, rn);                       // line 21
          dd_fma(acc[1 % K], rhj, wn);
          dd_fma(acc[2 % K], rhj, sj);
          dd_fma(acc[3 % K], rhj, zc);
          dd_fma(acc[4 % K], rn, rn);
          __stcs(V.x + gi, xn);
          __stcs(V.r + gi, rn);
          __stcs(V.k + gi, kn);
          __stcs(zout + gi, wn);
        }
      }
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
