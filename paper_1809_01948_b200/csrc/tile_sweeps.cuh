// tile_sweeps.cuh -- every step of the stencil path as a TMA-staged 2.5D
// z-marching kernel (the hot path on B200).
//
// Same arithmetic, same operation order as the line kernels of
// stencil_kernels.cuh -- only the data movement differs:
//   * a CTA owns a tile of TY full x-lines of a plane (3D) or one x-line (2D)
//     and marches the outer dimension (z in 3D, y in 2D) over a chunk of planes;
//   * one elected thread streams every vector the step needs into shared memory
//     with cp.async.bulk (TMA bulk copies) one plane ahead, completion tracked by
//     mbarriers, so ~100 KB per SM is in flight while the CTA computes;
//   * the stencil operands (w and z in the sweeps; x, g / r, s in the
//     replacement; x or r in init and gap) are staged as planes with one halo
//     line on each side (a ring of SvDepth slots, 3 by default: z, z+1 resident,
//     z+2 in flight); the -z leg comes from registers (the previous step's centre
//     values);
//   * block Jacobi b >= 4: a transform stage overwrites each landed plane with
//     M^-1 v once (xf_pair), then a plain stencil runs;
//   * peer-memory transport: sweeps A / C also store their slab's boundary planes
//     into the neighbours' ghost planes (Vecs::hz / hw);
//   * one row pair per thread; 16-byte shared loads / global streaming stores
//     when nx is even; a warp-uniform interior path drops the boundary selects.
// Per row the kernels touch DRAM exactly once per vector (tile halos hit L2).
//
// Modes (Alg. 2 lines):
//   TM_A    sweep A, lines 5-12          TM_C    sweep C, lines 16-21
//   TM_RR1  eq:rr r, k, s, l TM_RR2  eq:rr w, z + line-21 dots
//   TM_GAP  eq:res_gap           TM_INIT1 / TM_INIT2  lines 2-3
// Comparison solvers on the same machinery:
//   TM_CL1  Alg. 1 line 17 + lines 4-6: p := r + beta (p - omega s),
//           s := A M^-1 p, (r^0, s)     -- stencil of the DERIVED operand p
//   TM_CL2  Alg. 1 lines 8-11: q := r - alpha s (derived), y := A M^-1 q,
//           (q, y), (y, y)              -- reads r, s only, writes nothing
//   TM_CL3  Alg. 1 lines 13-15: x, r; (r^0, r), (r, r)
//   TM_PC   p-CG iteration (reading A19): n := A M^-1 w, z, q, s, p, x, r, u, w;
//           next iteration's (r, u), (w, u), (r, r)
//   TM_PCI1 / TM_PCI2  p-CG init: r0, u0; w0 := A M^-1 r0, (r0, u0), (w0, u0)
// A DERIVED mode stages NSV vectors with halos and applies the stencil to one
// operand formed from them element by element (derive<MODE>), so the operand is
// never written to HBM; it is formed with the same operations as the oracle's
// stored vector, hence bitwise equal.
#pragma once

#include "dd.cuh"
#include "state.cuh"
#include "stencil_kernels.cuh"
#include "tma.cuh"


#define TNT 512  // threads per CTA

enum TileMode { TM_A = 0, TM_C, TM_RR1, TM_RR2, TM_GAP, TM_INIT1, TM_INIT2,
                TM_CL1, TM_CL2, TM_CL3, TM_PC, TM_PCI1, TM_PCI2,
                // the same steps plus the vector norms of the automated-replacement
                // bound f^r: sums of squares ride the step's reduction
                TM_AN, TM_CN, TM_RR1N, TM_RR2N, TM_INIT1N,
                // split schedule (option schedule 2): the stand-alone SpMVs
                TM_SPB, TM_SPD, TM_N };

template <int M> struct BaseOf { enum { v = M }; };
template <> struct BaseOf<TM_AN> { enum { v = TM_A }; };
template <> struct BaseOf<TM_CN> { enum { v = TM_C }; };
template <> struct BaseOf<TM_RR1N> { enum { v = TM_RR1 }; };
template <> struct BaseOf<TM_RR2N> { enum { v = TM_RR2 }; };
template <> struct BaseOf<TM_INIT1N> { enum { v = TM_INIT1 }; };

// per mode: staged stencil vectors (NSV), whether they form ONE derived operand
// (DER), whether the operand enters as A M^-1 v (PREC) or A v, the maximum number
// of streamed vectors, outputs, dot products
template <int M> struct TileTraits;
template <> struct TileTraits<TM_A> { enum { NSV = 2, DER = 0, PREC = 1, NSTR = 5, NOUT = 4, K = 2 }; };
template <> struct TileTraits<TM_C> { enum { NSV = 2, DER = 0, PREC = 1, NSTR = 7, NOUT = 4, K = 5 }; };
template <> struct TileTraits<TM_RR1> { enum { NSV = 2, DER = 0, PREC = 0, NSTR = 2, NOUT = 4, K = 3 }; };
template <> struct TileTraits<TM_RR2> { enum { NSV = 2, DER = 0, PREC = 0, NSTR = 1, NOUT = 2, K = 5 }; };
template <> struct TileTraits<TM_GAP> { enum { NSV = 1, DER = 0, PREC = 0, NSTR = 2, NOUT = 0, K = 1 }; };
template <> struct TileTraits<TM_INIT1> { enum { NSV = 1, DER = 0, PREC = 0, NSTR = 1, NOUT = 3, K = 2 }; };
template <> struct TileTraits<TM_INIT2> { enum { NSV = 1, DER = 0, PREC = 1, NSTR = 1, NOUT = 1, K = 1 }; };
template <> struct TileTraits<TM_CL1> { enum { NSV = 3, DER = 1, PREC = 1, NSTR = 1, NOUT = 2, K = 1 }; };
template <> struct TileTraits<TM_CL2> { enum { NSV = 2, DER = 1, PREC = 1, NSTR = 0, NOUT = 0, K = 2 }; };
template <> struct TileTraits<TM_CL3> { enum { NSV = 2, DER = 1, PREC = 1, NSTR = 3, NOUT = 2, K = 2 }; };
template <> struct TileTraits<TM_PC> { enum { NSV = 1, DER = 0, PREC = 1, NSTR = 7, NOUT = 8, K = 3 }; };
template <> struct TileTraits<TM_PCI1> { enum { NSV = 1, DER = 0, PREC = 0, NSTR = 1, NOUT = 2, K = 2 }; };
template <> struct TileTraits<TM_PCI2> { enum { NSV = 1, DER = 0, PREC = 1, NSTR = 0, NOUT = 1, K = 2 }; };
// + norms: A: k, w, m, t, g, s, l, z, q, y; C: x, u, n, v; RR1: x, k, s, l; RR2: z;
// INIT1: x0, k0
template <> struct TileTraits<TM_AN> { enum { NSV = 2, DER = 0, PREC = 1, NSTR = 5, NOUT = 4, K = 12 }; };

// Depth of the streamed-vector ring (planes in shared memory: the current one +
// SD-1 in flight).  Sweep A streams only 5 vectors, so it fits a third slot and
// keeps two planes of them in flight -- the bytes in flight its 13-pass budget
// needs to run at the copy rate when the power cap lowers the SM clock.
template <int M> struct StreamDepth { enum { v = 2 }; };
template <> struct StreamDepth<TM_A> { enum { v = 3 }; };
template <> struct StreamDepth<TM_AN> { enum { v = 3 }; };
template <> struct StreamDepth<TM_CL3> { enum { v = 3 }; };  // measured: CL3 +4%; CL1, PC: no gain
// Depth of the stencil-plane ring (planes z, z+1 resident, the rest in flight).  The
// stand-alone SpMV tiles of the split schedule stream nothing else and do little work
// per plane: a 6-slot ring keeps four planes in flight per CTA.
template <int M> struct SvDepth { enum { v = 3 }; };
template <> struct SvDepth<TM_SPB> { enum { v = 6 }; };
template <> struct SvDepth<TM_SPD> { enum { v = 6 }; };
// The replacement and init steps stream one or two vectors per plane next to two
// staged operands: a 4-deep stencil ring and a 3-deep stream ring keep two planes in
// flight (measured, cfg4: rr1 78% -> 90%, init 66% -> 72% of HBM; a 5-deep ring adds
// nothing; the gap step loses with it, so it keeps the default)
template <> struct SvDepth<TM_RR1> { enum { v = 4 }; };
template <> struct SvDepth<TM_RR2> { enum { v = 4 }; };
template <> struct SvDepth<TM_RR1N> { enum { v = 4 }; };
template <> struct SvDepth<TM_RR2N> { enum { v = 4 }; };
template <> struct SvDepth<TM_INIT1> { enum { v = 4 }; };
template <> struct SvDepth<TM_INIT2> { enum { v = 4 }; };
template <> struct SvDepth<TM_INIT1N> { enum { v = 4 }; };
template <> struct StreamDepth<TM_RR1> { enum { v = 3 }; };
template <> struct StreamDepth<TM_RR2> { enum { v = 3 }; };
template <> struct StreamDepth<TM_RR1N> { enum { v = 3 }; };
template <> struct StreamDepth<TM_RR2N> { enum { v = 3 }; };
template <> struct StreamDepth<TM_INIT1> { enum { v = 3 }; };
template <> struct StreamDepth<TM_INIT2> { enum { v = 3 }; };
template <> struct StreamDepth<TM_INIT1N> { enum { v = 3 }; };

// The line-21 dots after a replacement (eq:rr, then P:187): (r^, r), (r^, s)
// and (r, r) need only the replaced r and s, which RR1 forms -- RR1 accumulates them
// (w: it streams r^ too) and stores each CTA's block totals (Vecs::stash); RR2 (r: it
// forms w = A k and z = A l from the stored k = M^-1 r, l = M^-1 s, so its stencils need
// no M^-1) accumulates only (r^, w), (r^, z) and takes the other three block totals from
// the stash into dot slots 0, 2, 4 before its grid reduction.  Same rows, same thread
// order, same per-value block tree (dd_block_reduce) and the same grid: the totals are
// the bits the one-kernel form gives.  RR2 is then no longer fp64-issue-bound.
template <int M> struct Stash { enum { w = 0, r = 0 }; };
template <> struct Stash<TM_RR1> { enum { w = 1, r = 0 }; };
template <> struct Stash<TM_RR1N> { enum { w = 1, r = 0 }; };
template <> struct Stash<TM_RR2> { enum { w = 0, r = 1 }; };
template <> struct Stash<TM_RR2N> { enum { w = 0, r = 1 }; };
#define STASH_K 3  // stashed dots per CTA
template <> struct TileTraits<TM_CN> { enum { NSV = 2, DER = 0, PREC = 1, NSTR = 7, NOUT = 4, K = 9 }; };
template <> struct TileTraits<TM_RR1N> { enum { NSV = 2, DER = 0, PREC = 0, NSTR = 2, NOUT = 4, K = 7 }; };
template <> struct TileTraits<TM_RR2N> { enum { NSV = 2, DER = 0, PREC = 0, NSTR = 1, NOUT = 2, K = 6 }; };
template <> struct TileTraits<TM_INIT1N> { enum { NSV = 1, DER = 0, PREC = 0, NSTR = 1, NOUT = 3, K = 4 }; };
template <> struct TileTraits<TM_SPB> { enum { NSV = 1, DER = 0, PREC = 1, NSTR = 0, NOUT = 1, K = 0 }; };
template <> struct TileTraits<TM_SPD> { enum { NSV = 1, DER = 0, PREC = 1, NSTR = 0, NOUT = 1, K = 0 }; };

// sum of squares for a bound norm: Dot2 (v, v) like every other dot (reading A30), so
// the bound f^r and the replacement decisions are the oracle's bitwise
__device__ __forceinline__ void nrm_add(Dd& a, double v) { dd_fma(a, v, v); }

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
  int32_t bj;         // preconditioner: 1 Jacobi; 2, 4, 8 block Jacobi along x (reading A33)
  double bi[64];      // bj > 1: the (common) bj x bj inverse block, row-major
  // x-segmented tiles (grids with nx > 1024, nx even): a tile is TY lines x sx columns
  int32_t sx;         // segment width (even); == nx when lines are not segmented
  int32_t nseg;       // segments per line
  int32_t lstride;    // shared-memory stride of a staged stencil line segment (sx + 16)
  int32_t pdl;        // launch with programmatic dependent launch (option "pdl")
  int32_t peer;       // sweeps A / C store their boundary planes in the neighbours (Vecs::hz/hw)
};

// halo columns staged on each side of a segment (>= 2 for the x legs; 8 keeps every
// staged line 16-byte aligned for any even x0)
#define SEG_HX 8

// stage `n` vectors' line segments: nl lines of len doubles starting at element e0
// (line stride nx in global memory, ls in shared memory); every range is 16-byte
// aligned by construction (nx, e0, len even)
__device__ __forceinline__ void stage_lines(double* dst, int stride, const double* const* src,
                                            int n, int64_t e0, int64_t nx, int nl, int len,
                                            int ls, uint64_t* bar) {
  const uint32_t bytes = (uint32_t)len * 8u;
  mbar_arrive_expect_tx(bar, bytes * (uint32_t)(n * nl));
  for (int v = 0; v < n; ++v)
    for (int l = 0; l < nl; ++l)
      bulk_g2s(dst + (size_t)v * stride + (size_t)l * ls, src[v] + e0 + (int64_t)l * nx, bytes,
               bar);
}

__device__ __forceinline__ int align_off(const double* p) {
  return (int)(((uintptr_t)p & 15u) >> 3);
}

// stage `n` vectors' element range [e0, e0 + len) into dst slots
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

// the same with a mask of the legs that may be dropped (DROP: boundary bits checked;
// legs outside it are always present for the warp)
template <unsigned DROP>
__device__ __forceinline__ double legm(unsigned b, unsigned bit, double acc, double term) {
  return ((DROP & bit) == 0u || (b & bit)) ? acc + term : acc;
}

template <bool PREC>
__device__ __forceinline__ double pre(double d, double v) {
  return PREC ? d * v : v;
}

// fl(A M^-1 v) (PREC) or fl(A v) for the row pair (r, r+1) of plane z.  W points
// at row r of plane z in shared memory, W1 at row r of plane z+1; m0/m1 are the
// plane z-1 centre values.  Legs in ascending column order (A5), added left to
// right from +0.0; with PREC every leg is fl(c * fl(dinv * v)), exactly the
// oracle's "n := M^-1 z; v := A n".  Products shared by the two rows are formed
// once (same values).  bnd bits: 1 zm, 2 ym, 4 xm, 8 xp, 16 yp, 32 zp.
template <int DIM, bool VEC, unsigned DROP, bool PREC>
__device__ __forceinline__ void stencil_pair(const TileGeo& g, int nx, const double* W,
                                             const double* W1, double zm0, double zm1,
                                             unsigned b0, unsigned b1, double& c0, double& c1,
                                             double& t0, double& t1) {
  const double d = g.dinv;
  ld2<VEC>(W, c0, c1);
  const double pm = pre<PREC>(d, W[-1]), p0 = pre<PREC>(d, c0), p1 = pre<PREC>(d, c1);
  const double p2 = pre<PREC>(d, W[2]);
  double ym0 = 0.0, ym1 = 0.0, yp0 = 0.0, yp1 = 0.0, zp0, zp1;
  if (DIM == 3) {
    ld2<VEC>(W - nx, ym0, ym1);
    ld2<VEC>(W + nx, yp0, yp1);
  }
  ld2<VEC>(W1, zp0, zp1);
  const double czm = g.c[DIM == 3 ? 5 : 3], czp = g.c[DIM == 3 ? 6 : 4];
  double a = 0.0;
  a = legm<DROP>(b0, 1u, a, czm * pre<PREC>(d, zm0));
  if (DIM == 3) a = legm<DROP>(b0, 2u, a, g.c[3] * pre<PREC>(d, ym0));
  a = legm<DROP>(b0, 4u, a, g.c[1] * pm);
  a = a + g.c[0] * p0;
  a = legm<DROP>(b0, 8u, a, g.c[2] * p1);
  if (DIM == 3) a = legm<DROP>(b0, 16u, a, g.c[4] * pre<PREC>(d, yp0));
  a = legm<DROP>(b0, 32u, a, czp * pre<PREC>(d, zp0));
  t0 = a;
  a = 0.0;
  a = legm<DROP>(b1, 1u, a, czm * pre<PREC>(d, zm1));
  if (DIM == 3) a = legm<DROP>(b1, 2u, a, g.c[3] * pre<PREC>(d, ym1));
  a = legm<DROP>(b1, 4u, a, g.c[1] * p0);
  a = a + g.c[0] * p1;
  a = legm<DROP>(b1, 8u, a, g.c[2] * p2);
  if (DIM == 3) a = legm<DROP>(b1, 16u, a, g.c[4] * pre<PREC>(d, yp1));
  a = legm<DROP>(b1, 32u, a, czp * pre<PREC>(d, zp1));
  t1 = a;
}

// ---------------------------------------------------------------------------
// Block Jacobi on the stencil path (reading A33): blocks of bj consecutive x
// points (nx % bj == 0), all with the same bj x bj matrix (constant coefficients,
// the -x/+x legs inside a block always exist), so one inverse g.bi serves every
// block.  (M^-1 v)_i = sum_k bi[i][k] v_k, ascending k from +0.0 (the oracle's order).
// B: the block size as a template constant (2, 4, 8); bi: the inverse block staged
// in shared memory (row-major B x B); rows are picked by the thread's position.
template <int B>
__device__ __forceinline__ double bj_row(const double* bi, int i, const double* P) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < B; ++k) acc = acc + bi[i * B + k] * P[k];
  return acc;
}

// rows i0, i0+1 of the block at P (loaded once)
template <int B, bool VEC>
__device__ __forceinline__ void bj_pair(const double* bi, int i0, const double* P, double& a,
                                        double& c) {
  double v[B];
#pragma unroll
  for (int k = 0; k < B; k += 2) ld2<VEC>(P + k, v[k], v[k + 1]);
  double x = 0.0, y = 0.0;
#pragma unroll
  for (int k = 0; k < B; ++k) {
    x = x + bi[i0 * B + k] * v[k];
    y = y + bi[(i0 + 1) * B + k] * v[k];
  }
  a = x;
  c = y;
}

// stencil_pair with M^-1 = block Jacobi: raw centre pair (c0, c1), preconditioned
// centre pair (pc0, pc1) and fl(A M^-1 v) for the row pair (r, r+1); i0 = x % B
// of row r (even).  zm0/zm1 are the PRECONDITIONED values of plane z-1.  Legs as
// in stencil_pair (A5); a dropped leg's value may be read past the line but is
// never added.
template <int DIM, bool VEC, unsigned DROP, int B>
__device__ __forceinline__ void stencil_pair_bj(const TileGeo& g, const double* bi, int nx, int i0,
                                                const double* W, const double* W1, double zm0,
                                                double zm1, unsigned b0, unsigned b1, double& c0,
                                                double& c1, double& pc0, double& pc1, double& t0,
                                                double& t1) {
  const double* blk = W - i0;  // element 0 of this pair's block (16-byte aligned: i0, B even)
  double v[B];
#pragma unroll
  for (int k = 0; k < B; k += 2) ld2<VEC>(blk + k, v[k], v[k + 1]);
  c0 = v[0];
  c1 = v[1];
  if (B > 2) {  // the raw centre pair sits at i0, i0+1 of the block
    ld2<VEC>(W, c0, c1);
  }
  double x0 = 0.0, x1 = 0.0, xm = 0.0, xp = 0.0;
#pragma unroll
  for (int k = 0; k < B; ++k) {
    x0 = x0 + bi[i0 * B + k] * v[k];
    x1 = x1 + bi[(i0 + 1) * B + k] * v[k];
  }
  pc0 = x0;
  pc1 = x1;
  if (i0 > 0) {  // x-1 inside this block
#pragma unroll
    for (int k = 0; k < B; ++k) xm = xm + bi[(i0 - 1) * B + k] * v[k];
  } else {
    xm = bj_row<B>(bi, B - 1, blk - B);
  }
  if (i0 + 2 < B) {  // x+2 inside this block
#pragma unroll
    for (int k = 0; k < B; ++k) xp = xp + bi[(i0 + 2) * B + k] * v[k];
  } else {
    xp = bj_row<B>(bi, 0, blk + B);
  }
  double ym0 = 0.0, ym1 = 0.0, yp0 = 0.0, yp1 = 0.0, zp0, zp1;
  if (DIM == 3) {
    bj_pair<B, VEC>(bi, i0, blk - nx, ym0, ym1);
    bj_pair<B, VEC>(bi, i0, blk + nx, yp0, yp1);
  }
  bj_pair<B, VEC>(bi, i0, W1 - i0, zp0, zp1);
  const double czm = g.c[DIM == 3 ? 5 : 3], czp = g.c[DIM == 3 ? 6 : 4];
  double a = 0.0;
  a = legm<DROP>(b0, 1u, a, czm * zm0);
  if (DIM == 3) a = legm<DROP>(b0, 2u, a, g.c[3] * ym0);
  a = legm<DROP>(b0, 4u, a, g.c[1] * xm);
  a = a + g.c[0] * pc0;
  a = legm<DROP>(b0, 8u, a, g.c[2] * pc1);
  if (DIM == 3) a = legm<DROP>(b0, 16u, a, g.c[4] * yp0);
  a = legm<DROP>(b0, 32u, a, czp * zp0);
  t0 = a;
  a = 0.0;
  a = legm<DROP>(b1, 1u, a, czm * zm1);
  if (DIM == 3) a = legm<DROP>(b1, 2u, a, g.c[3] * ym1);
  a = legm<DROP>(b1, 4u, a, g.c[1] * pc0);
  a = a + g.c[0] * pc1;
  a = legm<DROP>(b1, 8u, a, g.c[2] * xp);
  if (DIM == 3) a = legm<DROP>(b1, 16u, a, g.c[4] * yp1);
  a = legm<DROP>(b1, 32u, a, czp * zp1);
  t1 = a;
}

// (M^-1 v) for the pair of row values (v0, v1) held by this thread when the block's
// other values sit in the neighbouring lanes (RR1 / INIT1 form r = b - A x per row)
template <int B>
__device__ __forceinline__ void bj_pair_shfl(const double* bi, unsigned mask, int i0, double v0,
                                             double v1, double& o0, double& o1) {
  const int base = (threadIdx.x & 31) - i0 / 2;  // lane holding block elements 0, 1
  double a = 0.0, c = 0.0;
#pragma unroll
  for (int k = 0; k < B; k += 2) {
    const double e0 = __shfl_sync(mask, v0, base + k / 2);
    const double e1 = __shfl_sync(mask, v1, base + k / 2);
    a = a + bi[i0 * B + k] * e0;
    a = a + bi[i0 * B + k + 1] * e1;
    c = c + bi[(i0 + 1) * B + k] * e0;
    c = c + bi[(i0 + 1) * B + k + 1] * e1;
  }
  o0 = a;
  o1 = c;
}

// The derived operand of a DERIVED mode from the staged values v[0..NSV-1] of
// one element (same expression, same order as the oracle's stored vector).
template <int MODE>
__device__ __forceinline__ double derive(double v0, double v1, double v2, double al, double be,
                                         double om) {
  if (MODE == TM_CL1) return v0 + be * (v1 - om * v2);  // Alg. 1 l.17: r + beta (p - omega s)
  return v0 - al * v1;                                  // Alg. 1 l.8: q := r - alpha s
}

// derived values of the element pair at P (vector k at P + k * svs)
template <bool VEC, int NSV, int MODE>
__device__ __forceinline__ void derive_pair(const double* P, int svs, double al, double be,
                                            double om, double& a, double& b) {
  double a0, b0, a1 = 0.0, b1 = 0.0, a2 = 0.0, b2 = 0.0;
  ld2<VEC>(P, a0, b0);
  if (NSV > 1) ld2<VEC>(P + svs, a1, b1);
  if (NSV > 2) ld2<VEC>(P + 2 * svs, a2, b2);
  a = derive<MODE>(a0, a1, a2, al, be, om);
  b = derive<MODE>(b0, b1, b2, al, be, om);
}

template <int NSV, int MODE>
__device__ __forceinline__ double derive_one(const double* P, int svs, double al, double be,
                                             double om) {
  return derive<MODE>(P[0], NSV > 1 ? P[svs] : 0.0, NSV > 2 ? P[2 * svs] : 0.0, al, be, om);
}

// stencil_pair for a DERIVED operand: W points at row r of plane z in the slot
// of staged vector 0 (vector k at W + k * svs), W1 likewise for plane z+1; zm0/zm1
// are the derived values of plane z-1.  Returns the derived centre pair (c0, c1)
// and fl(A M^-1 op) (PREC) or fl(A op) for the row pair, legs as in stencil_pair.
template <int DIM, bool VEC, unsigned DROP, bool PREC, int NSV, int MODE>
__device__ __forceinline__ void stencil_pair_der(const TileGeo& g, int nx, const double* W,
                                                 int svs, const double* W1, double zm0,
                                                 double zm1, unsigned b0, unsigned b1,
                                                 double al, double be, double om, double& c0,
                                                 double& c1, double& t0, double& t1) {
  const double d = g.dinv;
  derive_pair<VEC, NSV, MODE>(W, svs, al, be, om, c0, c1);
  const double pm = pre<PREC>(d, derive_one<NSV, MODE>(W - 1, svs, al, be, om));
  const double p0 = pre<PREC>(d, c0), p1 = pre<PREC>(d, c1);
  const double p2 = pre<PREC>(d, derive_one<NSV, MODE>(W + 2, svs, al, be, om));
  double ym0 = 0.0, ym1 = 0.0, yp0 = 0.0, yp1 = 0.0, zp0, zp1;
  if (DIM == 3) {
    derive_pair<VEC, NSV, MODE>(W - nx, svs, al, be, om, ym0, ym1);
    derive_pair<VEC, NSV, MODE>(W + nx, svs, al, be, om, yp0, yp1);
  }
  derive_pair<VEC, NSV, MODE>(W1, svs, al, be, om, zp0, zp1);
  const double czm = g.c[DIM == 3 ? 5 : 3], czp = g.c[DIM == 3 ? 6 : 4];
  double a = 0.0;
  a = legm<DROP>(b0, 1u, a, czm * pre<PREC>(d, zm0));
  if (DIM == 3) a = legm<DROP>(b0, 2u, a, g.c[3] * pre<PREC>(d, ym0));
  a = legm<DROP>(b0, 4u, a, g.c[1] * pm);
  a = a + g.c[0] * p0;
  a = legm<DROP>(b0, 8u, a, g.c[2] * p1);
  if (DIM == 3) a = legm<DROP>(b0, 16u, a, g.c[4] * pre<PREC>(d, yp0));
  a = legm<DROP>(b0, 32u, a, czp * pre<PREC>(d, zp0));
  t0 = a;
  a = 0.0;
  a = legm<DROP>(b1, 1u, a, czm * pre<PREC>(d, zm1));
  if (DIM == 3) a = legm<DROP>(b1, 2u, a, g.c[3] * pre<PREC>(d, ym1));
  a = legm<DROP>(b1, 4u, a, g.c[1] * p0);
  a = a + g.c[0] * p1;
  a = legm<DROP>(b1, 8u, a, g.c[2] * p2);
  if (DIM == 3) a = legm<DROP>(b1, 16u, a, g.c[4] * pre<PREC>(d, yp1));
  a = legm<DROP>(b1, 32u, a, czp * pre<PREC>(d, zp1));
  t1 = a;
}

// Transform stage (XF) of the block-Jacobi modes.  When plane z+1 lands in its
// slot, each thread overwrites its own row pair -- and a share of the halo
// pairs -- of every staged operand v with fl(M^-1 v), the values the stencil
// legs take.  Every element is then preconditioned once per plane instead of
// once per leg that reads it (up to 7 times in 3D), with the same expression and
// order as bj_pair, hence the same bits.  Plane z+1
// is read by nobody else during step n (its +z leg uses the own pair, kept in
// registers), so the writes need no CTA barrier: the next step's barrier orders
// them before the neighbour reads.  A block-Jacobi block spans B/2 consecutive
// pairs owned by consecutive lanes of one warp (pairs are block-aligned), so a
// __syncwarp separates the block reads from the in-place writes.
#define XF_H 3  // halo pairs per thread: <= (2 halo + off + B) / 2 / TNT + 1

// transformed values of the element pair at slot element e; block Jacobi: every
// pair a thread transforms sits at its block position ib (pairs are block-aligned,
// TNT % B == 0), so rows ib, ib+1 of the inverse block come from registers (b0, b1)
template <bool VEC, int NSO, int BB>
__device__ __forceinline__ void xf_pair(const double* base, int svs, int e, int ib,
                                        const double* b0, const double* b1, double (&o)[NSO][2]) {
  {
#pragma unroll
    for (int v = 0; v < NSO; ++v) {
      const double* P = base + v * svs + e - ib;
      double x = 0.0, y = 0.0;
#pragma unroll
      for (int k = 0; k < BB; k += 2) {
        double w0, w1;
        ld2<VEC>(P + k, w0, w1);
        x = x + b0[k] * w0;
        x = x + b0[k + 1] * w1;
        y = y + b1[k] * w0;
        y = y + b1[k + 1] * w1;
      }
      o[v][0] = x;
      o[v][1] = y;
    }
  }
}

template <bool VEC, int NSO>
__device__ __forceinline__ void xf_store(double* base, int svs, int e, const double (&o)[NSO][2]) {
#pragma unroll
  for (int v = 0; v < NSO; ++v) {
    if (VEC) {
      *reinterpret_cast<double2*>(base + v * svs + e) = make_double2(o[v][0], o[v][1]);
    } else {
      base[v * svs + e] = o[v][0];
      base[v * svs + e + 1] = o[v][1];
    }
  }
}

// stencil_pair on transformed planes: the centre pair (p0, p1), the z-1 and z+1
// pairs come from registers, the x and y legs from the transformed plane at W
template <int DIM, bool VEC, unsigned DROP>
__device__ __forceinline__ void stencil_pair_xf(const TileGeo& g, int nx, const double* W,
                                                double p0, double p1, double zm0, double zm1,
                                                double zp0, double zp1, unsigned b0,
                                                unsigned b1, double& t0, double& t1) {
  const double pm = W[-1], p2 = W[2];
  double ym0 = 0.0, ym1 = 0.0, yp0 = 0.0, yp1 = 0.0;
  if (DIM == 3) {
    ld2<VEC>(W - nx, ym0, ym1);
    ld2<VEC>(W + nx, yp0, yp1);
  }
  const double czm = g.c[DIM == 3 ? 5 : 3], czp = g.c[DIM == 3 ? 6 : 4];
  double a = 0.0;
  a = legm<DROP>(b0, 1u, a, czm * zm0);
  if (DIM == 3) a = legm<DROP>(b0, 2u, a, g.c[3] * ym0);
  a = legm<DROP>(b0, 4u, a, g.c[1] * pm);
  a = a + g.c[0] * p0;
  a = legm<DROP>(b0, 8u, a, g.c[2] * p1);
  if (DIM == 3) a = legm<DROP>(b0, 16u, a, g.c[4] * yp0);
  a = legm<DROP>(b0, 32u, a, czp * zp0);
  t0 = a;
  a = 0.0;
  a = legm<DROP>(b1, 1u, a, czm * zm1);
  if (DIM == 3) a = legm<DROP>(b1, 2u, a, g.c[3] * ym1);
  a = legm<DROP>(b1, 4u, a, g.c[1] * p0);
  a = a + g.c[0] * p1;
  a = legm<DROP>(b1, 8u, a, g.c[2] * p2);
  if (DIM == 3) a = legm<DROP>(b1, 16u, a, g.c[4] * yp1);
  a = legm<DROP>(b1, 32u, a, czp * zp1);
  t1 = a;
}

// Per-row arithmetic of each mode.  S = stream slot at this row, st = stride;
// c0/c1 = the stencil operands' centre values, t0/t1 = their stencil products.
template <int MODE, int K, int NOUTC, bool NRM, bool BJ>
__device__ __forceinline__ void row_update(const double* S, int st, bool rr, const double* zrr_g,
                                           double pc0, double pc1, double c0, double c1,
                                           double t0, double t1, double al, double be, double om,
                                           double dinv, Dd* acc, double* o) {
  if (MODE == TM_A) {  // c0 = w_i, c1 = z_{i-1}; t0 = t_i, t1 = v_{i-1}
    const double kj = S[0], gj = S[st], lj = S[2 * st], sj = S[3 * st], rj = S[4 * st];
    const double zoc = rr ? __ldg(zrr_g) : c1; // replaced z_{i-1} (A26), read from global
    const double m = BJ ? pc0 : dinv * c0;     // m_i
    const double nn = BJ ? pc1 : dinv * c1;    // n_{i-1}
    o[0] = kj + be * (gj - om * lj);           // line 5: g
    o[1] = c0 + be * (sj - om * zoc);          // line 6: s
    o[2] = m + be * (lj - om * nn);            // line 7: l
    o[3] = t0 + be * (zoc - om * t1);          // line 8: z
    const double qq = rj - al * o[1];          // line 9
    const double yy = c0 - al * o[3];          // line 11
    dd_fma(acc[0], qq, yy);                    // line 12
    dd_fma(acc[1 % K], yy, yy);
    if (NRM) {
      nrm_add(acc[2 % K], kj); nrm_add(acc[3 % K], c0); nrm_add(acc[4 % K], m);
      nrm_add(acc[5 % K], t0); nrm_add(acc[6 % K], o[0]); nrm_add(acc[7 % K], o[1]);
      nrm_add(acc[8 % K], o[2]); nrm_add(acc[9 % K], o[3]); nrm_add(acc[10 % K], qq);
      nrm_add(acc[11 % K], yy);
    }
  } else if (MODE == TM_C) {  // c0 = w_i, c1 = z_i; t0 = t_i, t1 = v_i
    const double xj = S[0], gj = S[st], kj = S[2 * st], lj = S[3 * st], rj = S[4 * st];
    const double sj = S[5 * st], rhj = S[6 * st];
    const double m = BJ ? pc0 : dinv * c0;     // m_i
    const double nn = BJ ? pc1 : dinv * c1;    // n_i (line 13)
    const double uu = kj - al * lj;            // line 10
    const double qq = rj - al * sj;            // line 9
    const double yy = c0 - al * c1;            // line 11
    o[0] = (xj + al * gj) + om * uu;           // line 17: x
    o[1] = qq - om * yy;                       // line 18: r
    o[2] = uu - om * (m - al * nn);            // line 19: k
    o[3] = yy - om * (t0 - al * t1);           // line 20: w
    dd_fma(acc[0], rhj, o[1]);                 // line 21
    dd_fma(acc[1 % K], rhj, o[3]);
    dd_fma(acc[2 % K], rhj, sj);
    dd_fma(acc[3 % K], rhj, c1);
    dd_fma(acc[4 % K], o[1], o[1]);
    if (NRM) {
      nrm_add(acc[5 % K], xj); nrm_add(acc[6 % K], uu); nrm_add(acc[7 % K], nn);
      nrm_add(acc[8 % K], t1);
    }
  } else if (MODE == TM_RR1) {  // c = x, g; t0 = A x, t1 = A g; streams b, r^
    const double rj = S[0] - t0;               // r := b - A x
    const double rhj = S[st];
    o[0] = rj;
    o[1] = dinv * rj;                          // k := M^-1 r
    o[2] = t1;                                 // s := A g
    o[3] = dinv * t1;                          // l := M^-1 s
    constexpr int KD = NRM ? 4 : 0;            // the stashed line-21 dots (Stash)
    dd_fma(acc[KD % K], rhj, rj);              // (r^, r)
    dd_fma(acc[(KD + 1) % K], rhj, t1);        // (r^, s)
    dd_fma(acc[(KD + 2) % K], rj, rj);         // (r, r)
    if (NRM) {  // (block Jacobi: k, l norms after the shuffle in t_tile)
      nrm_add(acc[0], c0); nrm_add(acc[2 % K], o[2]);
      if (!BJ) {
        nrm_add(acc[1 % K], o[1]);
        nrm_add(acc[3 % K], o[3]);
      }
    }
  } else if (MODE == TM_RR2) {  // c = k, l; t0 = A k = A M^-1 r, t1 = A l = A M^-1 s
    const double rhj = S[0];
    o[0] = t0;                                 // w := A k
    o[1] = t1;                                 // z := A l
    dd_fma(acc[1 % K], rhj, t0);               // line 21 on the replaced vectors; slots
    dd_fma(acc[3 % K], rhj, t1);               // 0, 2, 4 come from RR1's stash
    if (NRM) nrm_add(acc[5 % K], t1);
  } else if (MODE == TM_GAP) {  // c = x; t0 = A x
    const double dg = (S[0] - t0) - S[st];     // (b - A x) - r
    dd_fma(acc[0], dg, dg);
  } else if (MODE == TM_INIT1) {  // c = x0; t0 = A x0
    const double bj = S[0];
    const double rj = bj - t0;                 // r0 := b - A x0
    o[0] = rj;
    o[1] = rj;                                 // r^ := r0 (A2)
    o[2] = dinv * rj;                          // k0 := M^-1 r0
    dd_fma(acc[0], rj, rj);
    dd_fma(acc[1 % K], bj, bj);
    if (NRM) {
      nrm_add(acc[2 % K], c0);
      if (!BJ) nrm_add(acc[3 % K], o[2]);
    }
  } else if (MODE == TM_INIT2) {  // c = r0; t0 = A M^-1 r0 = A k0
    o[0] = t0;                                 // w0
    dd_fma(acc[0], S[0], t0);                  // (r^, w0)
  } else if (MODE == TM_CL1) {  // c0 = p_i (derived, l.17), t0 = A M^-1 p_i (l.4-5)
    o[0] = c0;                                 // p_i
    o[1] = t0;                                 // s_i
    dd_fma(acc[0], S[0], t0);                  // l.6: (r^0, s_i)
  } else if (MODE == TM_CL2) {  // c0 = q_i (derived, l.8), t0 = y_i = A M^-1 q_i (l.9-10)
    dd_fma(acc[0], c0, t0);                    // l.11: (q, y)
    dd_fma(acc[1 % K], t0, t0);                //       (y, y)
  } else if (MODE == TM_CL3) {  // c0 = q_i, t0 = y_i; streams x, p, r^0
    const double xj = S[0], pj = S[st], rhj = S[2 * st];
    const double gj = BJ ? pc1 : dinv * pj;    // l.4: g := M^-1 p (BJ: lane shuffle)
    const double uj = BJ ? pc0 : dinv * c0;    // l.9: u := M^-1 q
    o[0] = (xj + al * gj) + om * uj;           // l.13: x
    o[1] = c0 - om * t0;                       // l.14: r
    dd_fma(acc[0], rhj, o[1]);                 // l.15: (r^0, r)
    dd_fma(acc[1 % K], o[1], o[1]);            //       ||r||^2 (A8)
  } else if (MODE == TM_PC) {  // c0 = w_i, t0 = n_i = A M^-1 w_i; streams z,q,s,p,x,r,u
    const double mj = BJ ? pc0 : dinv * c0;    // m := M^-1 w
    const double zj = S[0], qj = S[st], sj = S[2 * st], pj = S[3 * st];
    const double xj = S[4 * st], rj = S[5 * st], uj = S[6 * st];
    const double zn = t0 + be * zj;            // z := n + beta z
    const double qn = mj + be * qj;            // q := m + beta q
    const double sn = c0 + be * sj;            // s := w + beta s
    const double pn = uj + be * pj;            // p := u + beta p
    const double xn = xj + al * pn;            // x := x + alpha p
    const double rn = rj - al * sn;            // r := r - alpha s
    const double un = uj - al * qn;            // u := u - alpha q
    const double wn = c0 - al * zn;            // w := w - alpha z
    o[0] = zn; o[1 % NOUTC] = qn; o[2 % NOUTC] = sn; o[3 % NOUTC] = pn;
    o[4 % NOUTC] = xn; o[5 % NOUTC] = rn; o[6 % NOUTC] = un; o[7 % NOUTC] = wn;
    dd_fma(acc[0], rn, un);                    // next iteration's (r, u)
    dd_fma(acc[1 % K], wn, un);                //                  (w, u)
    dd_fma(acc[2 % K], rn, rn);                //                  ||r||^2
  } else if (MODE == TM_PCI1) {  // c = x0; t0 = A x0; stream b
    const double bj = S[0];
    const double rj = bj - t0;                 // r0 := b - A x0
    o[0] = rj;
    o[1 % NOUTC] = dinv * rj;                  // u0 := M^-1 r0
    dd_fma(acc[0], rj, rj);
    dd_fma(acc[1 % K], bj, bj);
  } else if (MODE == TM_SPB || MODE == TM_SPD) {  // lines 13-14 / 22-23: v_i / t_{i+1}
    o[0] = t0;
  } else if (MODE == TM_PCI2) {  // c = r0; t0 = A M^-1 r0 = A u0
    const double uj = BJ ? pc0 : dinv * c0;    // u0 (same value as stored)
    o[0] = t0;                                 // w0
    dd_fma(acc[0], c0, uj);                    // (r0, u0)
    dd_fma(acc[1 % K], t0, uj);                // (w0, u0)
  }
}

// Generic tile kernel.  VEC: every staged range and every vector is 16-byte
// aligned (nx even) -> paired loads and stores.  One row pair per thread:
// TP <= 2 * TNT.
// BJ: block-Jacobi block size (0 Jacobi); SEG: x-segmented tiles (nx > 1024)
// Peer-memory transport (Vecs::hz / hw): copy this thread's row pair of the slab's
// first / last plane of z_i (sweep A) or w_{i+1} (sweep C) -- stored by the same thread
// earlier in the unit -- into the neighbours' ghost planes.  Out of line: it runs at the
// end of the (at most two) boundary units and stays out of the step loop's registers.
template <bool VEC>
__device__ __noinline__ bool peer_put(double* hp_lo, double* hp_hi, const double* own,
                                      int64_t pxy, int64_t nol, int64_t z0, int64_t z1,
                                      int64_t po, bool valid1) {
  bool stored = false;
  for (int sd = 0; sd < 2; ++sd) {
    double* const hp = sd == 0 ? hp_lo : hp_hi;
    const int64_t zb = sd == 0 ? 0 : nol - 1;
    if (!hp || zb < z0 || zb >= z1) continue;
    const double a = own[zb * pxy + po];
    const double c = valid1 ? own[zb * pxy + po + 1] : 0.0;
    st2<VEC>(hp + po, a, c, valid1);
    stored = true;
  }
  return stored;
}

// PEER: the instance the peer-memory transport launches (tile_launch picks it when
// TileGeo::peer): sweeps A / C also store their boundary planes in the neighbours.  A
// template flag so the default instances carry no trace of it (measured: even an
// untaken runtime branch cost sweep A 0.5-1.3%).
template <int M> struct HasPeer { enum { v = BaseOf<M>::v == TM_A || BaseOf<M>::v == TM_C }; };

// Timeline instrumentation (experiments only: scripts/timeline.py builds a variant
// library with -DPBICG_TIMELINE; the product build carries none of it).  Thread 0 of
// every CTA appends one record per launch: %globaltimer at entry, after the PDL wait,
// when the first unit's first plane has landed, after the unit loop and at exit.
#ifdef PBICG_TIMELINE
struct TlRec {
  unsigned long long t[8];  // entry, wait, first plane, loop end, exit, grid reduce done,
                            // publish done, spare
  unsigned long long id;    // block | grid << 16 | mode << 32 | smid << 48
  unsigned long long units;
};
__device__ TlRec* g_tl_buf;
__device__ unsigned int* g_tl_cnt;
__device__ unsigned int g_tl_cap;
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TL_DECL unsigned long long tl_t[8] = {0, 0, 0, 0, 0, 0, 0, 0}; unsigned long long tl_units = 0
#define TL_STAMP(k) do { if (threadIdx.x == 0 && tl_t[k] == 0) tl_t[k] = tl_now(); } while (0)
#define TL_UNIT() (++tl_units)
#define TL_FLUSH(mode)                                                                       \
  do {                                                                                       \
    if (threadIdx.x == 0) tl_t[4] = tl_now();                                                \
    if (threadIdx.x == 0 && g_tl_buf) {                                                      \
      unsigned smid;                                                                         \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));                                      \
      const unsigned i = atomicAdd(g_tl_cnt, 1u);                                            \
      if (i < g_tl_cap) {                                                                    \
        TlRec r;                                                                             \
        for (int k_ = 0; k_ < 8; ++k_) r.t[k_] = tl_t[k_];                                   \
        r.id = blockIdx.x | ((unsigned long long)gridDim.x << 16) |                          \
               ((unsigned long long)(mode) << 32) | ((unsigned long long)smid << 48);        \
        r.units = tl_units;                                                                  \
        g_tl_buf[i] = r;                                                                     \
      }                                                                                      \
    }                                                                                        \
  } while (0)
#else
#define TL_DECL
#define TL_STAMP(k) do { } while (0)
#define TL_UNIT() do { } while (0)
#define TL_FLUSH(mode) do { } while (0)
#endif

// The body of one tile step.
template <int DIM, int MODE_, bool VEC, int BJ = 0, bool SEG = false, bool PEER = false>
__device__ __forceinline__ void t_tile_body(const TileGeo& g, const Vecs& V, Scal* __restrict__ sc,
                                            Dd* __restrict__ part, const Hist& h) {
  using T = TileTraits<MODE_>;
  constexpr int MODE = BaseOf<MODE_>::v;
  constexpr bool NRM = MODE_ != MODE;
  constexpr int NSV = T::NSV, NST = T::NSTR;
  constexpr int NSTR_MAX = NST > 0 ? NST : 1;  // array extent
  constexpr bool HAS_STR = NST > 0;
  constexpr bool DER = T::DER != 0;
  constexpr int NSO = DER ? 1 : NSV;           // stencil operands
  constexpr int NOUT = T::NOUT > 0 ? T::NOUT : 1;
  constexpr int K = T::K > 0 ? T::K : 1;
  constexpr bool PREC = T::PREC != 0;
  constexpr bool BJP = BJ > 0 && PREC && !DER;  // stencil operands enter as A (block M)^-1 v
  constexpr int BB = BJ > 0 ? BJ : 2;          // block size for the helpers' array extents
  // transform stage (xf_pair) for block Jacobi b >= 4.  Measured on cfg4 (it/s, per-leg
  // form -> transform): b = 8: 89 -> 162, b = 4: 177 -> 197; b = 2: 226 -> 210 and the
  // derived operands of classic BiCGStab: 292 -> 276, so those keep the per-leg form
  // (their per-leg work is one or two flops; the transform's halo pairs and stores cost more)
  // Derived operands (classic BiCGStab's p_i, q_i) under block Jacobi always take the
  // transform stage: each staged element is derived once, then transformed in place
  // (xf_plane), and the stencil runs on M^-1 of the derived plane.
  constexpr bool XF = BJ > 0 && PREC && (DER || BB >= 4);
  __shared__ double s_bi[64];                  // the inverse block (row-major BB x BB)
  TL_DECL;
  TL_STAMP(0);
  if (BJ > 0) {
    for (int q = threadIdx.x; q < BB * BB; q += blockDim.x) s_bi[q] = g.bi[q];
  }
  // PDL (tile_launch): nothing above reads the previous kernel's results; wait for it
  // to complete (a no-op without PDL)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  TL_STAMP(1);
  // the state the last CTA's bookkeeping starts from (Snap, state.cuh): loaded now by a
  // thread that issues no TMA, consumed after the grid reduction
  __shared__ Snap s_snap;
  if (T::K > 0 && threadIdx.x == 32) snap_load(s_snap, sc);
  constexpr int SD = StreamDepth<MODE_>::v;  // stream ring depth; stencil barriers follow
  constexpr int SVR = SvDepth<MODE_>::v;      // stencil-plane ring depth
  static_assert(SD + SVR <= 8, "the mbarriers fit the 64-byte shared-memory header");
  static_assert(K <= RED_K, "partials buffer holds RED_K pairs per CTA");
  if (MODE == TM_A || MODE == TM_C || MODE == TM_CL1 || MODE == TM_CL2 || MODE == TM_CL3 ||
      MODE == TM_PC || MODE == TM_SPB || MODE == TM_SPD) {
    if (sc->done) return;
  } else if (MODE == TM_RR1 || MODE == TM_RR2) {
    if (sc->done || !sc->rr_fire) return;
  } else if (MODE == TM_GAP) {
    if (sc->gap_iter >= sc->iter) return;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);  // [0,SD) streams, [SD,SD+3) stencil
  double* st = reinterpret_cast<double*>(smem_raw + 64);
  double* sv = st + SD * NST * g.st_stride;
  const int tid = threadIdx.x;
  const int nx = (int)g.nx;
  const int sts = g.st_stride, svs = g.sv_stride;

  const int it = sc->iter;
  const double al = sc->alpha, be = sc->beta, om = sc->omega;
  const bool rr = MODE == TM_A && sc->use_rr != 0;
  const double* svp[3] = {nullptr, nullptr, nullptr};
  const double* stp[NSTR_MAX];
  int nstr = NSTR_MAX;
  double* outp[NOUT];
  if (MODE == TM_A) {
    svp[0] = (it & 1) ? V.w1 : V.w0;                 // w_i
    svp[1] = (it & 1) ? V.z0 : V.z1;                 // z_{i-1} pre-replacement
    stp[0] = V.k; stp[1 % NSTR_MAX] = V.g; stp[2 % NSTR_MAX] = V.l; stp[3 % NSTR_MAX] = V.s;
    stp[4 % NSTR_MAX] = V.r;                         // (replaced z_{i-1}: global load, A26)
    outp[0] = V.g; outp[1 % NOUT] = V.s; outp[2 % NOUT] = V.l;
    outp[3 % NOUT] = (it & 1) ? V.z1 : V.z0;         // z_i
  } else if (MODE == TM_C) {
    svp[0] = (it & 1) ? V.w1 : V.w0;                 // w_i
    svp[1] = (it & 1) ? V.z1 : V.z0;                 // z_i
    stp[0] = V.x; stp[1 % NSTR_MAX] = V.g; stp[2 % NSTR_MAX] = V.k; stp[3 % NSTR_MAX] = V.l;
    stp[4 % NSTR_MAX] = V.r; stp[5 % NSTR_MAX] = V.s;
    stp[NSTR_MAX - 1] = V.rh;
    outp[0] = V.x; outp[1 % NOUT] = V.r; outp[2 % NOUT] = V.k;
    outp[3 % NOUT] = (it & 1) ? V.w0 : V.w1;         // w_{i+1}
  } else if (MODE == TM_RR1) {
    svp[0] = V.x; svp[1] = V.g;
    stp[0] = V.b; stp[1 % NSTR_MAX] = V.rh;
    outp[0] = V.r; outp[1 % NOUT] = V.k; outp[2 % NOUT] = V.s; outp[3 % NOUT] = V.l;
  } else if (MODE == TM_RR2) {
    svp[0] = V.k; svp[1] = V.l;                      // M^-1 r, M^-1 s as RR1 stored them
    stp[0] = V.rh;
    outp[0] = (it & 1) ? V.w0 : V.w1;                // w_{i+1}
    outp[1 % NOUT] = V.zrr;                          // replaced z_i (A26)
  } else if (MODE == TM_GAP) {
    svp[0] = V.x;
    stp[0] = V.b;
    stp[1 % NSTR_MAX] = (sc->method == 1 && (it & 1)) ? V.k : V.r;  // Alg. 1: r double-buffered
  } else if (MODE == TM_CL1 || MODE == TM_CL2 || MODE == TM_CL3) {
    // Alg. 1 buffers: r_i in {r, k}[i&1], p_i in {g, l}[i&1], s_i in {s, zrr}[i&1]
    const bool odd = (it & 1) != 0;
    double* const Rc = odd ? V.k : V.r;   // r_i
    double* const Ro = odd ? V.r : V.k;   // r_{i+1}
    double* const Pc = odd ? V.l : V.g;   // p_i
    double* const Po = odd ? V.g : V.l;   // p_{i-1}
    double* const Sc = odd ? V.zrr : V.s; // s_i
    double* const So = odd ? V.s : V.zrr; // s_{i-1}
    if (MODE == TM_CL1) {
      svp[0] = Rc; svp[1] = Po; svp[2] = So;          // r_i, p_{i-1}, s_{i-1}
      stp[0] = V.rh;
      outp[0] = Pc; outp[1 % NOUT] = Sc;               // p_i, s_i
    } else if (MODE == TM_CL2) {
      svp[0] = Rc; svp[1] = Sc;                        // q_i = r_i - alpha s_i
    } else {
      svp[0] = Rc; svp[1] = Sc;
      stp[0] = V.x; stp[1 % NSTR_MAX] = Pc; stp[2 % NSTR_MAX] = V.rh;
      outp[0] = V.x; outp[1 % NOUT] = Ro;              // x_{i+1}, r_{i+1}
    }
  } else if (MODE == TM_PC) {
    // p-CG buffers: z -> z0, q -> l, s, p -> g, x, r, u -> k; w_i in {w0, w1}[i&1]
    svp[0] = (it & 1) ? V.w1 : V.w0;
    stp[0] = V.z0; stp[1 % NSTR_MAX] = V.l; stp[2 % NSTR_MAX] = V.s; stp[3 % NSTR_MAX] = V.g;
    stp[4 % NSTR_MAX] = V.x; stp[5 % NSTR_MAX] = V.r; stp[6 % NSTR_MAX] = V.k;
    outp[0] = V.z0; outp[1 % NOUT] = V.l; outp[2 % NOUT] = V.s; outp[3 % NOUT] = V.g;
    outp[4 % NOUT] = V.x; outp[5 % NOUT] = V.r; outp[6 % NOUT] = V.k;
    outp[7 % NOUT] = (it & 1) ? V.w0 : V.w1;
  } else if (MODE == TM_PCI1) {
    svp[0] = V.x;
    stp[0] = V.b;
    outp[0] = V.r; outp[1 % NOUT] = V.k;              // r0, u0
  } else if (MODE == TM_SPB) {  // v_i = A M^-1 z_i (z_i as sweep A wrote it)
    svp[0] = (it & 1) ? V.z1 : V.z0;
    outp[0] = V.vv;
  } else if (MODE == TM_SPD) {  // t_{i+1} = A M^-1 w_{i+1} (buffer named by sweep C2)
    svp[0] = sc->spd_par ? V.w1 : V.w0;
    outp[0] = V.tv;
  } else if (MODE == TM_PCI2) {
    svp[0] = V.r;
    outp[0] = V.w0;
  } else if (MODE == TM_INIT1) {
    svp[0] = V.x;
    stp[0] = V.b;
    outp[0] = V.r; outp[1 % NOUT] = V.rh; outp[2 % NOUT] = V.k;
  } else if (MODE == TM_INIT2) {
    svp[0] = V.r;
    stp[0] = V.rh;
    outp[0] = V.w0;
  }
  if (tid == 0) {
    for (int i = 0; i < SD + SVR; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  uint32_t ph = 0;        // parity bits: bit s (streams 0..SD-1), bit SD+s (stencil 0..2)
  int svc = 0, stc = 0;   // ring counters (slots filled so far)
  Dd acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = dd_zero();
  const int r = 2 * tid;  // this thread's row pair within the tile
  bool remote = false;    // this thread stored into a peer's ghost plane
  // peer ghost planes of this sweep's z_i (A) / w_{i+1} (C): only a uniform flag stays
  // live across the loop; the pointers are resolved in the (boundary-plane) branch
  constexpr bool peer = PEER && (MODE == TM_A || MODE == TM_C);

  for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
    const int col = u % g.ncols, q = u / g.ncols;
    // SEG: col = ycol * nseg + segment; x0s/sxc = the segment's first column / width
    const int ycol = SEG ? col / g.nseg : col;
    const int x0s = SEG ? (col % g.nseg) * g.sx : 0;
    const int sxc = SEG ? (nx - x0s < g.sx ? nx - x0s : g.sx) : nx;
    const int64_t y0 = (int64_t)ycol * g.TY;
    const int tyc = (int)((g.ny - y0) < g.TY ? (g.ny - y0) : g.TY);
    const int TP = tyc * sxc;
    const int ly = r / sxc, cx = r % sxc;         // this row pair's line / column in the tile
    const int ls = SEG ? g.lstride : nx;          // y stride of the staged stencil planes
    const int nlines = DIM == 3 ? tyc + 2 : 1;    // SEG: staged lines per stencil plane
    const int64_t z0 = (int64_t)q * g.chunk;
    const int64_t z1 = (z0 + g.chunk) < g.nol ? (z0 + g.chunk) : g.nol;
    const int nst = (int)(z1 - z0), nsv = nst + 2;
    const int64_t toff = DIM == 3 ? y0 * g.nx : 0;
    // per-row boundary bits (constant over the unit)
    const bool act = r < TP, valid1 = r + 1 < TP;
    unsigned b0 = 0, b1 = 0;
    {
      const int x0 = SEG ? x0s + cx : r % nx, x1 = SEG ? x0s + cx + 1 : (r + 1) % nx;
      const int64_t gy0 = SEG ? y0 + ly : y0 + r / nx, gy1 = SEG ? y0 + ly : y0 + (r + 1) / nx;
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
    const unsigned amask = __ballot_sync(0xffffffffu, act);  // blocks are all-in or all-out
    const int i0 = BJ > 0 ? ((SEG ? x0s + cx : r % nx) % BB) : 0;  // position in its block
    const unsigned xy_all = DIM == 3 ? 30u : 12u;
    const bool xy_int = __all_sync(0xffffffffu, !act || ((b0 & xy_all) == xy_all &&
                                                         (b1 & xy_all) == xy_all));
    const unsigned y_all = DIM == 3 ? 18u : 0u;  // in-plane y legs (3D)
    const bool yz_int = __all_sync(0xffffffffu, !act || ((b0 & y_all) == y_all &&
                                                         (b1 & y_all) == y_all));
    double m1[NSO][2];  // plane z-1 centre values per stencil operand
    double cr[NSO][2];  // XF: raw centre pair of plane z
    double tr[NSO][2];  // XF: transformed centre pair of plane z
#pragma unroll
    for (int v = 0; v < NSO; ++v)
      m1[v][0] = m1[v][1] = cr[v][0] = cr[v][1] = tr[v][0] = tr[v][1] = 0.0;
    // SEG: element index of (line y0 - 1 (3D) / the line (2D), column x0s - SEG_HX)
    const int64_t sv_e0 = SEG ? (DIM == 3 ? (y0 - 1) * g.nx : 0) + x0s - SEG_HX : 0;
    const int64_t st_e0 = SEG ? (DIM == 3 ? y0 * g.nx : 0) + x0s : 0;
    auto stage_sv = [&](int s, int64_t zp) {  // stencil plane zp into ring slot s
      if (SEG)
        stage_lines(sv + (size_t)s * NSV * svs, svs, svp, NSV, zp * g.pxy + sv_e0, g.nx, nlines,
                    sxc + 2 * SEG_HX, ls, &bar[SD + s]);
      else
        stage(sv + (size_t)s * NSV * svs, svs, svp, NSV, zp * g.pxy + toff - g.halo,
              TP + 2 * g.halo, &bar[SD + s]);
    };
    auto stage_st = [&](int s, int64_t zp) {  // streamed vectors of plane zp into slot s
      if (SEG)
        stage_lines(st + (size_t)s * NST * sts, sts, stp, nstr, zp * g.pxy + st_e0, g.nx, tyc,
                    sxc, g.sx, &bar[s]);
      else
        stage(st + (size_t)s * NST * sts, sts, stp, nstr, zp * g.pxy + toff, TP, &bar[s]);
    };
    // this row pair's offset in a stencil slot / a stream slot
    auto sv_off = [&](int64_t zp) -> int {
      return SEG ? (ly + (DIM == 3 ? 1 : 0)) * ls + SEG_HX + cx
                 : align_off(svp[0] + zp * g.pxy + toff - g.halo) + g.halo + r;
    };
    // XF: transform plane zp in slot s (own pair + a share of the halo pairs);
    // returns the own pair raw (craw) and transformed (ctr).  Full-line tiles only
    // (block Jacobi needs nx % b == 0 <= 1024).  Every pair this thread transforms
    // sits at block position i0, so rows i0, i0+1 of the inverse block are registers.
    static_assert(!(XF && SEG), "the transform stage runs on full-line tiles");
    double bir0[BB], bir1[BB];
#pragma unroll
    for (int q = 0; q < BB; ++q) {
      bir0[q] = XF ? s_bi[i0 * BB + q] : 0.0;
      bir1[q] = XF ? s_bi[(i0 + 1) * BB + q] : 0.0;
    }
    auto xf_plane = [&](int s, int64_t zp, double (&craw)[NSO][2], double (&ctr)[NSO][2]) {
      double* base = sv + (size_t)s * NSV * svs;
      // E0: slot element of tile row 0.  Halo pairs h: nb (a multiple of the pairs per
      // block, so blocks stay inside a warp) end at E0, the rest start at the tile's end.
      const int E0 = align_off(svp[0] + zp * g.pxy + toff - g.halo) + g.halo;
      const int TPe = TP + (TP & 1);
      constexpr int BP = BB / 2;
      const int nb = ((E0 + 1) / 2 + BP - 1) / BP * BP;
      const int H = nb + (g.halo - (TP & 1) + 1) / 2;
      if (DER) {  // derive the operand into staged vector 0 (own pair + halo pairs)
        if (act) {
          const int e = sv_off(zp);
          double a, b;
          derive_pair<VEC, NSV, MODE>(base + e, svs, al, be, om, a, b);
          xf_store<VEC, 1>(base, svs, e, {{a, b}});
        }
#pragma unroll
        for (int k = 0; k < XF_H; ++k) {
          const int h = tid + k * TNT;
          const int e = h < nb ? E0 - 2 * (nb - h) : E0 + TPe + 2 * (h - nb);
          if (h >= H || e < 0 || e + 1 >= svs) continue;
          double a, b;
          derive_pair<VEC, NSV, MODE>(base + e, svs, al, be, om, a, b);
          xf_store<VEC, 1>(base, svs, e, {{a, b}});
        }
        __syncwarp();  // a block's derived values before any lane transforms it
      }
      if (act) {
        const int e = sv_off(zp);
#pragma unroll
        for (int v = 0; v < NSO; ++v) ld2<VEC>(base + v * svs + e, craw[v][0], craw[v][1]);
        xf_pair<VEC, NSO, BB>(base, svs, e, i0, bir0, bir1, ctr);
      }
      // one operand and one halo pair at a time (registers); per pair the warp's
      // block reads precede its in-place writes (__syncwarp)
#pragma unroll
      for (int v = 0; v < NSO; ++v) {
        double* bv = base + v * svs;
#pragma unroll
        for (int k = 0; k < XF_H; ++k) {
          const int h = tid + k * TNT;
          int e = h < nb ? E0 - 2 * (nb - h) : E0 + TPe + 2 * (h - nb);
          if (h >= H || e < 0 || e + 1 >= svs) e = -1;
          double o[1][2] = {{0.0, 0.0}};
          if (e >= 0) xf_pair<VEC, 1, BB>(bv, svs, e, i0, bir0, bir1, o);
          __syncwarp();
          if (k == 0 && act) xf_store<VEC, 1>(bv, svs, sv_off(zp), {{ctr[v][0], ctr[v][1]}});
          if (e >= 0) xf_store<VEC, 1>(bv, svs, e, o);
        }
      }
      fence_proxy_async_smem();  // the slot is re-staged by TMA after a later barrier
    };
    if (tid == 0) {
      for (int m = 0; m < SVR && m < nsv; ++m) stage_sv((svc + m) % SVR, z0 - 1 + m);
      if (HAS_STR) {
        for (int m = 0; m < SD - 1 && m < nst; ++m) stage_st((stc + m) % SD, z0 + m);
      }
    }
    {  // plane z0-1 -> registers
      const int s = svc % SVR;
      mbar_wait(&bar[SD + s], (ph >> (SD + s)) & 1u);
      ph ^= 1u << (SD + s);
      TL_STAMP(2);
      TL_UNIT();
      const double* b0p = sv + (size_t)s * NSV * svs + sv_off(z0 - 1);
      if (DER && XF) {  // M^-1 of the derived plane z0-1 (transform stage, all threads)
        double raw[NSO][2];
        xf_plane(s, z0 - 1, raw, m1);
      } else if (act) {
        if (DER) {
          derive_pair<VEC, NSV, MODE>(b0p, svs, al, be, om, m1[0][0], m1[0][1]);
        } else if (BJP) {  // the -z leg takes M^-1 of plane z0-1
#pragma unroll
          for (int v = 0; v < NSO; ++v)
            bj_pair<BB, VEC>(s_bi, i0, b0p + v * svs - i0, m1[v][0], m1[v][1]);
        } else {
#pragma unroll
          for (int v = 0; v < NSO; ++v) ld2<VEC>(b0p + v * svs, m1[v][0], m1[v][1]);
        }
      }
      const int s1 = (svc + 1) % SVR;  // plane z0
      mbar_wait(&bar[SD + s1], (ph >> (SD + s1)) & 1u);
      ph ^= 1u << (SD + s1);
      if (XF) xf_plane(s1, z0, cr, tr);  // ordered before step 0's reads by its barrier
    }
    // ring slots of step n, advanced incrementally (no modulo per step): the slot plane
    // z+SVR-1 is staged into, planes z and z+1, the stream slot and the stream slot
    // being refilled; the 16-byte phase of a plane's first staged element flips per
    // plane only when the plane stride is odd
    int k_new = svc % SVR, k_z = (svc + 1) % SVR, k_z1 = (svc + 2) % SVR;
    int k_st = stc % SD, k_stn = (stc + SD - 1) % SD;
    const int pstep = (int)(g.pxy & 1);
    const int ao_sv0 = SEG ? 0 : align_off(svp[0] + z0 * g.pxy + toff - g.halo);
    const int ao_st0 = (SEG || !HAS_STR) ? 0 : align_off(stp[0] + z0 * g.pxy + toff);
    const int64_t gin = SEG ? (DIM == 3 ? (y0 + ly) * g.nx : 0) + x0s + cx : toff + r;
    int64_t gz = z0 * g.pxy;  // z * pxy
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
        if (n + SVR < nsv) stage_sv(k_new, z + SVR - 1);  // plane z+SVR-1
        if (HAS_STR && n + SD - 1 < nst)  // streams z+SD-1 into the slot step n-1 freed
          stage_st(k_stn, z + SD - 1);
      }
      const int s_z = k_z, s_z1 = k_z1, s_st = k_st;
      mbar_wait(&bar[SD + s_z1], (ph >> (SD + s_z1)) & 1u);
      ph ^= 1u << (SD + s_z1);
      if (HAS_STR) {
        mbar_wait(&bar[s_st], (ph >> s_st) & 1u);
        ph ^= 1u << s_st;
      }
      double cn[NSO][2], tn[NSO][2];  // XF: own pair of plane z+1, raw / transformed
      if (XF) xf_plane(s_z1, z + 1, cn, tn);
      if (!act) continue;
      // plane offsets: sv_off / align_off without re-deriving them from addresses
      const int ov_z = SEG ? (ly + (DIM == 3 ? 1 : 0)) * ls + SEG_HX + cx
                           : (ao_sv0 ^ (n & pstep)) + g.halo + r;
      const int ov_z1 = SEG ? ov_z : (ao_sv0 ^ ((n + 1) & pstep)) + g.halo + r;
      const double* Wz = sv + (size_t)s_z * NSV * svs + ov_z;
      const double* Wz1 = sv + (size_t)s_z1 * NSV * svs + ov_z1;
      const double* S0 = !HAS_STR ? nullptr
                         : SEG    ? st + (size_t)s_st * NST * sts + ly * g.sx + cx
                                  : st + (size_t)s_st * NST * sts + (ao_st0 ^ (n & pstep)) + r;
      const bool zin = (g.o0 + z) > 0 && (g.o0 + z) < g.nog - 1;
      const unsigned zb = ((g.o0 + z) > 0 ? 1u : 0u) | ((g.o0 + z) < g.nog - 1 ? 32u : 0u);
      double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, t[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      double pc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // block Jacobi: M^-1 of the centre pair
      if (XF) {  // plane z holds the transformed operands; centre, z+-1 from registers
        if (xy_int && zin) {
#pragma unroll
          for (int v = 0; v < NSO; ++v)
            stencil_pair_xf<DIM, VEC, 0u>(g, ls, Wz + v * svs, tr[v][0], tr[v][1], m1[v][0],
                                            m1[v][1], tn[v][0], tn[v][1], 0u, 0u, t[v][0],
                                            t[v][1]);
        } else if (yz_int && zin) {  // x legs only
#pragma unroll
          for (int v = 0; v < NSO; ++v)
            stencil_pair_xf<DIM, VEC, 12u>(g, ls, Wz + v * svs, tr[v][0], tr[v][1], m1[v][0],
                                             m1[v][1], tn[v][0], tn[v][1], b0, b1, t[v][0],
                                             t[v][1]);
        } else {
#pragma unroll
          for (int v = 0; v < NSO; ++v)
            stencil_pair_xf<DIM, VEC, 63u>(g, ls, Wz + v * svs, tr[v][0], tr[v][1], m1[v][0],
                                             m1[v][1], tn[v][0], tn[v][1], b0 | zb, b1 | zb,
                                             t[v][0], t[v][1]);
        }
#pragma unroll
        for (int v = 0; v < NSO; ++v) {
          c[v][0] = cr[v][0];
          c[v][1] = cr[v][1];
          pc[v][0] = tr[v][0];
          pc[v][1] = tr[v][1];
          cr[v][0] = cn[v][0];
          cr[v][1] = cn[v][1];
          tr[v][0] = tn[v][0];
          tr[v][1] = tn[v][1];
        }
      } else if (BJP) {
        if (xy_int && zin) {
#pragma unroll
          for (int v = 0; v < NSO; ++v)
            stencil_pair_bj<DIM, VEC, 0u, BB>(g, s_bi, ls, i0, Wz + v * svs, Wz1 + v * svs,
                                              m1[v][0], m1[v][1], 0u, 0u, c[v][0], c[v][1],
                                              pc[v][0], pc[v][1], t[v][0], t[v][1]);
        } else if (yz_int && zin) {  // x legs only
#pragma unroll
          for (int v = 0; v < NSO; ++v)
            stencil_pair_bj<DIM, VEC, 12u, BB>(g, s_bi, ls, i0, Wz + v * svs, Wz1 + v * svs,
                                               m1[v][0], m1[v][1], b0, b1, c[v][0], c[v][1],
                                               pc[v][0], pc[v][1], t[v][0], t[v][1]);
        } else {
#pragma unroll
          for (int v = 0; v < NSO; ++v)
            stencil_pair_bj<DIM, VEC, 63u, BB>(g, s_bi, ls, i0, Wz + v * svs, Wz1 + v * svs,
                                                 m1[v][0], m1[v][1], b0 | zb, b1 | zb, c[v][0],
                                                 c[v][1], pc[v][0], pc[v][1], t[v][0], t[v][1]);
        }
      } else if (DER) {
        if (xy_int && zin)
          stencil_pair_der<DIM, VEC, 0u, PREC, NSV, MODE>(g, ls, Wz, svs, Wz1, m1[0][0],
                                                            m1[0][1], 0u, 0u, al, be, om, c[0][0],
                                                            c[0][1], t[0][0], t[0][1]);
        else if (yz_int && zin)  // x legs only
          stencil_pair_der<DIM, VEC, 12u, PREC, NSV, MODE>(g, ls, Wz, svs, Wz1, m1[0][0],
                                                             m1[0][1], b0, b1, al, be, om,
                                                             c[0][0], c[0][1], t[0][0], t[0][1]);
        else
          stencil_pair_der<DIM, VEC, 63u, PREC, NSV, MODE>(g, ls, Wz, svs, Wz1, m1[0][0],
                                                             m1[0][1], b0 | zb, b1 | zb, al, be,
                                                             om, c[0][0], c[0][1], t[0][0],
                                                             t[0][1]);
      } else if (xy_int && zin) {
#pragma unroll
        for (int v = 0; v < NSO; ++v)
          stencil_pair<DIM, VEC, 0u, PREC>(g, ls, Wz + v * svs, Wz1 + v * svs, m1[v][0],
                                           m1[v][1], 0u, 0u, c[v][0], c[v][1], t[v][0], t[v][1]);
      } else if (yz_int && zin) {  // a warp holding a line's first / last x: x legs only
#pragma unroll
        for (int v = 0; v < NSO; ++v)
          stencil_pair<DIM, VEC, 12u, PREC>(g, ls, Wz + v * svs, Wz1 + v * svs, m1[v][0],
                                            m1[v][1], b0, b1, c[v][0], c[v][1], t[v][0],
                                            t[v][1]);
      } else {
#pragma unroll
        for (int v = 0; v < NSO; ++v)
          stencil_pair<DIM, VEC, 63u, PREC>(g, ls, Wz + v * svs, Wz1 + v * svs, m1[v][0],
                                            m1[v][1], b0 | zb, b1 | zb, c[v][0], c[v][1],
                                            t[v][0], t[v][1]);
      }
#pragma unroll
      for (int v = 0; v < NSO; ++v) {
        m1[v][0] = (BJP || XF) ? pc[v][0] : c[v][0];
        m1[v][1] = (BJP || XF) ? pc[v][1] : c[v][1];
      }
      double o0[NOUT], o1[NOUT];
#pragma unroll
      for (int k = 0; k < NOUT; ++k) o0[k] = o1[k] = 0.0;
      const int64_t gi = gz + gin;
      double px0 = pc[1 % NSO][0], px1 = pc[1 % NSO][1];  // row_update's second M^-1 pair
      if (BJ > 0 && MODE == TM_CL3)  // g := M^-1 p of the streamed p_i: neighbouring lanes
        bj_pair_shfl<BB>(s_bi, amask, i0, S0[sts], S0[sts + 1], px0, px1);
      row_update<MODE, K, NOUT, NRM, (BJ > 0)>(S0, sts, rr, V.zrr + gi, pc[0][0], px0,
                                         c[0][0], c[1][0], t[0][0], t[1][0], al, be, om, g.dinv,
                                         acc, o0);
      if (valid1)
        row_update<MODE, K, NOUT, NRM, (BJ > 0)>(HAS_STR ? S0 + 1 : nullptr, sts, rr, V.zrr + gi + 1,
                                           pc[0][1], px1, c[0][1], c[1][1], t[0][1],
                                           t[1][1], al, be, om, g.dinv, acc, o1);
      if (BJ > 0 && (MODE == TM_RR1 || MODE == TM_INIT1 || MODE == TM_PCI1)) {
        // k := M^-1 r (and l := M^-1 s; p-CG u0 := M^-1 r0): the block's r values sit
        // in neighbouring lanes
        const int ko = MODE == TM_INIT1 ? 2 : 1;
        bj_pair_shfl<BB>(s_bi, amask, i0, o0[0], o1[0], o0[ko % NOUT], o1[ko % NOUT]);
        if (MODE == TM_RR1)
          bj_pair_shfl<BB>(s_bi, amask, i0, o0[2 % NOUT], o1[2 % NOUT], o0[3 % NOUT],
                           o1[3 % NOUT]);
        if (NRM) {
          const int kn = MODE == TM_RR1 ? 1 : 3;
          nrm_add(acc[kn % K], o0[ko % NOUT]);
          nrm_add(acc[kn % K], o1[ko % NOUT]);
          if (MODE == TM_RR1) {
            nrm_add(acc[3 % K], o0[3 % NOUT]);
            nrm_add(acc[3 % K], o1[3 % NOUT]);
          }
        }
      }
      if (T::NOUT > 0) {
#pragma unroll
        for (int k = 0; k < NOUT; ++k) st2<VEC>(outp[k] + gi, o0[k], o1[k], valid1);
      }
    }
    if ((MODE == TM_A || MODE == TM_C) && peer && act && (z0 == 0 || z1 == g.nol)) {
      // peer-memory transport: the slab's first / last plane of z_i (sweep A) or w_{i+1}
      // (sweep C), which this thread stored during the unit, also goes straight into the
      // neighbour's ghost plane over NVLink; the reduction flags this kernel raises
      // publish it (fence below)
      const int64_t po = SEG ? (DIM == 3 ? (y0 + ly) * g.nx : 0) + x0s + cx : toff + r;
      const bool odd = (it & 1) != 0;
      double* const hp_lo = MODE == TM_A ? (odd ? V.hz[1][0] : V.hz[0][0])
                                         : (odd ? V.hw[0][0] : V.hw[1][0]);
      double* const hp_hi = MODE == TM_A ? (odd ? V.hz[1][1] : V.hz[0][1])
                                         : (odd ? V.hw[0][1] : V.hw[1][1]);
      remote |= peer_put<VEC>(hp_lo, hp_hi, outp[3 % NOUT], g.pxy, g.nol, z0, z1, po, valid1);
    }
    __syncthreads();  // unit done: every slot is free
    svc = (svc + nsv) % SVR;
    stc = (stc + nst) % SD;
  }
  TL_STAMP(3);
  // PDL: this CTA's sweep is done; the next kernel may be scheduled (it still waits
  // for this grid's completion, the grid reduction included, before reading anything)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // remote ghost stores visible system-wide before this CTA's ticket: the last CTA's
  // release of the reduction flag then publishes them with the partials
  if (remote) __threadfence_system();
  if (Stash<MODE_>::w && !NRM) {
    // RR1: no scalar of its own; each CTA's block totals of the three dots for RR2
    dd_block_reduce<K>(acc);
    if (tid == 0) {
#pragma unroll
      for (int j = 0; j < STASH_K; ++j) V.stash[(size_t)blockIdx.x * STASH_K + j] = acc[j];
    }
  } else if (T::K > 0) {
    Dd tot[K];
    const int slot = MODE == TM_A ? T_SWEEPA : MODE == TM_C ? T_SWEEPC : MODE == TM_RR2 ? T_RR2
                   : MODE == TM_GAP ? T_GAP : MODE == TM_INIT1 ? T_INIT1 : MODE == TM_INIT2 ? T_INIT2
                   : MODE == TM_CL1 ? T_CL1 : MODE == TM_CL2 ? T_CL2 : MODE == TM_CL3 ? T_CL3
                   : MODE == TM_PC ? T_PC : MODE == TM_PCI1 ? T_PCI1 : MODE == TM_RR1 ? T_RR1
                   : T_PCI2;
    // RR2: dot slots 0, 2, 4 take RR1's stashed block totals (same grid, same units)
    constexpr unsigned OVR = Stash<MODE_>::r ? 0x15u : 0u;
    const bool last = dd_grid_reduce<K, OVR>(acc, part, &sc->counter[slot], tot, V.stash);
    if (Stash<MODE_>::w && tid == 0) {  // RR1N: the dots ride after the four norms
#pragma unroll
      for (int j = 0; j < STASH_K; ++j)
        V.stash[(size_t)blockIdx.x * STASH_K + j] = acc[K - STASH_K + j];
    }
    if (last && tid == 0) {
      TL_STAMP(5);
      if (MODE == TM_A) publish<F_SWEEPA>(sc, h, tot, &s_snap);
      else if (MODE == TM_C) publish<F_SWEEPC>(sc, h, tot, &s_snap);
      else if (MODE == TM_RR2) publish<F_RR2>(sc, h, tot, &s_snap);
      else if (MODE == TM_GAP) publish<F_GAP>(sc, h, tot, &s_snap);
      else if (MODE == TM_INIT1 || MODE == TM_PCI1) publish<F_INIT1>(sc, h, tot, &s_snap);
      else if (MODE == TM_INIT2) publish<F_INIT2>(sc, h, tot, &s_snap);
      else if (MODE == TM_CL1) publish<F_CL1>(sc, h, tot, &s_snap);
      else if (MODE == TM_CL2) publish<F_CL2>(sc, h, tot, &s_snap);
      else if (MODE == TM_CL3) publish<F_CL3>(sc, h, tot, &s_snap);
      else if (MODE == TM_PC) publish<F_PC>(sc, h, tot, &s_snap);
      else if (MODE == TM_RR1) publish<F_RR1>(sc, h, tot, &s_snap);
      else publish<F_PINIT2>(sc, h, tot, &s_snap);
      TL_STAMP(6);
    }
  }
  TL_FLUSH(MODE_);
}

template <int DIM, int MODE_, bool VEC, int BJ = 0, bool SEG = false, bool PEER = false>
__global__ void __launch_bounds__(TNT, 1) t_tile(TileGeo g, Vecs V, Scal* __restrict__ sc,
                                                 Dd* __restrict__ part, Hist h) {
  t_tile_body<DIM, MODE_, VEC, BJ, SEG, PEER>(g, V, sc, part, h);
}

// host-side helper: shared-memory bytes of a t_tile<., MODE, .> launch
template <int M>
inline size_t tile_smem_bytes_t(const TileGeo& g) {
  // + 16 doubles of slack: block-Jacobi reads of a dropped leg may run past the last slot
  return 64 + sizeof(double) * ((size_t)StreamDepth<M>::v * TileTraits<M>::NSTR * g.st_stride +
                                (size_t)SvDepth<M>::v * TileTraits<M>::NSV * g.sv_stride + 16);
}

inline size_t tile_smem_bytes(const TileGeo& g, int mode) {
  switch (mode) {
    case TM_A: return tile_smem_bytes_t<TM_A>(g);
    case TM_C: return tile_smem_bytes_t<TM_C>(g);
    case TM_RR1: return tile_smem_bytes_t<TM_RR1>(g);
    case TM_RR2: return tile_smem_bytes_t<TM_RR2>(g);
    case TM_GAP: return tile_smem_bytes_t<TM_GAP>(g);
    case TM_INIT1: return tile_smem_bytes_t<TM_INIT1>(g);
    case TM_INIT2: return tile_smem_bytes_t<TM_INIT2>(g);
    case TM_CL1: return tile_smem_bytes_t<TM_CL1>(g);
    case TM_CL2: return tile_smem_bytes_t<TM_CL2>(g);
    case TM_CL3: return tile_smem_bytes_t<TM_CL3>(g);
    case TM_PC: return tile_smem_bytes_t<TM_PC>(g);
    case TM_PCI1: return tile_smem_bytes_t<TM_PCI1>(g);
    case TM_AN: return tile_smem_bytes_t<TM_AN>(g);
    case TM_CN: return tile_smem_bytes_t<TM_CN>(g);
    case TM_RR1N: return tile_smem_bytes_t<TM_RR1N>(g);
    case TM_RR2N: return tile_smem_bytes_t<TM_RR2N>(g);
    case TM_INIT1N: return tile_smem_bytes_t<TM_INIT1N>(g);
    case TM_SPB: return tile_smem_bytes_t<TM_SPB>(g);
    case TM_SPD: return tile_smem_bytes_t<TM_SPD>(g);
    default: return tile_smem_bytes_t<TM_PCI2>(g);
  }
}

// Host launch of a tile kernel.  With g.pdl the launch carries programmatic stream
// serialization (PDL): the grid may be scheduled while the previous kernel of the
// stream is still draining; t_tile's griddepcontrol.wait holds every read of that
// kernel's results until it has completed and its writes are visible.
template <typename... A>
inline void tile_launch(void (*kern)(A...), int grid, size_t smem, cudaStream_t s,
                        const TileGeo& g, const Vecs& V, Scal* sc, Dd* part, Hist h) {
  if (!g.pdl) {
    kern<<<grid, TNT, smem, s>>>(g, V, sc, part, h);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(TNT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, g, V, sc, part, h);
}
