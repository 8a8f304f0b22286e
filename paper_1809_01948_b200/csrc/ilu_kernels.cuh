// ilu_kernels.cuh -- the ILU(0) / ICC(0) preconditioner application
// out := M^{-1} v = U^{-1} (L^{-1} v)  (Table 1 ICC(0), P:659-697, P:745;
// SURVEY 8(f) NEXT-4; reading A34).
//
// The factors come from the host (pbicgstab.cu ilu0_factor: Saad's IKJ ILU(0)
// restricted to the pattern, reciprocal pivots uinv).  The application is two
// sequential recurrences,
//   forward   y_i = v_i - sum_{k<i} l_ik y_k          (ascending k)
//   backward  x_i = (y_i - sum_{j>i} u_ij x_j) uinv_i   (ascending j),
// so every row is a function of rows computed before it; the GPU reproduces the
// sequential (oracle) values bitwise by computing each row with the same
// operations in the same order, scheduled along the dependency DAG:
//
// * k_ilu_st<DIM, BWD> -- 5/7-point stencils (constant coefficients; l_ik =
//   fl(c_leg uinv_k), u_ij = c_leg since the zero-fill factorisation of a
//   5/7-point stencil only updates the diagonal).  A "pipelined line wavefront":
//   one thread per x-line (y, z); thread (ty, tz) of a TY x TZ line tile handles x =
//   s - ty - tz at step s, taking the -x term from its own registers and the -y /
//   -z terms from its neighbour threads' step s-1 results through shared memory
//   (one barrier per step).  Tiles are taken in topological order (diagonals of
//   the tile grid) from a ticket counter by a persistent grid; a tile's boundary
//   lines read the neighbouring tiles' values from global memory after acquiring
//   their progress counters, published every ILU_K steps.  The critical path is
//   nx + ny + nz steps (the hyperplane count); at large sizes the kernel is HBM-
//   bound (v, uinv read, out written per row).
// * k_ilu_csr<BWD> -- general CSR: rows in level order (host-computed level sets),
//   one thread per row, persistent grid; a row spins on the per-row epoch flags
//   of its dependencies (all at earlier positions of the order), so no grid-wide
//   barrier per level is needed.
//
// Flags / progress carry an epoch (bumped by the last CTA of every launch) so they
// never need resetting; tickets and the arrival counter are reset by that CTA.
#pragma once
#include <cstdint>

#include "state.cuh"

#define ILU_T 256  // threads per CTA (one x-line each)
#define ILU_K 8    // steps between progress publications

struct IluOp {
  // stencil wavefront (kind 0)
  int32_t dim;
  int64_t nx, na, nb;     // x extent; line extents: a = y (3D) / local y (2D), b = local z (3D) / 1
  int64_t sa, sb;         // strides of a and b (nx; nx*ny in 3D)
  double cam, cbm, cxm;   // lower legs: -y, -z, -x coefficients (a = y, b = z)
  double cap, cbp, cxp;   // upper legs: +y, +z, +x
  int32_t TA, TB;         // line tile
  int32_t nta, ntb, ntiles;
  const int32_t* order;   // [ntiles] tile ids (ta + nta tb) in topological order (diagonals)
  unsigned long long* prog_f;  // [ntiles] forward progress: (epoch << 32) | x-count done
  unsigned long long* prog_b;  // [ntiles] backward progress
  // general CSR (kind 1): strictly lower / upper parts as column-major ELL in row order
  int64_t n;
  int32_t wl, wu;
  const int32_t* lcol;  // [wl][n] local columns (ascending per row), -1 = padding
  const double* lval;   // [wl][n] multipliers l_ik
  const int32_t* ucol;  // [wu][n]
  const double* uval;   // [wu][n] u_ij
  const int32_t* ford;  // [n] rows in forward level order
  const int32_t* bord;  // [n] rows in backward level order
  unsigned int* rflag;  // [n] per-row epoch flags (forward and backward use epochs 2e, 2e+1)
  // both
  const double* uinv;   // [n] reciprocal pivots (no ghosts)
  unsigned int* ctr;    // [8]: ticket f, arrive f, epoch f, -, ticket b, arrive b, epoch b, -
};

// gate: 0 always run, 1 skip when the solve is done, 2 skip unless a replacement fires
__device__ __forceinline__ bool ilu_skip(const Scal* sc, int gate) {
  if (gate == 0 || sc == nullptr) return false;
  if (sc->done) return true;
  return gate == 2 && !sc->rr_fire;
}

__device__ __forceinline__ unsigned long long ld_acq_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acq_gpu32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_gpu32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Kernel prologue / epilogue shared by both kinds: the launch's epoch (read by
// every CTA before any CTA can finish) and the last CTA's reset.
__device__ __forceinline__ unsigned int ilu_epoch(unsigned int* ctr) {
  return *(volatile unsigned int*)(ctr + 2);
}
__device__ __forceinline__ void ilu_finish(unsigned int* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int t = atomicAdd(ctr + 1, 1u);
    if (t == gridDim.x - 1) {  // every CTA has taken its last ticket
      ctr[0] = 0u;
      ctr[1] = 0u;
      atomicAdd(ctr + 2, 1u);  // next launch's epoch
    }
  }
}

// Stencil ILU(0) sweep.  BWD = false: out := L^{-1} v; BWD = true: out := U^{-1} out
// (in place; v unused).
template <int DIM, bool BWD>
__global__ void __launch_bounds__(ILU_T) k_ilu_st(IluOp P, Scal* __restrict__ sc, int gate,
                                                  const double* __restrict__ v,
                                                  double* __restrict__ out) {
  if (ilu_skip(sc, gate)) return;
  __shared__ double pub[2][2][ILU_T];  // [step parity][+a / +b consumer][thread]
  __shared__ int s_tile;
  unsigned int* ctr = P.ctr + (BWD ? 4 : 0);
  unsigned long long* prog = BWD ? P.prog_b : P.prog_f;
  const unsigned long long ep = (unsigned long long)ilu_epoch(ctr) << 32;
  const int tid = threadIdx.x;
  const int ta = tid % P.TA, tb = tid / P.TA;
  // leg coefficients in this direction: "m" legs feed the row from a / b / x - 1
  // (forward) or + 1 (backward)
  const double ca = BWD ? P.cap : P.cam, cb = BWD ? P.cbp : P.cbm, cx = BWD ? P.cxp : P.cxm;
  for (;;) {
    if (tid == 0) s_tile = (int)atomicAdd(ctr, 1u);
    __syncthreads();
    const int t = s_tile;
    if (t >= P.ntiles) break;
    const int tile = P.order[BWD ? P.ntiles - 1 - t : t];
    const int A = tile % P.nta, B = tile / P.nta;
    const int64_t a0 = (int64_t)A * P.TA, b0 = (int64_t)B * P.TB;
    const int na_t = (int)((P.na - a0) < P.TA ? (P.na - a0) : P.TA);
    const int nb_t = (int)((P.nb - b0) < P.TB ? (P.nb - b0) : P.TB);
    // this thread's line (forward: ascending; backward: mirrored inside the tile)
    const int la = BWD ? na_t - 1 - ta : ta, lb = BWD ? nb_t - 1 - tb : tb;
    const bool valid = ta < na_t && tb < nb_t;
    const int64_t a = a0 + la, b = b0 + lb;
    // does the row have the leg towards the previous line in a / b (the dependency)?
    const bool has_a = BWD ? (a + 1 < P.na) : (a > 0);
    const bool has_b = BWD ? (b + 1 < P.nb) : (b > 0);
    const bool own_a = ta > 0, own_b = tb > 0;  // neighbour line inside this tile
    // predecessor tiles (their progress gates the tile-boundary lines)
    const unsigned long long* pa = nullptr;
    const unsigned long long* pb = nullptr;
    if (BWD) {
      if (A + 1 < P.nta) pa = prog + (A + 1) + (int64_t)P.nta * B;
      if (B + 1 < P.ntb) pb = prog + A + (int64_t)P.nta * (B + 1);
    } else {
      if (A > 0) pa = prog + (A - 1) + (int64_t)P.nta * B;
      if (B > 0) pb = prog + A + (int64_t)P.nta * (B - 1);
    }
    const int64_t base = a * P.sa + b * P.sb;
    const int steps = (int)P.nx + na_t + nb_t - 2;
    double prev = 0.0, uprev = 0.0;  // own value (and forward: its uinv) at x -/+ 1
    for (int s0 = 0; s0 < steps; s0 += ILU_K) {
      const int s1 = (s0 + ILU_K) < steps ? (s0 + ILU_K) : steps;
      if (tid == 0) {
        const unsigned long long need =
            ep | (unsigned long long)((int64_t)s1 < P.nx ? s1 : P.nx);
        if (pa) while (ld_acq_gpu(pa) < need) __nanosleep(20);
        if (pb) while (ld_acq_gpu(pb) < need) __nanosleep(20);
      }
      __syncthreads();
      for (int s = s0; s < s1; ++s) {
        const int xs = s - ta - tb;  // steps into this line
        if (valid && xs >= 0 && xs < P.nx) {
          const int64_t x = BWD ? P.nx - 1 - xs : xs;
          const int64_t i = base + x;
          const int q = (s - 1) & 1;
          // ascending column order: forward -b, -a, -x; backward +x, +a, +b
          double acc = BWD ? __ldcg(out + i) : __ldg(v + i);
          if (!BWD) {
            if (has_b) {
              const double term = own_b ? pub[q][1][tid - P.TA]
                                        : (cb * __ldg(P.uinv + i - P.sb)) * __ldcg(out + i - P.sb);
              acc = acc - term;
            }
            if (has_a) {
              const double term = own_a ? pub[q][0][tid - 1]
                                        : (ca * __ldg(P.uinv + i - P.sa)) * __ldcg(out + i - P.sa);
              acc = acc - term;
            }
            if (xs > 0) acc = acc - (cx * uprev) * prev;
            out[i] = acc;
            const double ui = __ldg(P.uinv + i);
            pub[s & 1][0][tid] = (ca * ui) * acc;  // the +a neighbour's -a term
            pub[s & 1][1][tid] = (cb * ui) * acc;  // the +b neighbour's -b term
            prev = acc;
            uprev = ui;
          } else {
            if (xs > 0) acc = acc - cx * prev;
            if (has_a) acc = acc - (own_a ? pub[q][0][tid - 1] : ca * __ldcg(out + i + P.sa));
            if (has_b) acc = acc - (own_b ? pub[q][1][tid - P.TA] : cb * __ldcg(out + i + P.sb));
            const double xi = acc * __ldg(P.uinv + i);
            out[i] = xi;
            pub[s & 1][0][tid] = ca * xi;
            pub[s & 1][1][tid] = cb * xi;
            prev = xi;
          }
        }
        __syncthreads();
      }
      if (tid == 0) {  // x-count every line of the tile has finished after step s1 - 1
        int64_t done = (int64_t)s1 - (na_t - 1) - (nb_t - 1);
        if (done < 0) done = 0;
        if (done > P.nx) done = P.nx;
        __threadfence();
        st_rel_gpu(prog + tile, ep | (unsigned long long)done);
      }
    }
  }
  ilu_finish(ctr);
}

// General CSR ILU(0) sweep, rows in level order, one thread per row.  Warps claim
// 32 consecutive positions of the order from a ticket counter, so every row a
// thread waits for is held by a warp that is already running (no deadlock for any
// grid size).
template <bool BWD>
__global__ void __launch_bounds__(256) k_ilu_csr(IluOp P, Scal* __restrict__ sc, int gate,
                                                 const double* __restrict__ v,
                                                 double* __restrict__ out) {
  if (ilu_skip(sc, gate)) return;
  unsigned int* ctr = P.ctr + (BWD ? 4 : 0);
  // forward and backward share the row flags: forward of launch e stores 2e + 1,
  // backward 2e + 2 (the two epoch counters advance together, one apply = both)
  const unsigned int ep = 2u * ilu_epoch(ctr) + (BWD ? 2u : 1u);
  const int32_t* ord = BWD ? P.bord : P.ford;
  const int lane = threadIdx.x & 31;
  const int W = BWD ? P.wu : P.wl;
  const int32_t* col = BWD ? P.ucol : P.lcol;
  const double* val = BWD ? P.uval : P.lval;
  for (;;) {
    unsigned int p0 = 0;
    if (lane == 0) p0 = atomicAdd(ctr, 32u);
    p0 = __shfl_sync(0xffffffffu, p0, 0);
    if ((int64_t)p0 >= P.n) break;
    const int64_t p = (int64_t)p0 + lane;
    if (p < P.n) {
      const int64_t i = ord[p];
      double acc = BWD ? __ldcg(out + i) : __ldg(v + i);
      for (int q = 0; q < W; ++q) {
        const int32_t c = col[(int64_t)q * P.n + i];
        if (c < 0) break;
        while (ld_acq_gpu32(P.rflag + c) < ep) __nanosleep(20);
        acc = acc - val[(int64_t)q * P.n + i] * __ldcg(out + c);
      }
      if (BWD) acc = acc * __ldg(P.uinv + i);
      __stcg(out + i, acc);
      st_rel_gpu32(P.rflag + i, ep);
    }
  }
  ilu_finish(ctr);
}
