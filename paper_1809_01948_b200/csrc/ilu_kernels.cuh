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
//   one compute thread per x-line (y, z); thread (ty, tz) of a TY x TZ line tile
//   handles x = s - ty - tz at step s, taking the -x term from its own registers and
//   the -y / -z terms from its neighbour threads' step s-1 results through shared
//   memory (one named barrier per step).  A wavefront's rows are never contiguous, so
//   global memory is touched by transposed warp instructions only (a block of ILU_K
//   steps of a line = one 64-byte run), staged through shared memory.  Tiles are
//   taken in topological order (diagonals of the tile grid) from a ticket counter by
//   a persistent grid; a tile's boundary lines take the neighbouring tiles' values
//   from global memory after acquiring their progress counters, published every
//   ILU_K steps -- both by helper warps, off the compute warps' path.  The critical
//   path is nx + ny + nz steps plus the tile lags.
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

#ifndef ILU_T
#define ILU_T 256  // threads per CTA (one x-line each)
#endif
#ifndef ILU_K
#define ILU_K 8    // steps between progress publications
#endif
#ifndef ILU_MINB
#define ILU_MINB 1  // register cap of k_ilu_st: CTAs per SM the compiler must allow
#endif
#ifndef ILU_OCC3
#define ILU_OCC3 1  // CTAs per SM of the 3D sweeps (resident tiles = ILU_OCC3 x SMs)
#endif

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
  unsigned long long* prog_f;  // [ntiles] forward progress: (epoch << 32) | steps done (k_ilu_st)
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

__device__ __forceinline__ void cp_async8(double* smem, const double* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(g)
               : "memory");
}
__device__ __forceinline__ double ld_vol_shared(const double* p) {
  double v;
  asm volatile("ld.volatile.shared.f64 %0, [%1];"
               : "=d"(v)
               : "r"((uint32_t)__cvta_generic_to_shared((const void*)p))
               : "memory");
  return v;
}
// predicated, on a shared-window address computed once (no branch, no address
// conversion per copy)
__device__ __forceinline__ void cp_async8_if(uint32_t smem, const double* g, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q cp.async.ca.shared.global [%0], [%1], 8;\n\t}" ::"r"(smem),
      "l"(g), "r"((int)pred)
      : "memory");
}
__device__ __forceinline__ void st_global_if(double* p, double v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f64 [%0], %1;\n\t}" ::"l"(p),
      "d"(v), "r"((int)pred)
      : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// dynamic shared memory of k_ilu_st: per thread, double-buffered, the ILU_K steps' own
// operands (v or y, uinv; the row's result replaces the first), and the two term rings
// (-a / -b terms by step within the block): a column per thread plus, double-buffered,
// ILU_BMAX columns for the neighbouring tile's values (a-side: lines ta = 0, indexed
// by tb; b-side: tb = 0, by ta)
#ifndef ILU_BMAX
#define ILU_BMAX 32
#endif
// Global memory is touched only by "transposed" warp instructions: ILU_K consecutive
// lanes cover the ILU_K consecutive x of one line's block (one 64-byte run), so a warp
// instruction touches 32 / ILU_K lines instead of 32 (a wavefront's rows are never
// contiguous: one row per line).  kIluPfs pads the per-thread operand rows so those
// lanes' shared-memory slots (stride 2 * kIluPfs per step) fall into distinct banks.
static_assert(ILU_K == 4 || ILU_K == 8 || ILU_K == 16, "ILU_K lanes per line must divide a warp");
static_assert(ILU_T % 32 == 0, "whole compute warps; one more warp helps");
constexpr int kIluLpi = 32 / ILU_K;             // lines per transposed warp instruction
constexpr int kIluPfs = ILU_T + kIluLpi / 2;    // operand row stride (2 * kIluPfs = kIluLpi mod 16)
constexpr int kIluRs = ILU_T + 2 * ILU_BMAX + kIluLpi;  // term ring row stride (= kIluLpi mod 16)
constexpr int kIluZc = ILU_T + 2 * ILU_BMAX;     // ring column of zeros (the terms of missing legs)
constexpr int kIluNbj = ILU_BMAX / kIluLpi;     // transposed instructions per boundary block
constexpr size_t kIluSmem = sizeof(double) * (2 * ILU_K * 2 * kIluPfs + 2 * ILU_K * kIluRs);

// named barriers of k_ilu_st (0 = __syncthreads of all kIluThreads threads)
constexpr int kIluThreads = ILU_T + 64;  // compute threads + loader warp + publisher warp
constexpr int kIluBarStep = 1;   // the compute warps' per-step barrier
constexpr int kIluBarFull = 2;   // 2, 3: boundary terms of a block parked (helper arrives)
constexpr int kIluBarEmpty = 4;  // 4, 5: block finished and stored (compute threads arrive)
__device__ __forceinline__ void ilu_bar_step() {
  asm volatile("bar.sync %0, %1;" ::"n"(kIluBarStep), "n"(ILU_T) : "memory");
}
// FULL: the loader warp arrives, the compute threads wait; EMPTY: the compute threads
// arrive, both helper warps wait
__device__ __forceinline__ void ilu_full_sync(int q) {
  asm volatile("bar.sync %0, %1;" ::"r"(kIluBarFull + q), "n"(ILU_T + 32) : "memory");
}
__device__ __forceinline__ void ilu_full_arrive(int q) {
  asm volatile("bar.arrive %0, %1;" ::"r"(kIluBarFull + q), "n"(ILU_T + 32) : "memory");
}
__device__ __forceinline__ void ilu_empty_sync(int q) {
  asm volatile("bar.sync %0, %1;" ::"r"(kIluBarEmpty + q), "n"(ILU_T + 64) : "memory");
}
__device__ __forceinline__ void ilu_empty_arrive(int q) {
  asm volatile("bar.arrive %0, %1;" ::"r"(kIluBarEmpty + q), "n"(ILU_T + 64) : "memory");
}

// Stencil ILU(0) sweep.  BWD = false: out := L^{-1} v; BWD = true: out := U^{-1} out
// (in place; v unused).  ILU_T compute threads (one x-line each) and one helper warp.
// Compute warps: operands are prefetched one block of ILU_K steps ahead by transposed
// cp.async into shared memory; a row's result replaces its operand there and the
// block's results leave by transposed stores.  A step is branch-free: four shared
// loads, the row's arithmetic (+0.0 terms for missing legs; idle lanes compute on
// garbage nobody reads), three shared stores and ONE named barrier of the compute
// warps (a warp's transposed copies and stores serve its own 32 lines: warp-level
// ordering).  Helper warp: everything with a long latency that would otherwise sit
// between two step barriers -- it polls the predecessor tiles' progress, loads their
// boundary values from L2 (transposed) two blocks ahead, parks them as finished terms
// in the rings (FULL / EMPTY named barriers per block parity), and publishes this
// tile's progress (a release store, i.e. a GPU-scope fence) once a block's rows are
// stored.
template <int DIM, bool BWD>
__global__ void __launch_bounds__(kIluThreads, ILU_MINB) k_ilu_st(IluOp P, Scal* __restrict__ sc, int gate,
                                                  const double* __restrict__ v,
                                                  double* __restrict__ out) {
  if (ilu_skip(sc, gate)) return;
  __shared__ int s_tile;
  extern __shared__ __align__(16) double ilu_smem[];
  double* pf = ilu_smem;                                  // [2][ILU_K][2][kIluPfs]
  double* ringA = ilu_smem + 2 * ILU_K * 2 * kIluPfs;     // [ILU_K][kIluRs]
  double* ringB = ringA + ILU_K * kIluRs;                 // [ILU_K][kIluRs]
  unsigned int* ctr = P.ctr + (BWD ? 4 : 0);
  unsigned long long* prog = BWD ? P.prog_b : P.prog_f;
  const unsigned long long ep = (unsigned long long)ilu_epoch(ctr) << 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ta = tid % P.TA, tb = tid / P.TA;
  const int nx = (int)P.nx;
  // leg coefficients in this direction: "m" legs feed the row from a / b / x - 1
  // (forward) or + 1 (backward)
  const double ca = BWD ? P.cap : P.cam, cb = BWD ? P.cbp : P.cbm, cx = BWD ? P.cxp : P.cxm;
  // transposed access: instruction j of a block serves the lines of threads
  // tj0 + j * kIluLpi (this warp's), this lane step kk of the block
  const int kk = lane % ILU_K, lj = lane / ILU_K, tj0 = (tid & ~31) + lj;
  if (tid < ILU_K) ringA[tid * kIluRs + kIluZc] = ringB[tid * kIluRs + kIluZc] = 0.0;
  for (;;) {
    __syncthreads();  // the previous tile's rings and s_tile are no longer read
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
    const bool valid = ta < na_t && tb < nb_t;
    const int64_t a = a0 + (BWD ? na_t - 1 - ta : ta), b = b0 + (BWD ? nb_t - 1 - tb : tb);
    // does the row have the leg towards the previous line in a / b (the dependency)?
    const bool has_a = BWD ? (a + 1 < P.na) : (a > 0);
    const bool has_b = BWD ? (b + 1 < P.nb) : (b > 0);
    const int skew = valid ? ta + tb : (1 << 28);  // x = s - skew; idle lines: x < 0 always
    // where this line's -a / -b terms come from: the neighbour thread's ring column, or
    // (tile-boundary lines) the boundary columns of the block's parity
    // (a line without that leg reads the zero column)
    const int srcA = !has_a ? kIluZc : (ta > 0 ? tid - 1 : ILU_T + tb);
    const int srcB = !has_b ? kIluZc : (tb > 0 ? tid - P.TA : ILU_T + ta);
    const int bndA = has_a && ta == 0 ? ILU_BMAX : 0, bndB = has_b && tb == 0 ? ILU_BMAX : 0;
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
    const int steps = nx + na_t + nb_t - 2;
    // transposed access: 32-bit row offsets inside the tile (host: ilu_setup keeps a
    // tile's extent below 2^30 rows), row (j, block sb) = tile base + jo[j] +/- sb
    const int64_t tbase = a0 * P.sa + b0 * P.sb;
    const double* srcT = (BWD ? out : v) + tbase;
    const double* uinvT = P.uinv + tbase;
    double* outT = out + tbase;
    int jo[ILU_K], jskew[ILU_K];
#pragma unroll
    for (int j = 0; j < ILU_K; ++j) {
      const int tj = tj0 + j * kIluLpi;
      const int tja = tj % P.TA, tjb = tj / P.TA;
      const bool ok = tja < na_t && tjb < nb_t;
      const int lbase = ok ? (BWD ? na_t - 1 - tja : tja) * (int)P.sa + (BWD ? nb_t - 1 - tjb : tjb) * (int)P.sb : 0;
      jskew[j] = ok ? tja + tjb : (1 << 28);  // idle lines: x < 0 always
      jo[j] = ok ? (BWD ? lbase + nx - 1 - kk + jskew[j] : lbase + kk - jskew[j]) : 0;
    }
    // own operands of block [sb, sb + ILU_K) into buffer q (asynchronous copies)
    const uint32_t pfs0 = (uint32_t)__cvta_generic_to_shared(pf + (size_t)kk * 2 * kIluPfs + tj0);
    auto fetch_own = [&](int sb, int q) {
      const uint32_t dq = pfs0 + (uint32_t)(q * ILU_K * 2 * kIluPfs * sizeof(double));
      const int xk = sb + kk;
#pragma unroll
      for (int j = 0; j < ILU_K; ++j) {
        const bool ok = (unsigned)(xk - jskew[j]) < (unsigned)nx;
        const int o = ok ? (BWD ? jo[j] - sb : jo[j] + sb) : 0;
        cp_async8_if(dq + j * kIluLpi * sizeof(double), srcT + o, ok);
        cp_async8_if(dq + (j * kIluLpi + kIluPfs) * sizeof(double), uinvT + o, ok);
      }
      cp_async_commit();
    };
    // results of block [sb, sb + ILU_K) (left in the operand slots of buffer q) -> out
    auto flush_own = [&](int sb, int q) {
      const double* dq = pf + ((size_t)(q * ILU_K + kk) * 2) * kIluPfs + tj0;
      const int xk = sb + kk;
#pragma unroll
      for (int j = 0; j < ILU_K; ++j) {
        const bool ok = (unsigned)(xk - jskew[j]) < (unsigned)nx;
        const int o = ok ? (BWD ? jo[j] - sb : jo[j] + sb) : 0;
        st_global_if(outT + o, dq[j * kIluLpi], ok);
      }
    };
    const int nblk = (steps + ILU_K - 1) / ILU_K;
    if (warp == ILU_T / 32 + 1) {
      // ---- publisher warp: a block's rows are stored -> this tile's progress (a release
      // store, i.e. a GPU-scope fence: kept off every other warp's path)
      for (int n = 0; n < nblk; ++n) {
        ilu_empty_sync(n & 1);
        if (lane == 0)
          st_rel_gpu(prog + tile, ep | (n + 1 < nblk ? (unsigned long long)(n + 1) * ILU_K : 0xFFFFFFFFull));
        __syncwarp();
      }
      continue;
    }
    if (warp == ILU_T / 32) {
      // ---- loader warp: everything that waits on other CTAs.
      // Tile boundaries (a-side: lines ta = 0, slot = tb; b-side: tb = 0, slot = ta): a
      // boundary line of this tile at step s' reads the predecessor's edge line at the
      // same x, which that tile computes at its step s' + TA - 1 (a-side: its thread
      // TA - 1 of the same b line) or s' + TB - 1 (b-side), whatever the line: so for
      // block [sb, sb + ILU_K) the predecessor must have completed sb + ILU_K + TA - 1 /
      // TB - 1 steps (progress = completed steps; polled only when the last value seen
      // does not cover the block).  The block's values are loaded from L2 (transposed,
      // both sides in flight together) and parked as finished terms in the boundary
      // columns of the block's parity; FULL[parity] hands them to the compute warps,
      // EMPTY[parity] (arrived by every compute thread after the block's stores) gives
      // the columns back.
      unsigned long long seen[2] = {0ull, 0ull};
      int64_t sbase[2][kIluNbj];  // the neighbouring tile's row at x = 0 (forward) / nx - 1
#pragma unroll
      for (int side = 0; side < 2; ++side)
#pragma unroll
        for (int j = 0; j < kIluNbj; ++j) {
          const int slot = j * kIluLpi + lj;
          const int sa_ = side ? slot : 0, sb_ = side ? 0 : slot;
          sbase[side][j] = (a0 + (BWD ? na_t - 1 - sa_ : sa_)) * P.sa +
                           (b0 + (BWD ? nb_t - 1 - sb_ : sb_)) * P.sb +
                           (side ? (BWD ? P.sb : -P.sb) : (BWD ? P.sa : -P.sa));
        }
      auto prepare = [&](int m) {
        const int sb = m * ILU_K, q = m & 1;
        double yv[2][kIluNbj], uv[2][kIluNbj];
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          const unsigned long long* pp = side ? pb : pa;
          if (!pp) continue;  // (uniform)
          if (lane == 0) {
            const unsigned long long need =
                ep | (unsigned long long)(sb + ILU_K + (side ? P.TB : P.TA) - 1);
            while (seen[side] < need) {
              seen[side] = ld_acq_gpu(pp);
              if (seen[side] < need) __nanosleep(20);
            }
          }
          __syncwarp();
          const int nslot = side ? na_t : nb_t;
#pragma unroll
          for (int j = 0; j < kIluNbj; ++j) {
            const int xs = sb + kk - (j * kIluLpi + lj);
            const bool ok = j * kIluLpi + lj < nslot && (unsigned)xs < (unsigned)nx;
            const int64_t i = sbase[side][j] + (BWD ? nx - 1 - xs : xs);
            yv[side][j] = ok ? __ldcg(out + i) : 0.0;
            uv[side][j] = (!BWD && ok) ? __ldg(P.uinv + i) : 0.0;
          }
        }
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          if (!(side ? pb : pa)) continue;
          const double c = side ? cb : ca;
          double* ring = (side ? ringB : ringA) + ((kk + ILU_K - 1) % ILU_K) * kIluRs + ILU_T +
                         q * ILU_BMAX + lj;
#pragma unroll
          for (int j = 0; j < kIluNbj; ++j)
            ring[j * kIluLpi] = BWD ? c * yv[side][j] : (c * uv[side][j]) * yv[side][j];
        }
        __syncwarp();
        ilu_full_arrive(q);
      };
      prepare(0);
      if (nblk > 1) prepare(1);
      for (int n = 0; n < nblk; ++n) {
        ilu_empty_sync(n & 1);  // block n: its boundary columns are consumed
        if (n + 2 < nblk) prepare(n + 2);
      }
      continue;
    }
    // ---- compute warps
    double prev = 0.0, uprev = 0.0;  // own value (and forward: its uinv) at x -/+ 1
    fetch_own(0, 0);  // prologue: block 0's operands
    int cur = 0;
    for (int s0 = 0; s0 < steps; s0 += ILU_K) {
      const bool more = s0 + ILU_K < steps;
      __syncwarp();  // buffer cur ^ 1 was flushed by this warp's lanes
      if (more)      // next block's operands
        fetch_own(s0 + ILU_K, cur ^ 1);
      else
        cp_async_commit();  // (empty group: keeps wait_group 1 meaningful)
      cp_async_wait1();  // this block's own copies (this lane's) have landed ...
      __syncwarp();      // ... and the warp's other lanes'
      double* pfc = pf + (size_t)cur * ILU_K * 2 * kIluPfs + tid;
      const double* rA = ringA + srcA + cur * bndA;
      const double* rB = ringB + srcB + cur * bndB;
      const int xs0 = s0 - skew;
      ilu_full_sync(cur);  // the block's boundary terms are parked
      // the step's own operands are read before the previous step's barrier (they do
      // not depend on it): only the two term loads follow a barrier
      double vk = pfc[0], uk = pfc[kIluPfs];
#pragma unroll
      for (int k = 0; k < ILU_K; ++k) {
        // ascending column order: forward -b, -a, -x; backward +x, +a, +b
        // (volatile loads, issued back to back: the compiler otherwise waits for the
        // first term's subtraction before it loads the second)
        const double tA = ld_vol_shared(rA + ((k + ILU_K - 1) % ILU_K) * kIluRs);
        const double tB = ld_vol_shared(rB + ((k + ILU_K - 1) % ILU_K) * kIluRs);
        // a missing leg's term is +0.0 (x - (+0.0) = x bitwise, -0.0 included)
        const double tX = xs0 + k > 0 ? (BWD ? cx * prev : (cx * uprev) * prev) : 0.0;
        const double ui = uk;
        double acc = vk, res;
        if (!BWD) {
          acc = ((acc - tB) - tA) - tX;
          res = acc;
          ringA[k * kIluRs + tid] = (ca * ui) * acc;  // the +a neighbour's -a term
          ringB[k * kIluRs + tid] = (cb * ui) * acc;  // the +b neighbour's -b term
          uprev = ui;
        } else {
          acc = ((acc - tX) - tA) - tB;
          res = acc * ui;
          ringA[k * kIluRs + tid] = ca * res;
          ringB[k * kIluRs + tid] = cb * res;
        }
        pfc[k * 2 * kIluPfs] = res;  // leaves with the block's transposed stores
        prev = res;
        if (k + 1 < ILU_K) {
          vk = pfc[(k + 1) * 2 * kIluPfs];
          uk = pfc[(k + 1) * 2 * kIluPfs + kIluPfs];
        }
        ilu_bar_step();
      }
      flush_own(s0, cur);
      ilu_empty_arrive(cur);
      cur ^= 1;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  ilu_finish(ctr);
}

// 2D stencils: warp-decoupled line wavefront (k_ilu_2d).  A tile is 32 x I2_W
// consecutive lines (y); warp w owns 32 of them, lane l one line, and at its local
// step sigma lane l handles xs = sigma - l, so the -y (+y) term of lane l is lane
// l - 1's previous-step result, one shuffle away.  Lane 0 takes it from warp w - 1's
// lane 31 -- published into a shared-memory ring edge[w - 1] and handed over once
// per block of I2_K steps (counter ecnt; econs gives the ring back-pressure) -- or,
// for w = 0, from the previous tile (global memory after its progress flag).  No
// CTA barrier per step; warps lag their predecessor by about 40 steps.  Own operands
// are prefetched a block ahead into registers; steps are branch-free (selects,
// predicated stores), and the warp is reconverged after the hand-over spins: a warp
// left diverged takes the slow path of every shuffle (measured 5x slower per step).
#define I2_W 8     // warps per CTA
#define I2_K 8     // steps per prefetch block (and per edge hand-over)
#define I2_R 128   // edge ring slots per warp

__device__ __forceinline__ void st_global_pred(double* p, double v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f64 [%0], %1;\n\t}" ::"l"(p),
      "d"(v), "r"((int)pred)
      : "memory");
}


template <bool BWD>
__global__ void __launch_bounds__(32 * I2_W) k_ilu_2d(IluOp P, Scal* __restrict__ sc, int gate,
                                                      const double* __restrict__ v,
                                                      double* __restrict__ out) {
  if (ilu_skip(sc, gate)) return;
  // warp w's lane 31 publishes its per-step results (the -y / +y term of warp w + 1's
  // lane 0) into edge[w] and, once per block, the x-count in ecnt[w]; warp w + 1 reads
  // a whole block of them at its block start (econs = what it has consumed)
  __shared__ double edge[I2_W][I2_R];
  __shared__ volatile int ecnt[I2_W], econs[I2_W];
  __shared__ int s_tile;
  unsigned int* ctr = P.ctr + (BWD ? 4 : 0);
  unsigned long long* prog = BWD ? P.prog_b : P.prog_f;
  const unsigned long long ep = (unsigned long long)ilu_epoch(ctr) << 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double ca = BWD ? P.cap : P.cam, cx = BWD ? P.cxp : P.cxm;
  const int nx = (int)P.nx;
  for (;;) {
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(ctr, 1u);
    if (threadIdx.x < I2_W) {
      ecnt[threadIdx.x] = 0;
      econs[threadIdx.x] = 0;
    }
    __syncthreads();
    const int t = s_tile;
    if (t >= P.ntiles) break;
    const int A = P.order[BWD ? P.ntiles - 1 - t : t];
    const int64_t a0 = (int64_t)A * P.TA;
    const int na_t = (int)((P.na - a0) < P.TA ? (P.na - a0) : P.TA);
    const int ta = 32 * w + lane;
    const bool valid = ta < na_t;
    const int64_t a = a0 + (BWD ? na_t - 1 - ta : ta);
    const bool has_a = BWD ? (a + 1 < P.na) : (a > 0);
    const int64_t base = a * P.sa;
    const int64_t da = BWD ? P.sa : -P.sa;
    const int nvw = (na_t + 31) / 32;  // warps with lines
    if (w < nvw) {
      const int lmax = (na_t - 32 * w) < 32 ? (na_t - 32 * w - 1) : 31;  // last valid lane
      const int wsteps = nx + lmax;
      const bool glob = w == 0 && lane == 0 && has_a;   // dependency from the previous tile
      const bool fring = w > 0 && lane == 0 && has_a;   // ... from warp w - 1
      const bool tring = lane == 31 && w + 1 < nvw;     // lane 31 feeds warp w + 1
      const bool last = ta == na_t - 1;                 // the tile's last line
      const bool succ = BWD ? A > 0 : A + 1 < P.nta;    // ... is read by the next tile
      const unsigned long long* pa = nullptr;
      if (glob) pa = prog + (BWD ? A + 1 : A - 1);
      // own operands of steps [sg0, sg0 + I2_K): registers, one block ahead
      auto fetch = [&](int sg0, double (&o0)[I2_K], double (&o1)[I2_K]) {
#pragma unroll
        for (int k = 0; k < I2_K; ++k) {
          const int xs = sg0 + k - lane;
          const bool ok = valid && xs >= 0 && xs < nx;
          const int64_t i = base + (BWD ? nx - 1 - xs : xs);
          o0[k] = ok ? (BWD ? __ldcg(out + i) : __ldg(v + i)) : 0.0;
          o1[k] = ok ? __ldg(P.uinv + i) : 0.0;
        }
      };
      double up0[I2_K];  // lane 0: the -y / +y term of its block (other warp / other tile)
      auto fetch_up = [&](int sg0) {
#pragma unroll
        for (int k = 0; k < I2_K; ++k) up0[k] = 0.0;
        if (fring) {
          const int need = (sg0 + I2_K) < nx ? (sg0 + I2_K) : nx;
          while (ecnt[w - 1] < need) {
          }
#pragma unroll
          for (int k = 0; k < I2_K; ++k)
            if (sg0 + k < nx) up0[k] = ld_vol_shared(&edge[w - 1][(sg0 + k) & (I2_R - 1)]);
          econs[w] = sg0 + I2_K;
        } else if (glob) {
          const unsigned long long need =
              ep | (unsigned long long)((sg0 + I2_K) < nx ? (sg0 + I2_K) : nx);
          while (ld_acq_gpu(pa) < need) __nanosleep(20);
#pragma unroll
          for (int k = 0; k < I2_K; ++k) {
            const int xs = sg0 + k;
            if (xs < nx) {
              const int64_t i = base + (BWD ? nx - 1 - xs : xs);
              up0[k] = BWD ? ca * __ldcg(out + i + da)
                           : (ca * __ldg(P.uinv + i + da)) * __ldcg(out + i + da);
            }
          }
        }
      };
      double c0[I2_K], c1[I2_K], n0[I2_K], n1[I2_K];
      fetch(0, c0, c1);
      double prev = 0.0, uprev = 0.0, pubprev = 0.0;
      for (int sg0 = 0; sg0 < wsteps; sg0 += I2_K) {
        const bool more = sg0 + I2_K < wsteps;
        if (more) fetch(sg0 + I2_K, n0, n1);
        if (tring) {  // ring back-pressure: warp w + 1 has consumed x < sg0 + I2_K - 31 - I2_R
          while (econs[w + 1] < sg0 + I2_K - 31 - I2_R) {
          }
        }
        fetch_up(sg0);
        // reconverge after lane 0's / lane 31's spins: a warp left diverged would take
        // the slow (WARPSYNC) path of every shuffle in the step loop (measured 5x slower)
        __syncwarp();
        // branch-free steps: every lane computes, selects keep the inactive ones inert
#pragma unroll
        for (int k = 0; k < I2_K; ++k) {
          const int sg = sg0 + k;
          const int xs = sg - lane;
          const bool act = valid && xs >= 0 && xs < nx;
          const double sh = __shfl_up_sync(0xffffffffu, pubprev, 1);  // lane l-1, step sg-1
          const double up = lane == 0 ? up0[k] : sh;
          double res, pub;
          if (!BWD) {  // -y, -x (ascending column order)
            double acc = c0[k];
            const double t1 = acc - up;
            acc = has_a ? t1 : acc;
            const double t2 = acc - (cx * uprev) * prev;
            acc = xs > 0 ? t2 : acc;
            res = acc;
            const double ui = c1[k];
            pub = (ca * ui) * acc;  // the +y neighbour's -y term
            prev = act ? acc : prev;
            uprev = act ? ui : uprev;
          } else {  // +x, +y
            double acc = c0[k];
            const double t1 = acc - cx * prev;
            acc = xs > 0 ? t1 : acc;
            const double t2 = acc - up;
            acc = has_a ? t2 : acc;
            res = acc * c1[k];
            pub = ca * res;
            prev = act ? res : prev;
          }
          {  // predicated store, no branch: the address is clamped for idle lanes
            const int xc = xs < 0 ? 0 : (xs >= nx ? nx - 1 : xs);
            st_global_pred(out + base + (BWD ? nx - 1 - xc : xc), res, act);
          }
          if (tring && act) edge[w][xs & (I2_R - 1)] = pub;
          pubprev = act ? pub : 0.0;
        }
        if (tring) {  // lane 31's x-count after this block
          __threadfence_block();
          const int done = sg0 + I2_K - 31;
          ecnt[w] = done < nx ? done : nx;
        }
        if (last && succ) {  // the successor tile reads only this line, stored by this
          int done = sg0 + I2_K - lane;  // thread: its release store alone orders it
          if (done > nx) done = nx;
          if (done > 0) st_rel_gpu(prog + A, ep | (unsigned long long)done);
        }
        if (more) {
#pragma unroll
          for (int k = 0; k < I2_K; ++k) {
            c0[k] = n0[k];
            c1[k] = n1[k];
          }
        }
      }
    }
    __syncthreads();
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
