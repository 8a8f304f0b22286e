// csr_kernels.cuh -- general sparse (CSR in, column-major ELL on the device)
// path: the split 4-phase schedule of Algorithm 2.
//
// A general matrix is too expensive to re-apply inside the AXPY sweeps (the
// matrix bytes dominate), so t_i = A M^-1 w_i and v_i = A M^-1 z_i are stored
// as in the paper's own schedule:
//   sweepA (lines 5-12) -> spmvB (lines 13-14) -> sweepC (lines 17-21)
//   [-> rr1 -> rr2 (eq:rr)] -> spmvD (lines 22-23)
// Each row is summed in its stored (ascending column) order (reading A5); a
// padded slot (rows shorter than the ELL width) is skipped, never added.
// Buffers: V.w0 = w, V.w1 = t, V.z0 = z, V.z1 = v, V.zrr = replaced z (A26),
// V.nv = n_i = M^-1 z_i (written by sweep A), V.mv = m_i = M^-1 w_i (written by
// sweep C / rr2 / init2): the SpMVs read n and m, so each gathered operand is
// one vector (the same values the oracle forms in lines 13 and 22).
#pragma once
#include "dd.cuh"
#include "state.cuh"
#include "stencil_kernels.cuh"  // Vecs
#include "tma.cuh"

struct CsrOp {
  int64_t n;             // local rows
  int32_t width;         // ELL slots per row
  const int32_t* col;    // [width][n] column-major, LOCAL index (may be < 0 / >= n: ghosts)
  const double* val;     // [width][n]
  const int32_t* len;    // [n] row lengths, or nullptr when every row has `width` entries
  const double* dinv;    // [n + 2H] ghosted Jacobi inverse diagonal (A3)
  int32_t bj;            // preconditioner block size: 1 Jacobi, 2..32 block Jacobi (A33)
  const double* binv;    // bj > 1: [n][bj] row j of its block's inverse (row-major)
  // window SpMV operands, sliced ELL (SELL-32): rows in slices of 32 (one warp), slot k
  // of the slice's 32 rows contiguous -- element (j, k) at ((j / 32) width + k) 32 + j % 32,
  // so every load of a row's slots is the row's base + an immediate k * 32 elements
  const double* sval;    // values (padding 0)
  const int16_t* sdcol;  // column - row (|.| <= half bandwidth <= (WRS - 3 WTB) / 2)
};

// Preconditioner kinds of the per-row kernels' PK template parameter: Jacobi and
// block Jacobi are applied inside the kernels (prec_row); with ILU(0) (reading A34)
// the preconditioned vectors k, l, m, n (and classic BiCGStab's M^-1 p, M^-1 q) are
// produced by the k_ilu_* sweeps between the kernels, which read them from memory.
#define PK_JAC 0
#define PK_BJ 1
#define PK_ILU 2

// M^{-1} applied to the value v of row j (reading A3 / A33).  Jacobi: fl(dinv_j v).
// Block Jacobi: the bj rows of a block are bj consecutive lanes of one warp
// (blocks are aligned and n_local % bj == 0), so the block's values are read by
// shuffles and (M^{-1}v)_j = sum_k binv_jk v_{kb+k}, ascending k from +0.0 -- the
// oracle's order.  Every lane of the warp must call it (warp-uniform loops, WROW_LOOP).
// BJ = false: Jacobi with dj = dinv_j preloaded by the caller (0 on idle lanes).
template <bool BJ>
__device__ __forceinline__ double prec_row(const CsrOp& A, int64_t j, bool in, double v,
                                          double dj) {
  if (!BJ) return dj * v;
  const int lane = threadIdx.x & 31;
  const int base = lane & ~(A.bj - 1);
  const double* __restrict__ row = A.binv + (in ? j : 0) * A.bj;  // 16-byte aligned (bj even)
  double acc = 0.0;
  for (int k = 0; k < A.bj; k += 2) {
    const double2 rw = in ? __ldg(reinterpret_cast<const double2*>(row + k)) : make_double2(0.0, 0.0);
    const double v0 = __shfl_sync(0xffffffffu, v, base + k);
    const double v1 = __shfl_sync(0xffffffffu, v, base + k + 1);
    acc = acc + rw.x * v0;
    acc = acc + rw.y * v1;
  }
  return acc;
}

// fl(A v)_j or fl(A M^-1 v)_j, summed left to right in stored (ascending
// column) order from +0.0 (A5).  Slots are processed in groups of ELL_U with all
// loads of a group issued before its adds (memory-level parallelism); the
// matrix is streamed with evict-first loads so L1/L2 keep the gathered window.
#define ELL_U 9
#define WIN_U 27
template <bool PREC>
__device__ __forceinline__ double ell_row(const CsrOp& A, const double* __restrict__ v, int64_t j) {
  const int len = A.len ? A.len[j] : A.width;
  double acc = 0.0;
  int p = 0;
  for (; p + ELL_U <= len; p += ELL_U) {
    int c[ELL_U];
    double a[ELL_U], x[ELL_U];
#pragma unroll
    for (int u = 0; u < ELL_U; ++u) {
      c[u] = __ldcs(A.col + (int64_t)(p + u) * A.n + j);
      a[u] = __ldcs(A.val + (int64_t)(p + u) * A.n + j);
    }
#pragma unroll
    for (int u = 0; u < ELL_U; ++u)
      x[u] = PREC ? __ldg(A.dinv + c[u]) * __ldg(v + c[u]) : __ldg(v + c[u]);
#pragma unroll
    for (int u = 0; u < ELL_U; ++u) acc = acc + a[u] * x[u];
  }
  for (; p < len; ++p) {
    const int c = __ldcs(A.col + (int64_t)p * A.n + j);
    const double a = __ldcs(A.val + (int64_t)p * A.n + j);
    const double x = PREC ? __ldg(A.dinv + c) * __ldg(v + c) : __ldg(v + c);
    acc = acc + a * x;
  }
  return acc;
}

#define ROW_LOOP for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < A.n; \
                      j += (int64_t)gridDim.x * blockDim.x)
// warp-uniform variant for steps that apply M^{-1} (prec_row shuffles): the whole
// warp iterates while any lane has a row; `in` marks the lanes that do
// (every prec_row call sits in converged code: loads/stores are predicated on `in`)
#define WROW_LOOP                                                                     \
  for (int64_t j0_ = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~(int64_t)31; \
       j0_ < A.n; j0_ += (int64_t)gridDim.x * blockDim.x) {                          \
    const int64_t j = j0_ + (threadIdx.x & 31);                                       \
    const bool in = j < A.n;                                                          \
    const double dj = (!BJ && in) ? A.dinv[j] : 0.0; /* Jacobi: dinv_j, loaded once */
#define WROW_END }

// NRM (automated replacement): the step's reduction also carries the
// Dot2 sums of squares of the vectors the bound f^r needs (reading A30)
__device__ __forceinline__ void c_nrm(Dd& a, double v) { dd_fma(a, v, v); }

template <bool NRM, int PK>
__global__ void __launch_bounds__(256) c_init1(CsrOp A, Vecs V, Scal* __restrict__ sc,
                                               Dd* __restrict__ part, Hist h) {
  constexpr bool BJ = PK == PK_BJ;
  constexpr int K = NRM ? 4 : 2;
  Dd acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = dd_zero();
  WROW_LOOP
    const double bj = in ? V.b[j] : 0.0;
    const double rj = in ? bj - ell_row<false>(A, V.x, j) : 0.0;
    // k0 := M^-1 r0 (ILU(0): k_ilu_* after this kernel)
    const double kj = PK == PK_ILU ? 0.0 : prec_row<BJ>(A, j, in, rj, dj);
    if (in) {
      V.r[j] = rj;
      V.rh[j] = rj;
      if (PK != PK_ILU) V.k[j] = kj;
      dd_fma(acc[0], rj, rj);
      dd_fma(acc[1], bj, bj);
      if (NRM) {
        c_nrm(acc[2 % K], V.x[j]);
        c_nrm(acc[3 % K], kj);
      }
    }
  WROW_END
  Dd tot[K];
  if (dd_grid_reduce<K>(acc, part, &sc->counter[T_INIT1], tot) && threadIdx.x == 0)
    publish<F_INIT1>(sc, h, tot);
}

template <int PK>
__global__ void __launch_bounds__(256) c_init2(CsrOp A, Vecs V, Scal* __restrict__ sc,
                                               Dd* __restrict__ part, Hist h) {
  constexpr bool BJ = PK == PK_BJ;
  Dd acc[1] = {dd_zero()};
  WROW_LOOP
    const double wj = in ? ell_row<false>(A, V.k, j) : 0.0;  // w0 = A k0 = A M^-1 r0
    // m0 = M^-1 w0 (line 2; ILU(0): k_ilu_* after this kernel)
    const double mj = PK == PK_ILU ? 0.0 : prec_row<BJ>(A, j, in, wj, dj);
    if (in) {
      V.w0[j] = wj;
      if (PK != PK_ILU) V.mv[j] = mj;
      dd_fma(acc[0], V.rh[j], wj);
    }
  WROW_END
  Dd tot[1];
  if (dd_grid_reduce<1>(acc, part, &sc->counter[T_INIT2], tot) && threadIdx.x == 0)
    publish<F_INIT2>(sc, h, tot);
}

// lines 5-12 with stored t_i, v_{i-1}; n_{i-1} = M^-1 z_{i-1} (pre-replacement, A26)
template <bool NRM, int PK>
__global__ void __launch_bounds__(256) c_sweepA(CsrOp A, Vecs V, Scal* __restrict__ sc,
                                                Dd* __restrict__ part, Hist h) {
  constexpr bool BJ = PK == PK_BJ;
  constexpr int K = NRM ? 12 : 2;
  if (sc->done) return;
  const double al = sc->alpha, be = sc->beta, om = sc->omega;
  const bool rr = sc->use_rr != 0;
  Dd acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = dd_zero();
  WROW_LOOP
    const double wc = in ? V.w0[j] : 0.0, zc = in ? V.z0[j] : 0.0;
    // m_i, n_{i-1} (ILU(0): as stored by k_ilu_*; nv still holds the pre-replacement n, A26)
    const double m = PK == PK_ILU ? (in ? V.mv[j] : 0.0) : prec_row<BJ>(A, j, in, wc, dj);
    const double n = PK == PK_ILU ? (in ? V.nv[j] : 0.0) : prec_row<BJ>(A, j, in, zc, dj);
    double zn = 0.0;
    if (in) {
      const double zo = rr ? V.zrr[j] : zc;
      const double t = V.w1[j], v = V.z1[j];
      const double lj = V.l[j];
      const double gn = V.k[j] + be * (V.g[j] - om * lj);
      const double sn = wc + be * (V.s[j] - om * zo);
      const double ln = m + be * (lj - om * n);
      zn = t + be * (zo - om * v);
      const double q = V.r[j] - al * sn;
      const double y = wc - al * zn;
      dd_fma(acc[0], q, y);
      dd_fma(acc[1], y, y);
      if (NRM) {  // k, w, m, t, g, s, l, z, q, y of iteration i
        c_nrm(acc[2 % K], V.k[j]); c_nrm(acc[3 % K], wc); c_nrm(acc[4 % K], m);
        c_nrm(acc[5 % K], t); c_nrm(acc[6 % K], gn); c_nrm(acc[7 % K], sn);
        c_nrm(acc[8 % K], ln); c_nrm(acc[9 % K], zn); c_nrm(acc[10 % K], q);
        c_nrm(acc[11 % K], y);
      }
      V.g[j] = gn;
      V.s[j] = sn;
      V.l[j] = ln;
      V.z0[j] = zn;
    }
    if (PK != PK_ILU) {
      const double nj = prec_row<BJ>(A, j, in, zn, dj);  // n_i = M^-1 z_i (line 13)
      if (in) V.nv[j] = nj;
    }
  WROW_END
  Dd tot[K];
  if (dd_grid_reduce<K>(acc, part, &sc->counter[T_SWEEPA], tot) && threadIdx.x == 0)
    publish<F_SWEEPA>(sc, h, tot);
}

// ---------------------------------------------------------------------------
// SpMV y = A u of one step, with the step's epilogue (store, dots).  The same
// modes run as the gather kernel c_spmv_g (any matrix) and as the window kernel
// c_spmv_win (banded matrices, operand window staged in shared memory).
enum SpmvMode {
  SP_V = 0,   // Alg. 2 line 14: v_i = A n_i
  SP_T,       // Alg. 2 line 23: t_{i+1} = A m_{i+1}
  SP_CLS,     // Alg. 1 lines 5-6: s_i = A (M^-1 p_i) [mv]; (r^0, s_i)
  SP_CLY,     // Alg. 1 lines 10-11: y_i = A (M^-1 q_i) [nv]; q_i = r_i - alpha s_i; (q,y), (y,y)
  SP_PCW0,    // p-CG init: w0 = A u0 [k]; m0 = M^-1 w0; (r0,u0), (w0,u0)
  SP_PCN,     // p-CG: n_i = A m_i [mv]
  SP_GAP,     // eq:res_gap: ||(b - A x) - r|| [x]
  SP_I1,      // Alg. 2 line 2 (Jacobi): r0 = b - A x0, r^0 = r0, k0 = M^-1 r0; (r0,r0), (b,b) [x]
  SP_I2,      // Alg. 2 line 3 (Jacobi): w0 = A k0, m0 = M^-1 w0; (r^0, w0) [k]
  SP_N
};
template <int M> struct SpmvK { enum { K = 0 }; };
template <> struct SpmvK<SP_GAP> { enum { K = 1 }; };
template <> struct SpmvK<SP_I1> { enum { K = 2 }; };
template <> struct SpmvK<SP_I2> { enum { K = 1 }; };
template <> struct SpmvK<SP_CLS> { enum { K = 1 }; };
template <> struct SpmvK<SP_CLY> { enum { K = 2 }; };
template <> struct SpmvK<SP_PCW0> { enum { K = 2 }; };

template <int M>
__device__ __forceinline__ const double* spmv_in(const Vecs& V) {
  return (M == SP_V || M == SP_CLY) ? V.nv : (M == SP_PCW0 || M == SP_I2) ? V.k
       : (M == SP_GAP || M == SP_I1) ? V.x : V.mv;
}

template <int M, int K>
__device__ __forceinline__ void spmv_epi(const CsrOp& A, const Vecs& V, int64_t j, double y,
                                         double al, Dd* acc) {
  if (M == SP_V || M == SP_CLY || M == SP_PCN) __stcs(V.z1 + j, y);
  if (M == SP_T) __stcs(V.w1 + j, y);
  if (M == SP_CLS) {
    V.s[j] = y;
    dd_fma(acc[0], V.rh[j], y);
  } else if (M == SP_CLY) {
    const double q = V.r[j] - al * V.s[j];  // line 8, recomputed (same value)
    dd_fma(acc[0], q, y);
    dd_fma(acc[1 % K], y, y);
  } else if (M == SP_GAP) {
    const double d = (V.b[j] - y) - V.r[j];  // c_gap's expression
    dd_fma(acc[0], d, d);
  } else if (M == SP_I1) {  // c_init1's expressions (Jacobi)
    const double bj = V.b[j];
    const double rj = bj - y;
    V.r[j] = rj;
    V.rh[j] = rj;
    V.k[j] = A.dinv[j] * rj;
    dd_fma(acc[0], rj, rj);
    dd_fma(acc[1 % K], bj, bj);
  } else if (M == SP_I2) {  // c_init2's expressions (Jacobi)
    V.w0[j] = y;
    V.mv[j] = A.dinv[j] * y;
    dd_fma(acc[0], V.rh[j], y);
  } else if (M == SP_PCW0) {
    V.w0[j] = y;  // m0 = M^-1 w0 follows in c_prec_mv (warp-uniform M^-1)
    const double u = V.k[j];
    dd_fma(acc[0], V.r[j], u);
    dd_fma(acc[1 % K], y, u);
  }
}

template <int M>
__device__ __forceinline__ void spmv_fin(Scal* sc, Hist h, Dd* part, Dd (&acc)[SpmvK<M>::K > 0 ? SpmvK<M>::K : 1]) {
  constexpr int K = SpmvK<M>::K > 0 ? SpmvK<M>::K : 1;
  if (SpmvK<M>::K == 0) return;
  Dd tot[K];
  const int slot = M == SP_CLS ? T_CL1 : M == SP_CLY ? T_CL2 : M == SP_GAP ? T_GAP
                 : M == SP_I1 ? T_INIT1 : M == SP_I2 ? T_INIT2 : T_PCI2;
  if (dd_grid_reduce<K>(acc, part, &sc->counter[slot], tot) && threadIdx.x == 0) {
    if (M == SP_CLS) publish<F_CL1>(sc, h, tot);
    else if (M == SP_CLY) publish<F_CL2>(sc, h, tot);
    else if (M == SP_GAP) publish<F_GAP>(sc, h, tot);
    else if (M == SP_I1) publish<F_INIT1>(sc, h, tot);
    else if (M == SP_I2) publish<F_INIT2>(sc, h, tot);
    else publish<F_PINIT2>(sc, h, tot);
  }
}

// gather version (any sparsity within the ghost band)
template <int M>
__global__ void __launch_bounds__(256) c_spmv_g(CsrOp A, Vecs V, Scal* __restrict__ sc,
                                                Dd* __restrict__ part, Hist h) {
  constexpr int K = SpmvK<M>::K > 0 ? SpmvK<M>::K : 1;
  if (M != SP_PCW0 && sc->done) return;
  const double al = sc->alpha;
  const double* __restrict__ u = spmv_in<M>(V);
  Dd acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = dd_zero();
  ROW_LOOP { spmv_epi<M, K>(A, V, j, ell_row<false>(A, u, j), al, acc); }
  spmv_fin<M>(sc, h, part, acc);
}

// line 14: v_i = A n_i (gather version; c_spmv_win is the staged one)
__global__ void __launch_bounds__(256) c_spmvB(CsrOp A, Vecs V, Scal* __restrict__ sc) {
  if (sc->done) return;
  ROW_LOOP { V.z1[j] = ell_row<false>(A, V.nv, j); }
}

// lines 17-21
template <bool NRM, int PK>
// (256, 3): <= 85 registers keep 3 CTAs per SM for the block-Jacobi instance too
__global__ void __launch_bounds__(256, 3) c_sweepC(CsrOp A, Vecs V, Scal* __restrict__ sc,
                                                Dd* __restrict__ part, Hist h) {
  constexpr bool BJ = PK == PK_BJ;
  constexpr int K = NRM ? 9 : 5;
  if (sc->done) return;
  const double al = sc->alpha, om = sc->omega;
  Dd acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = dd_zero();
  WROW_LOOP
    const double wc = in ? V.w0[j] : 0.0, zc = in ? V.z0[j] : 0.0;
    // m_i, n_i (ILU(0): as stored by k_ilu_*)
    const double m = PK == PK_ILU ? (in ? V.mv[j] : 0.0) : prec_row<BJ>(A, j, in, wc, dj);
    const double n = PK == PK_ILU ? (in ? V.nv[j] : 0.0) : prec_row<BJ>(A, j, in, zc, dj);
    double wn = 0.0;
    if (in) {
    const double t = V.w1[j], v = V.z1[j];
    const double sj = V.s[j];
    const double u = V.k[j] - al * V.l[j];
    const double q = V.r[j] - al * sj;
    const double y = wc - al * zc;
    const double xj = V.x[j];
    const double xn = (xj + al * V.g[j]) + om * u;
    const double rn = q - om * y;
    const double kn = u - om * (m - al * n);
    wn = y - om * (t - al * v);
    const double rhj = V.rh[j];
    dd_fma(acc[0], rhj, rn);
    dd_fma(acc[1 % K], rhj, wn);
    dd_fma(acc[2 % K], rhj, sj);
    dd_fma(acc[3 % K], rhj, zc);
    dd_fma(acc[4 % K], rn, rn);
    if (NRM) {  // x_i, u_i, n_i, v_i
      c_nrm(acc[5 % K], xj); c_nrm(acc[6 % K], u); c_nrm(acc[7 % K], n);
      c_nrm(acc[8 % K], v);
    }
    V.x[j] = xn;
    V.r[j] = rn;
    V.k[j] = kn;
    V.w0[j] = wn;
    }
    if (PK != PK_ILU) {
      const double mn = prec_row<BJ>(A, j, in, wn, dj);  // m_{i+1} = M^-1 w_{i+1} (line 22)
      if (in) V.mv[j] = mn;
    }
  WROW_END
  Dd tot[K];
  if (dd_grid_reduce<K>(acc, part, &sc->counter[T_SWEEPC], tot) && threadIdx.x == 0)
    publish<F_SWEEPC>(sc, h, tot);
}

// ---------------------------------------------------------------------------
// TMA-staged sweeps (Jacobi): the same row arithmetic as c_sweepA / c_sweepC, with
// every input vector streamed into shared memory as CST_R-row chunks by bulk copies
// (cp.async.bulk + mbarrier, a two-stage ring: one chunk in flight while the other
// is computed), two rows per thread (16-byte shared loads, 16-byte streaming
// stores).  Chunks go to CTAs round-robin (static, deterministic); one CTA per SM.
#define CST_R 1024   // rows per chunk
#define CST_T 512    // threads per CTA (a row pair each)
#define CST_NIN 12   // input vectors staged per chunk (max over the two sweeps)
constexpr size_t kCstSmem = 64 + 2 * (size_t)CST_NIN * CST_R * sizeof(double);

// BJ (block Jacobi, A33): dinv is not staged; (M^-1 v)_j = sum_k binv_jk v_{block+k},
// ascending k from +0.0 (prec_row's order).  Blocks are aligned (b | CST_R) and a
// block's rows are the row pairs of b/2 consecutive lanes of one warp, so its values
// come by shuffles from those lanes' registers (old and new z, w alike).
// STS: the stencil split schedule (option schedule 2; k_sweepA2 / k_sweepC2's steps):
// scalar dinv (dsc), w and z double-buffered by iteration parity, t, v in tv, vv, and no
// M^-1 output (the stand-alone tile SpMVs apply the Jacobi scaling per leg).
template <int SW, bool NRM, bool BJ, bool STS = false>  // SW 0: sweep A (l. 5-12), 1: C (l. 17-21)
__global__ void __launch_bounds__(CST_T, 1) c_sweep_tma(CsrOp A, Vecs V, Scal* __restrict__ sc,
                                                        Dd* __restrict__ part, Hist h,
                                                        double dsc) {
  constexpr int K = SW == 0 ? (NRM ? 12 : 2) : (NRM ? 9 : 5);
  constexpr int NOUT = STS ? 4 : 5;
  static_assert(!(STS && (BJ || NRM)), "split stencil sweeps: Jacobi, no bound norms");
  if (sc->done) return;
  const int it = sc->iter;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  double* buf = reinterpret_cast<double*>(smem_raw + 64);
  const int tid = threadIdx.x;
  const double al = sc->alpha, be = sc->beta, om = sc->omega;
  const bool rr = SW == 0 && sc->use_rr != 0;
  // staged inputs, fixed slots (a bit of `mask` per staged vector)
  //   A: w, z (pre-replacement), t, v, l, k, g, s, r, dinv, replaced z
  //   C: w, z, t, v, s, k, l, r, x, g, r^0, dinv
  const double* in[CST_NIN];
  unsigned mask;
  const bool odd = (it & 1) != 0;
  if (SW == 0) {
    const double* wv = STS ? (odd ? V.w1 : V.w0) : V.w0;  // w_i
    const double* zv = STS ? (odd ? V.z0 : V.z1) : V.z0;  // z_{i-1} pre-replacement
    const double* a[11] = {wv, zv, STS ? V.tv : V.w1, STS ? V.vv : V.z1, V.l, V.k, V.g, V.s,
                           V.r, A.dinv, V.zrr};
    mask = (BJ || STS ? 0x1FFu : 0x3FFu) | (rr ? 0x400u : 0u);
#pragma unroll
    for (int v = 0; v < 11; ++v) in[v] = a[v];
    in[11] = nullptr;
  } else {
    const double* wv = STS ? (odd ? V.w1 : V.w0) : V.w0;  // w_i
    const double* zv = STS ? (odd ? V.z1 : V.z0) : V.z0;  // z_i
    const double* a[12] = {wv, zv, STS ? V.tv : V.w1, STS ? V.vv : V.z1, V.s, V.k, V.l, V.r,
                           V.x, V.g, V.rh, A.dinv};
    mask = BJ || STS ? 0x7FFu : 0xFFFu;
#pragma unroll
    for (int v = 0; v < 12; ++v) in[v] = a[v];
    // SpMV_D may run before the finalize step advances iter (P ranks, overlap): tell it
    // where w_{i+1} is
    if (STS && blockIdx.x == 0 && tid == 0) sc->spd_par = (it + 1) & 1;
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t nch = (A.n + CST_R - 1) / CST_R;
  auto stage = [&](int slot, int64_t c) {
    const int64_t j0 = c * CST_R;
    const int64_t rows = (A.n - j0) < CST_R ? (A.n - j0) : CST_R;
    const uint32_t bytes = (uint32_t)((rows * 8 + 15) & ~15LL);  // vectors carry 2 slack rows
    mbar_arrive_expect_tx(&bar[slot], bytes * (uint32_t)__popc(mask));
#pragma unroll
    for (int v = 0; v < CST_NIN; ++v)  // unrolled: `in` stays in registers
      if ((mask >> v) & 1u)
        bulk_g2s(buf + ((size_t)slot * CST_NIN + v) * CST_R, in[v] + j0, bytes, &bar[slot]);
  };
  // block Jacobi: M^-1 of the vector whose rows j, j+1 this thread holds (v0, v1); every
  // lane of the warp calls it (shuffles), idle lanes with zeros
  auto bjpair = [&](double v0, double v1, int64_t j, bool act, double& o0, double& o1) {
    const int lane = tid & 31;
    const int base = lane & ~(A.bj / 2 - 1);  // lane holding the block's rows 0, 1
    const double* __restrict__ r0 = A.binv + (act ? j : 0) * A.bj;  // 16-byte aligned rows
    const double* __restrict__ r1 = r0 + A.bj;
    double a = 0.0, c = 0.0;
    for (int k = 0; k < A.bj; k += 2) {
      const double e0 = __shfl_sync(0xffffffffu, v0, base + k / 2);
      const double e1 = __shfl_sync(0xffffffffu, v1, base + k / 2);
      const double2 p = act ? __ldg(reinterpret_cast<const double2*>(r0 + k)) : make_double2(0, 0);
      const double2 q = act ? __ldg(reinterpret_cast<const double2*>(r1 + k)) : make_double2(0, 0);
      a = a + p.x * e0;
      a = a + p.y * e1;
      c = c + q.x * e0;
      c = c + q.y * e1;
    }
    o0 = a;
    o1 = c;
  };
  Dd acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = dd_zero();
  if (tid == 0 && (int64_t)blockIdx.x < nch) stage(0, blockIdx.x);
  uint32_t ph = 0;
  int slot = 0;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, slot ^= 1) {
    // the other slot was released by the previous chunk's closing barrier
    if (tid == 0 && c + gridDim.x < nch) stage(slot ^ 1, c + gridDim.x);
    mbar_wait(&bar[slot], (ph >> slot) & 1u);
    ph ^= 1u << slot;
    const int64_t j = c * CST_R + 2 * tid;
    const bool act = j < A.n;  // (block Jacobi: n % b == 0, blocks all-in or all-out)
    const bool valid1 = j + 1 < A.n;
    const double* B = buf + (size_t)slot * CST_NIN * CST_R;
    double x0[CST_NIN], x1[CST_NIN];
#pragma unroll
    for (int v = 0; v < CST_NIN; ++v) {
      if (act && ((mask >> v) & 1u)) {
        const double2 q = *reinterpret_cast<const double2*>(B + (size_t)v * CST_R + 2 * tid);
        x0[v] = q.x;
        x1[v] = q.y;
      } else {
        x0[v] = x1[v] = 0.0;
      }
    }
    // M^-1 of w and z (block Jacobi: by shuffles; n % b == 0, so an active thread's
    // second row is valid)
    double mw[2] = {0.0, 0.0}, nz[2] = {0.0, 0.0};
    if (BJ) {
      bjpair(x0[0], x1[0], j, act, mw[0], mw[1]);
      bjpair(x0[1], x1[1], j, act, nz[0], nz[1]);
    }
    double o0[5] = {0, 0, 0, 0, 0}, o1[5] = {0, 0, 0, 0, 0};
    if (act) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double* xv = e == 0 ? x0 : x1;
        double* o = e == 0 ? o0 : o1;
        if (e == 1 && !valid1) break;
        if (SW == 0) {  // identical expressions to c_sweepA
          const double wc = xv[0], zc = xv[1], t = xv[2], v = xv[3], lj = xv[4];
          const double dj = STS ? dsc : xv[9];
          const double m = BJ ? mw[e] : dj * wc, n = BJ ? nz[e] : dj * zc;  // m_i, n_{i-1}
          const double zo = rr ? xv[10] : zc;
          const double gn = xv[5] + be * (xv[6] - om * lj);
          const double sn = wc + be * (xv[7] - om * zo);
          const double ln = m + be * (lj - om * n);
          const double zn = t + be * (zo - om * v);
          const double q = xv[8] - al * sn;
          const double y = wc - al * zn;
          dd_fma(acc[0], q, y);
          dd_fma(acc[1 % K], y, y);
          if (NRM) {
            c_nrm(acc[2 % K], xv[5]); c_nrm(acc[3 % K], wc); c_nrm(acc[4 % K], m);
            c_nrm(acc[5 % K], t); c_nrm(acc[6 % K], gn); c_nrm(acc[7 % K], sn);
            c_nrm(acc[8 % K], ln); c_nrm(acc[9 % K], zn); c_nrm(acc[10 % K], q);
            c_nrm(acc[11 % K], y);
          }
          o[0] = gn; o[1] = sn; o[2] = ln; o[3] = zn;
          o[4] = BJ ? 0.0 : dj * zn;  // n_i (line 13); block Jacobi below
        } else {  // identical expressions to c_sweepC
          const double wc = xv[0], zc = xv[1], t = xv[2], v = xv[3], sj = xv[4];
          const double dj = STS ? dsc : xv[11];
          const double m = BJ ? mw[e] : dj * wc, n = BJ ? nz[e] : dj * zc;  // m_i, n_i
          const double u = xv[5] - al * xv[6];
          const double q = xv[7] - al * sj;
          const double y = wc - al * zc;
          const double xj = xv[8];
          const double xn = (xj + al * xv[9]) + om * u;
          const double rn = q - om * y;
          const double kn = u - om * (m - al * n);
          const double wn = y - om * (t - al * v);
          const double rhj = xv[10];
          dd_fma(acc[0], rhj, rn);
          dd_fma(acc[1 % K], rhj, wn);
          dd_fma(acc[2 % K], rhj, sj);
          dd_fma(acc[3 % K], rhj, zc);
          dd_fma(acc[4 % K], rn, rn);
          if (NRM) {
            c_nrm(acc[5 % K], xj); c_nrm(acc[6 % K], u); c_nrm(acc[7 % K], n);
            c_nrm(acc[8 % K], v);
          }
          o[0] = xn; o[1] = rn; o[2] = kn; o[3] = wn;
          o[4] = BJ ? 0.0 : dj * wn;  // m_{i+1} (line 22); block Jacobi below
        }
      }
    }
    if (BJ) bjpair(o0[3], o1[3], j, act, o0[4], o1[4]);  // M^-1 of the new z (A) / w (C)
    if (act) {
      double* out[5];
      if (SW == 0) {
        out[0] = V.g; out[1] = V.s; out[2] = V.l;
        out[3] = STS ? (odd ? V.z1 : V.z0) : V.z0;  // z_i
        out[4] = V.nv;
      } else {
        out[0] = V.x; out[1] = V.r; out[2] = V.k;
        out[3] = STS ? (odd ? V.w0 : V.w1) : V.w0;  // w_{i+1}
        out[4] = V.mv;
      }
#pragma unroll
      for (int k = 0; k < NOUT; ++k) {
        if (valid1) {
          __stcs(reinterpret_cast<double2*>(out[k] + j), make_double2(o0[k], o1[k]));
        } else {
          __stcs(out[k] + j, o0[k]);
        }
      }
    }
    __syncthreads();  // this slot is free for the chunk after next
  }
  Dd tot[K];
  if (dd_grid_reduce<K>(acc, part, &sc->counter[SW == 0 ? T_SWEEPA : T_SWEEPC], tot) &&
      threadIdx.x == 0) {
    if (SW == 0) publish<F_SWEEPA>(sc, h, tot);
    else publish<F_SWEEPC>(sc, h, tot);
  }
}

// eq:rr: r := b - A x; k := M^-1 r; s := A g; l := M^-1 s
template <bool NRM, int PK>
__global__ void __launch_bounds__(256) c_rr1(CsrOp A, Vecs V, Scal* __restrict__ sc,
                                             Dd* __restrict__ part, Hist h) {
  constexpr bool BJ = PK == PK_BJ;
  if (sc->done || !sc->rr_fire) return;
  Dd acc[4] = {dd_zero(), dd_zero(), dd_zero(), dd_zero()};
  WROW_LOOP
    const double rj = in ? V.b[j] - ell_row<false>(A, V.x, j) : 0.0;
    const double sj = in ? ell_row<false>(A, V.g, j) : 0.0;
    // k := M^-1 r, l := M^-1 s (ILU(0): k_ilu_* after this kernel)
    const double kj = PK == PK_ILU ? 0.0 : prec_row<BJ>(A, j, in, rj, dj);
    const double lj = PK == PK_ILU ? 0.0 : prec_row<BJ>(A, j, in, sj, dj);
    if (in) {
      V.r[j] = rj;
      V.s[j] = sj;
      if (PK != PK_ILU) {
        V.k[j] = kj;
        V.l[j] = lj;
      }
      if (NRM) {  // replaced x_{i+1}, k_{i+1}, s_i, l_i
        c_nrm(acc[0], V.x[j]); c_nrm(acc[1], kj); c_nrm(acc[2], sj); c_nrm(acc[3], lj);
      }
    }
  WROW_END
  if (NRM) {
    Dd tot[4];
    if (dd_grid_reduce<4>(acc, part, &sc->counter[T_RR1], tot) && threadIdx.x == 0)
      publish<F_RR1>(sc, h, tot);
  }
}

// w := A k; z := A l (into zrr); line-21 dots on the replaced vectors
template <bool NRM, int PK>
__global__ void __launch_bounds__(256) c_rr2(CsrOp A, Vecs V, Scal* __restrict__ sc,
                                             Dd* __restrict__ part, Hist h) {
  constexpr bool BJ = PK == PK_BJ;
  constexpr int K = NRM ? 6 : 5;
  if (sc->done || !sc->rr_fire) return;
  Dd acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = dd_zero();
  WROW_LOOP
    const double wn = in ? ell_row<false>(A, V.k, j) : 0.0;  // w := A k = A M^-1 r
    const double zr = in ? ell_row<false>(A, V.l, j) : 0.0;  // z := A l = A M^-1 s
    // m_{i+1} follows the replaced w (A27; ILU(0): k_ilu_* after this kernel)
    const double mn = PK == PK_ILU ? 0.0 : prec_row<BJ>(A, j, in, wn, dj);
    if (in) {
      V.w0[j] = wn;
      if (PK != PK_ILU) V.mv[j] = mn;
      V.zrr[j] = zr;
      const double rhj = V.rh[j], rc = V.r[j];
      dd_fma(acc[0], rhj, rc);
      dd_fma(acc[1 % K], rhj, wn);
      dd_fma(acc[2 % K], rhj, V.s[j]);
      dd_fma(acc[3 % K], rhj, zr);
      dd_fma(acc[4 % K], rc, rc);
      if (NRM) c_nrm(acc[5 % K], zr);  // replaced z_i
    }
  WROW_END
  Dd tot[K];
  if (dd_grid_reduce<K>(acc, part, &sc->counter[T_RR2], tot) && threadIdx.x == 0)
    publish<F_RR2>(sc, h, tot);
}

// line 23: t_{i+1} = A m_{i+1} (also t_0 at init); gather version
__global__ void __launch_bounds__(256) c_spmvD(CsrOp A, Vecs V, Scal* __restrict__ sc) {
  if (sc->done) return;
  ROW_LOOP { V.w1[j] = ell_row<false>(A, V.mv, j); }
}

// ---------------------------------------------------------------------------
// Window SpMV y = A u for banded matrices (|col - row| <= bw): a CTA walks a
// contiguous row range in steps of WTB rows; the operand window
// [j0 - bw, j0 + WTB + bw) lives in a 2^k shared-memory ring filled by TMA
// bulk copies two steps ahead, so the 27 gathers per row are shared-memory
// loads (position = (e + off) & (WRS - 1)) and each operand element comes from
// HBM/L2 once per CTA.  Each row is summed in stored order from +0.0 (A5).
#define WTB 2048
#define WRS 16384
#define WNT 512

struct WinGeo {
  int64_t lo, hi;     // valid operand range [lo, hi) (ghosts included)
  int64_t off;        // element offset making (e + off) >= 0 and chunk-aligned
  int32_t bw;         // half bandwidth
  int32_t rows_cta;   // rows per CTA (multiple of WTB)
};

__device__ __forceinline__ void win_issue(double* ring, const double* __restrict__ u, int64_t x0,
                                          int64_t x1, const WinGeo& w, uint64_t* bar) {
  // load elements [x0, x1) clamped to the valid range, chunk by chunk (no wrap)
  int64_t a = x0 > w.lo ? x0 : w.lo;
  const int64_t b = x1 < w.hi ? x1 : w.hi;
  uint32_t total = 0;
  for (int64_t c = a; c < b;) {
    const int64_t cend = ((c + w.off) / WTB + 1) * WTB - w.off;
    const int64_t e = cend < b ? cend : b;
    total += (uint32_t)(((e - c) * 8 + 15) & ~15);
    c = e;
  }
  mbar_arrive_expect_tx(bar, total);
  for (int64_t c = a; c < b;) {
    const int64_t cend = ((c + w.off) / WTB + 1) * WTB - w.off;
    const int64_t e = cend < b ? cend : b;
    const uint32_t bytes = (uint32_t)(((e - c) * 8 + 15) & ~15);
    bulk_g2s(ring + ((c + w.off) & (WRS - 1)), u + c, bytes, bar);
    c = e;
  }
}

template <int WHICH>  // SpmvMode: input, output and epilogue of the step
__global__ void __launch_bounds__(WNT, 1) c_spmv_win(CsrOp A, Vecs V, Scal* __restrict__ sc,
                                                     WinGeo w, Dd* __restrict__ part, Hist h) {
  constexpr int K = SpmvK<WHICH>::K > 0 ? SpmvK<WHICH>::K : 1;
  constexpr bool INIT = WHICH == SP_PCW0 || WHICH == SP_I1 || WHICH == SP_I2;
  if (WHICH == SP_GAP ? sc->gap_iter >= sc->iter : (!INIT && sc->done)) return;
  const double al = sc->alpha;
  const double* __restrict__ u = spmv_in<WHICH>(V);
  Dd dacc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) dacc[k] = dd_zero();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  double* ring = reinterpret_cast<double*>(smem_raw + 64);
  const int64_t R0 = (int64_t)blockIdx.x * w.rows_cta;  // < A.n: grid = ceil(n / rows_cta)
  const int64_t R1 = (R0 + w.rows_cta) < A.n ? (R0 + w.rows_cta) : A.n;
  const int nsteps = (int)((R1 - R0 + WTB - 1) / WTB);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    win_issue(ring, u, R0 - w.bw, R0 + WTB + w.bw, w, &bar[0]);
    if (nsteps > 1) win_issue(ring, u, R0 + WTB + w.bw, R0 + 2 * WTB + w.bw, w, &bar[1]);
  }
  uint32_t ph = 0;
  for (int s = 0; s < nsteps; ++s) {
    const int b = s & 1;
    mbar_wait(&bar[b], (ph >> b) & 1u);
    ph ^= 1u << b;
    const int64_t j0 = R0 + (int64_t)s * WTB;
#pragma unroll
    for (int q = 0; q < WTB / WNT; ++q) {
      const int64_t j = j0 + threadIdx.x + q * WNT;
      if (j >= R1) break;
      const int len = A.len ? A.len[j] : A.width;
      const int rb = (int)((j + w.off) & (WRS - 1));  // ring position of row j's own column
      const size_t sb = ((size_t)(j >> 5) * A.width) * 32 + (j & 31);  // slot 0 (SELL-32)
      const double* __restrict__ av = A.sval + sb;    // advanced by whole groups, so
      const int16_t* __restrict__ ac = A.sdcol + sb;  // every load is base + immediate
      double acc = 0.0;
      int p = 0;
      // groups of WIN_U slots: all of a group's matrix loads in flight before its adds
      // (27 = the cfg5 row length: one group, +4.5% over groups of 9 -- measured).
      // Column = j + delta (int16), ring position (rb + delta) mod WRS.
      for (; p + WIN_U <= len; p += WIN_U, av += WIN_U * 32, ac += WIN_U * 32) {
        int c[WIN_U];
        double a[WIN_U];
#pragma unroll
        for (int k = 0; k < WIN_U; ++k) {
          c[k] = __ldcs(ac + k * 32);
          a[k] = __ldcs(av + k * 32);
        }
#pragma unroll
        for (int k = 0; k < WIN_U; ++k) acc = acc + a[k] * ring[(rb + c[k]) & (WRS - 1)];
      }
      for (; p + ELL_U <= len; p += ELL_U, av += ELL_U * 32, ac += ELL_U * 32) {
        int c[ELL_U];
        double a[ELL_U];
#pragma unroll
        for (int k = 0; k < ELL_U; ++k) {
          c[k] = __ldcs(ac + k * 32);
          a[k] = __ldcs(av + k * 32);
        }
#pragma unroll
        for (int k = 0; k < ELL_U; ++k) acc = acc + a[k] * ring[(rb + c[k]) & (WRS - 1)];
      }
      for (; p < len; ++p, av += 32, ac += 32) {
        const int c = __ldcs(ac);
        acc = acc + __ldcs(av) * ring[(rb + c) & (WRS - 1)];
      }
      spmv_epi<WHICH, K>(A, V, j, acc, al, dacc);
    }
    __syncthreads();  // step s done: its oldest chunk may be overwritten
    if (threadIdx.x == 0 && s + 2 < nsteps)
      win_issue(ring, u, j0 + 2 * WTB + w.bw, j0 + 3 * WTB + w.bw, w, &bar[b]);
  }
  spmv_fin<WHICH>(sc, h, part, dacc);
}

// mv := M^-1 w0 (p-CG init, after SP_PCW0)
template <int PK>
__global__ void __launch_bounds__(256) c_prec_mv(CsrOp A, Vecs V) {
  constexpr bool BJ = PK == PK_BJ;
  WROW_LOOP
    const double m = prec_row<BJ>(A, j, in, in ? V.w0[j] : 0.0, dj);
    if (in) V.mv[j] = m;
  WROW_END
}

// ---------------------------------------------------------------------------
// Classic BiCGStab (Alg. 1) on CSR: the element-wise steps around the
// SpMVs SP_CLS / SP_CLY.  Buffers: p -> g, M^-1 p -> mv, M^-1 q -> nv, y -> z1.
// l.17 of the previous iteration (i = 0: beta = omega = 0 and p = s = 0, so
// p_0 = r_0): p := r + beta (p - omega s); the SpMV operand mv := M^-1 p (l.4)
template <int PK>
__global__ void __launch_bounds__(256) c_cl_p(CsrOp A, Vecs V, Scal* __restrict__ sc) {
  constexpr bool BJ = PK == PK_BJ;
  if (sc->done) return;
  const double be = sc->beta, om = sc->omega;
  WROW_LOOP
    const double p = in ? V.r[j] + be * (V.g[j] - om * V.s[j]) : 0.0;
    const double g = PK == PK_ILU ? 0.0 : prec_row<BJ>(A, j, in, p, dj);
    if (in) {
      V.g[j] = p;
      if (PK != PK_ILU) V.mv[j] = g;  // ILU(0): mv := M^-1 p by k_ilu_* (from g)
    }
  WROW_END
}

// l.8-9: q := r - alpha s; the SpMV operand nv := u = M^-1 q
template <int PK>
__global__ void __launch_bounds__(256) c_cl_u(CsrOp A, Vecs V, Scal* __restrict__ sc) {
  constexpr bool BJ = PK == PK_BJ;
  if (sc->done) return;
  const double al = sc->alpha;
  WROW_LOOP
    const double q = in ? V.r[j] - al * V.s[j] : 0.0;
    if (PK == PK_ILU) {  // q stored in z0; nv := M^-1 q by k_ilu_*
      if (in) V.z0[j] = q;
    } else {
      const double u = prec_row<BJ>(A, j, in, q, dj);
      if (in) V.nv[j] = u;
    }
  WROW_END
}

// l.13-15: x := (x + alpha g) + omega u; r := q - omega y; (r^0, r), ||r||^2
__global__ void __launch_bounds__(256) c_cl_x(CsrOp A, Vecs V, Scal* __restrict__ sc,
                                              Dd* __restrict__ part, Hist h) {
  if (sc->done) return;
  const double al = sc->alpha, om = sc->omega;
  Dd acc[2] = {dd_zero(), dd_zero()};
  ROW_LOOP {
    const double q = V.r[j] - al * V.s[j];
    const double xn = (V.x[j] + al * V.mv[j]) + om * V.nv[j];
    const double rn = q - om * V.z1[j];
    V.x[j] = xn;
    V.r[j] = rn;
    dd_fma(acc[0], V.rh[j], rn);
    dd_fma(acc[1], rn, rn);
  }
  Dd tot[2];
  if (dd_grid_reduce<2>(acc, part, &sc->counter[T_CL3], tot) && threadIdx.x == 0)
    publish<F_CL3>(sc, h, tot);
}

// Classic BiCGStab's point-wise steps (Jacobi) on the same TMA chunk ring as the
// p-BiCGStab sweeps: the expressions of c_cl_p / c_cl_u / c_cl_x, a row pair per thread.
//   ST 0 (l.17): p := r + beta (p - omega s), mv := M^-1 p      in: r, p(g), s, dinv
//   ST 1 (l.8-9): nv := M^-1 (r - alpha s)                       in: r, s, dinv
//   ST 2 (l.13-15): x, r; (r^0, r), ||r||^2                       in: r, s, x, mv, nv, y(z1), r^0
template <int ST>
__global__ void __launch_bounds__(CST_T, 1) c_cl_tma(CsrOp A, Vecs V, Scal* __restrict__ sc,
                                                     Dd* __restrict__ part, Hist h) {
  constexpr int NIN = ST == 0 ? 4 : ST == 1 ? 3 : 7;
  if (sc->done) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  double* buf = reinterpret_cast<double*>(smem_raw + 64);
  const int tid = threadIdx.x;
  const double al = sc->alpha, be = sc->beta, om = sc->omega;
  const double* in[7];
  if (ST == 0) {
    in[0] = V.r; in[1] = V.g; in[2] = V.s; in[3] = A.dinv;
  } else if (ST == 1) {
    in[0] = V.r; in[1] = V.s; in[2] = A.dinv;
  } else {
    in[0] = V.r; in[1] = V.s; in[2] = V.x; in[3] = V.mv; in[4] = V.nv; in[5] = V.z1;
    in[6] = V.rh;
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t nch = (A.n + CST_R - 1) / CST_R;
  auto stage = [&](int slot, int64_t c) {
    const int64_t j0 = c * CST_R;
    const int64_t rows = (A.n - j0) < CST_R ? (A.n - j0) : CST_R;
    const uint32_t bytes = (uint32_t)((rows * 8 + 15) & ~15LL);  // vectors carry 2 slack rows
    mbar_arrive_expect_tx(&bar[slot], bytes * (uint32_t)NIN);
#pragma unroll
    for (int v = 0; v < NIN; ++v)
      bulk_g2s(buf + ((size_t)slot * CST_NIN + v) * CST_R, in[v] + j0, bytes, &bar[slot]);
  };
  Dd acc[2] = {dd_zero(), dd_zero()};
  if (tid == 0 && (int64_t)blockIdx.x < nch) stage(0, blockIdx.x);
  uint32_t ph = 0;
  int slot = 0;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, slot ^= 1) {
    if (tid == 0 && c + gridDim.x < nch) stage(slot ^ 1, c + gridDim.x);
    mbar_wait(&bar[slot], (ph >> slot) & 1u);
    ph ^= 1u << slot;
    const int64_t j = c * CST_R + 2 * tid;
    if (j < A.n) {
      const bool valid1 = j + 1 < A.n;
      const double* B = buf + (size_t)slot * CST_NIN * CST_R + 2 * tid;
      double x0[NIN], x1[NIN];
#pragma unroll
      for (int v = 0; v < NIN; ++v) {
        const double2 q = *reinterpret_cast<const double2*>(B + (size_t)v * CST_R);
        x0[v] = q.x;
        x1[v] = q.y;
      }
      double o0[2] = {0.0, 0.0}, o1[2] = {0.0, 0.0};
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double* xv = e == 0 ? x0 : x1;
        double* o = e == 0 ? o0 : o1;
        if (e == 1 && !valid1) break;
        if (ST == 0) {  // c_cl_p
          const double pn = xv[0] + be * (xv[1] - om * xv[2]);
          o[0] = pn;
          o[1] = xv[3] * pn;
        } else if (ST == 1) {  // c_cl_u
          o[0] = xv[2] * (xv[0] - al * xv[1]);
        } else {  // c_cl_x
          const double q = xv[0] - al * xv[1];
          const double xn = (xv[2] + al * xv[3]) + om * xv[4];
          const double rn = q - om * xv[5];
          o[0] = xn;
          o[1] = rn;
          dd_fma(acc[0], xv[6], rn);
          dd_fma(acc[1], rn, rn);
        }
      }
      double* out[2];
      if (ST == 0) { out[0] = V.g; out[1] = V.mv; }
      else if (ST == 1) { out[0] = V.nv; out[1] = V.nv; }
      else { out[0] = V.x; out[1] = V.r; }
      constexpr int NOUT = ST == 1 ? 1 : 2;
#pragma unroll
      for (int k = 0; k < NOUT; ++k) {
        if (valid1) __stcs(reinterpret_cast<double2*>(out[k] + j), make_double2(o0[k], o1[k]));
        else __stcs(out[k] + j, o0[k]);
      }
    }
    __syncthreads();  // this slot is free for the chunk after next
  }
  if (ST == 2) {
    Dd tot[2];
    if (dd_grid_reduce<2>(acc, part, &sc->counter[T_CL3], tot) && threadIdx.x == 0)
      publish<F_CL3>(sc, h, tot);
  }
}

// p-CG iteration (reading A19) after n_i = A m_i (SP_PCN): buffers z -> z0,
// q -> l, s, p -> g, x, r, u -> k, w -> w0, n -> z1, m -> mv (written for the
// next SpMV); the next iteration's (r,u), (w,u), ||r||^2
template <int PK>
__global__ void __launch_bounds__(256) c_pc(CsrOp A, Vecs V, Scal* __restrict__ sc,
                                            Dd* __restrict__ part, Hist h) {
  constexpr bool BJ = PK == PK_BJ;
  if (sc->done) return;
  const double al = sc->alpha, be = sc->beta;
  Dd acc[3] = {dd_zero(), dd_zero(), dd_zero()};
  WROW_LOOP
    const double wj = in ? V.w0[j] : 0.0;
    // m_i = M^-1 w_i (ILU(0): as stored by k_ilu_*)
    const double mj = PK == PK_ILU ? (in ? V.mv[j] : 0.0) : prec_row<BJ>(A, j, in, wj, dj);
    double wn = 0.0;
    if (in) {
    const double uj = V.k[j];
    const double zn = V.z1[j] + be * V.z0[j];
    const double qn = mj + be * V.l[j];
    const double sn = wj + be * V.s[j];
    const double pn = uj + be * V.g[j];
    const double xn = V.x[j] + al * pn;
    const double rn = V.r[j] - al * sn;
    const double un = uj - al * qn;
    wn = wj - al * zn;
    V.z0[j] = zn; V.l[j] = qn; V.s[j] = sn; V.g[j] = pn;
    V.x[j] = xn; V.r[j] = rn; V.k[j] = un; V.w0[j] = wn;
    dd_fma(acc[0], rn, un);
    dd_fma(acc[1], wn, un);
    dd_fma(acc[2], rn, rn);
    }
    if (PK != PK_ILU) {
      const double mn = prec_row<BJ>(A, j, in, wn, dj);
      if (in) V.mv[j] = mn;
    }
  WROW_END
  Dd tot[3];
  if (dd_grid_reduce<3>(acc, part, &sc->counter[T_PC], tot) && threadIdx.x == 0)
    publish<F_PC>(sc, h, tot);
}

__global__ void __launch_bounds__(256) c_gap(CsrOp A, Vecs V, Scal* __restrict__ sc,
                                             Dd* __restrict__ part, Hist h) {
  if (sc->gap_iter >= sc->iter) return;
  Dd acc[1] = {dd_zero()};
  ROW_LOOP {
    const double d = (V.b[j] - ell_row<false>(A, V.x, j)) - V.r[j];
    dd_fma(acc[0], d, d);
  }
  Dd tot[1];
  if (dd_grid_reduce<1>(acc, part, &sc->counter[T_GAP], tot) && threadIdx.x == 0)
    publish<F_GAP>(sc, h, tot);
}

__global__ void __launch_bounds__(256) c_apply(CsrOp A, const double* __restrict__ xin,
                                               double* __restrict__ yout) {
  ROW_LOOP { yout[j] = ell_row<false>(A, xin, j); }
}
