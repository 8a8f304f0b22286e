// dd.cuh -- compensated (Dot2) dot-product accumulation and the deterministic
// two-stage block / grid reduction used by every fused sweep.
//
// Reading A6: the paper only bounds the dot-product rounding error
// (P:49); all dots are Dot2 (Ogita-Rump-Oishi): TwoProd via fma, TwoSum, a
// double-double running pair (P, S), one final rounding fl(P + S).  The
// combine operator (+) of two partials is commutative bitwise and the tree
// shapes below are fixed, so results are run-to-run deterministic.
//
// This translation unit is compiled with -fmad=false: no mul+add is ever
// contracted; the only fma is the explicit one inside TwoProd.
#pragma once
#include <cstdint>

struct Dd {
  double hi, lo;
};

__device__ __forceinline__ Dd dd_zero() { return Dd{0.0, 0.0}; }

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  double z = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, z)), __dsub_rn(b, z));
}

// (P, S) += x * y   (TwoProd + TwoSum, then S = fl(S + fl(q + r)))
__device__ __forceinline__ void dd_fma(Dd& d, double x, double y) {
  double h = __dmul_rn(x, y);
  double r = __fma_rn(x, y, -h);
  double q;
  two_sum(d.hi, h, d.hi, q);
  d.lo = __dadd_rn(d.lo, __dadd_rn(q, r));
}

// (P1,S1) (+) (P2,S2): (P,q) = TwoSum(P1,P2), S = fl(fl(S1+S2) + q)
__device__ __forceinline__ Dd dd_add(Dd a, Dd b) {
  Dd c;
  double q;
  two_sum(a.hi, b.hi, c.hi, q);
  c.lo = __dadd_rn(__dadd_rn(a.lo, b.lo), q);
  return c;
}

__device__ __forceinline__ double dd_round(Dd a) { return __dadd_rn(a.hi, a.lo); }

__device__ __forceinline__ Dd dd_shfl_down(Dd a, int off) {
  Dd b;
  b.hi = __shfl_down_sync(0xffffffffu, a.hi, off);
  b.lo = __shfl_down_sync(0xffffffffu, a.lo, off);
  return b;
}

// Fixed-shape warp tree; lane 0 holds the result.
__device__ __forceinline__ Dd dd_warp_reduce(Dd a) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) a = dd_add(a, dd_shfl_down(a, off));
  return a;
}

// Block reduction of K partials; thread 0 returns the totals.  blockDim.x must
// be a multiple of 32 and <= 1024.  Ends with a __syncthreads().
template <int K>
__device__ __forceinline__ void dd_block_reduce(Dd (&acc)[K]) {
  __shared__ Dd sh[K][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    Dd v = dd_warp_reduce(acc[k]);
    if (lane == 0) sh[k][warp] = v;
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      Dd v = lane < nwarps ? sh[k][lane] : dd_zero();
      acc[k] = dd_warp_reduce(v);
    }
  }
  __syncthreads();
}

// Stage 2: every CTA publishes its K partials to part[blockIdx.x*K + k]; the
// last CTA to arrive (ticket) reduces all gridDim.x partials with a fixed
// strided + tree order and returns true with the totals in tot[] on thread 0.
// The ticket counter is reset by the last CTA so the kernel can be relaunched.
template <int K>
__device__ __forceinline__ bool dd_grid_reduce(Dd (&acc)[K], Dd* __restrict__ part,
                                               unsigned int* counter, Dd (&tot)[K]) {
  __shared__ bool s_last;
  dd_block_reduce<K>(acc);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) part[(size_t)blockIdx.x * K + k] = acc[k];
    __threadfence();
    unsigned int t = atomicAdd(counter, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  Dd v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = dd_zero();
  for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const Dd* p = part + (size_t)b * K + k;
      Dd pv;
      pv.hi = __ldcg(&p->hi);
      pv.lo = __ldcg(&p->lo);
      v[k] = dd_add(v[k], pv);
    }
  }
  dd_block_reduce<K>(v);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) tot[k] = v[k];
    *counter = 0u;
  }
  return true;
}
