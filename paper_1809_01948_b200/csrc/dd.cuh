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

template <int K> struct Pow2 { enum { v = K <= 1 ? 1 : K <= 2 ? 2 : K <= 4 ? 4 : K <= 8 ? 8 : 16 }; };
template <int P> struct Log2 { enum { v = P <= 1 ? 0 : P == 2 ? 1 : P == 4 ? 2 : P == 8 ? 3 : 4 }; };

__device__ __forceinline__ Dd dd_shfl_xor(Dd a, int m) {
  Dd b;
  b.hi = __shfl_xor_sync(0xffffffffu, a.hi, m);
  b.lo = __shfl_xor_sync(0xffffffffu, a.lo, m);
  return b;
}

// K values per lane reduced over the warp by transposition: at the first log2(P)
// levels (P = K rounded up to a power of two) each lane keeps half of its values and
// trades the other half with its partner, so one shuffle-and-add serves two values
// (9 combines per lane for K = 5 instead of 25); the remaining levels are a
// butterfly.  Lane l ends with the total of value l >> (5 - log2 P).  Every value is
// combined over exactly the pairs (i, i + off), off = 16, 8, ..., 1, of
// dd_warp_reduce's tree, and (+) is commutative bitwise, so the totals are that
// tree's bits.
template <int K>
__device__ __forceinline__ Dd dd_warp_reduce_multi(const Dd (&a)[K]) {
  constexpr int P = Pow2<K>::v, LP = Log2<P>::v;
  static_assert(K <= 16, "at most 16 values");
  Dd v[P];
#pragma unroll
  for (int j = 0; j < P; ++j) v[j] = j < K ? a[j] : dd_zero();
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int o = 16 >> t;
    if (t < LP) {
      const int half = P >> (t + 1);
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int j = 0; j < half; ++j) {
        const Dd send = up ? v[j] : v[j + half];
        const Dd keep = up ? v[j + half] : v[j];
        v[j] = dd_add(keep, dd_shfl_xor(send, o));
      }
    } else {
      v[0] = dd_add(v[0], dd_shfl_xor(v[0], o));
    }
  }
  return v[0];
}

// Block reduction of K partials; thread 0 returns the totals.  blockDim.x must
// be a multiple of 32 and <= 1024.  Ends with a __syncthreads().  Per value the
// tree is a warp tree (dd_warp_reduce's pairs) over the lanes, then one over the
// warps' totals (zeros past the last warp).
template <int K>
__device__ __forceinline__ void dd_block_reduce(Dd (&acc)[K]) {
  constexpr int S = 5 - Log2<Pow2<K>::v>::v;  // lane l holds value l >> S
  __shared__ Dd sh[K][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  {
    const Dd t = dd_warp_reduce_multi<K>(acc);
    const int k = lane >> S;
    if ((lane & ((1 << S) - 1)) == 0 && k < K) sh[k][warp] = t;
  }
  __syncthreads();
  if (warp == 0) {
    Dd v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = lane < nwarps ? sh[k][lane] : dd_zero();
    const Dd t = dd_warp_reduce_multi<K>(v);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      acc[k].hi = __shfl_sync(0xffffffffu, t.hi, k << S);
      acc[k].lo = __shfl_sync(0xffffffffu, t.lo, k << S);
    }
  }
  __syncthreads();
}

// Stage 2: every CTA publishes its K partials to part[blockIdx.x*K + k]; the
// last CTA to arrive (ticket) reduces all gridDim.x partials with a fixed
// strided + tree order and returns true with the totals in tot[] on thread 0.
// The ticket counter is reset by the last CTA so the kernel can be relaunched.
// OVR: a mask of value slots whose block totals are not this kernel's but come from
// ovr[blockIdx.x * popc(OVR) + j] (j-th set bit; the tile replacement step's stash).
template <int K, unsigned OVR = 0u>  // OVR: slots 0..7 only
__device__ __forceinline__ bool dd_grid_reduce(Dd (&acc)[K], Dd* __restrict__ part,
                                               unsigned int* counter, Dd (&tot)[K],
                                               const Dd* __restrict__ ovr = nullptr) {
  __shared__ bool s_last;
  dd_block_reduce<K>(acc);
  if (OVR != 0u && threadIdx.x == 0) {
    constexpr int NO = ((OVR >> 0) & 1) + ((OVR >> 1) & 1) + ((OVR >> 2) & 1) + ((OVR >> 3) & 1) +
                       ((OVR >> 4) & 1) + ((OVR >> 5) & 1) + ((OVR >> 6) & 1) + ((OVR >> 7) & 1);
    int j = 0;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if ((OVR >> k) & 1u) acc[k] = ovr[(size_t)blockIdx.x * NO + j++];
  }
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) part[(size_t)blockIdx.x * K + k] = acc[k];
    // one acq_rel ticket instead of fence + atomic + fence: release orders this CTA's
    // partials before its ticket; the last CTA's acquire orders every CTA's partials
    // before its reads (the other threads read after the barrier below, through L2)
    unsigned int t;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(t) : "l"(counter)
                 : "memory");
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  Dd v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = dd_zero();
  for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double2 pv = __ldcg(reinterpret_cast<const double2*>(part + (size_t)b * K + k));
      v[k] = dd_add(v[k], Dd{pv.x, pv.y});
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
