// tile_jac.cu -- the Jacobi instances of the stencil tile kernels (full-line tiles),
// compiled twice (-DPBICG_VEC=1: 16-byte paired path for even nx; 0: odd nx) in
// parallel with the host driver; pbicgstab.cu reaches them through tile_jac.h.
#include <cuda_runtime.h>

#include "tile_jac.h"
#include "tile_sweeps.cuh"

#ifndef PBICG_VEC
#error "compile with -DPBICG_VEC=0|1"
#endif

namespace {

constexpr bool kVec = PBICG_VEC != 0;

template <int DIM, int MODE>
void launch_one(int grid, size_t smem, cudaStream_t s, const TileGeo& g, const Vecs& V, Scal* sc,
                Dd* part, Hist h) {
  if constexpr (HasPeer<MODE>::v) {
    if (g.peer) {  // peer-memory transport: the instance that stores the boundary planes
      tile_launch(t_tile<DIM, MODE, kVec, 0, false, true>, grid, smem, s, g, V, sc, part, h);
      return;
    }
  }
  tile_launch(t_tile<DIM, MODE, kVec>, grid, smem, s, g, V, sc, part, h);
}

template <int DIM, int MODE>
cudaError_t attr_one(int smem, int* occ) {
  cudaError_t e = cudaFuncSetAttribute(t_tile<DIM, MODE, kVec>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if constexpr (HasPeer<MODE>::v) {
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(t_tile<DIM, MODE, kVec, 0, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  }
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, t_tile<DIM, MODE, kVec>, TNT, smem);
  return e;
}

#define JAC_MODES(X)                                                                         \
  X(TM_A) X(TM_C) X(TM_RR1) X(TM_RR2) X(TM_GAP) X(TM_INIT1) X(TM_INIT2) X(TM_CL1) X(TM_CL2) \
  X(TM_CL3) X(TM_PC) X(TM_PCI1) X(TM_PCI2) X(TM_AN) X(TM_CN) X(TM_RR1N) X(TM_RR2N)         \
  X(TM_INIT1N) X(TM_SPB) X(TM_SPD)

template <int DIM>
bool dispatch(int mode, int grid, size_t smem, cudaStream_t s, const TileGeo& g, const Vecs& V,
              Scal* sc, Dd* part, Hist h) {
  switch (mode) {
#define JAC_CASE(M) \
  case M: launch_one<DIM, M>(grid, smem, s, g, V, sc, part, h); return true;
    JAC_MODES(JAC_CASE)
#undef JAC_CASE
    default: return false;
  }
}

template <int DIM>
cudaError_t dispatch_attr(int mode, int smem, int* occ) {
  switch (mode) {
#define JAC_CASE(M) \
  case M: return attr_one<DIM, M>(smem, occ);
    JAC_MODES(JAC_CASE)
#undef JAC_CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

#define JAC_CAT2(a, b) a##b
#define JAC_CAT(a, b) JAC_CAT2(a, b)

bool JAC_CAT(tile_jac_launch_, PBICG_VEC)(int dim, int mode, int grid, size_t smem,
                                           cudaStream_t s, const TileGeo& g, const Vecs& V,
                                           Scal* sc, Dd* part, Hist h) {
  return dim == 3 ? dispatch<3>(mode, grid, smem, s, g, V, sc, part, h)
                  : dispatch<2>(mode, grid, smem, s, g, V, sc, part, h);
}

cudaError_t JAC_CAT(tile_jac_attr_, PBICG_VEC)(int dim, int mode, int smem, int* occ) {
  return dim == 3 ? dispatch_attr<3>(mode, smem, occ) : dispatch_attr<2>(mode, smem, occ);
}

#if defined(PBICG_TIMELINE) && PBICG_VEC
// timeline variant only: point the instrumentation at a device buffer (records, count)
extern "C" int pbicg_timeline_set(void* buf, void* cnt, unsigned cap) {
  TlRec* b = (TlRec*)buf;
  unsigned* c = (unsigned*)cnt;
  cudaError_t e = cudaMemcpyToSymbol(g_tl_buf, &b, sizeof(b));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_tl_cnt, &c, sizeof(c));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_tl_cap, &cap, sizeof(cap));
  return (int)e;
}
#endif
