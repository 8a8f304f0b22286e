// tile_bj.cu -- the block-Jacobi instances of the stencil tile kernels (reading
// A33), one translation unit per block size (compiled three times with
// -DPBICG_BJ_B=2|4|8, in parallel with pbicgstab.cu) so the build stays short.
// pbicgstab.cu reaches them only through the two functions below.
#include <cuda_runtime.h>

#include "tile_bj.h"
#include "tile_sweeps.cuh"

#ifndef PBICG_BJ_B
#error "compile with -DPBICG_BJ_B=2|4|8"
#endif

namespace {

template <int DIM, int MODE>
void launch_one(int grid, size_t smem, cudaStream_t s, const TileGeo& g, const Vecs& V, Scal* sc,
                Dd* part, Hist h) {
  if constexpr (HasPeer<MODE>::v) {
    if (g.peer) {  // peer-memory transport: the instance that stores the boundary planes
      tile_launch(t_tile<DIM, MODE, true, PBICG_BJ_B, false, true>, grid, smem, s, g, V, sc, part, h);
      return;
    }
  }
  tile_launch(t_tile<DIM, MODE, true, PBICG_BJ_B>, grid, smem, s, g, V, sc, part, h);
}

template <int DIM, int MODE>
cudaError_t attr_one(int smem, int* occ) {
  cudaError_t e = cudaFuncSetAttribute(t_tile<DIM, MODE, true, PBICG_BJ_B>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if constexpr (HasPeer<MODE>::v) {
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(t_tile<DIM, MODE, true, PBICG_BJ_B, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  }
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, t_tile<DIM, MODE, true, PBICG_BJ_B>,
                                                      TNT, smem);
  return e;
}

template <int DIM>
bool dispatch(int mode, int grid, size_t smem, cudaStream_t s, const TileGeo& g, const Vecs& V,
              Scal* sc, Dd* part, Hist h) {
  switch (mode) {
#define BJ_CASE(M) \
  case M: launch_one<DIM, M>(grid, smem, s, g, V, sc, part, h); return true;
    BJ_CASE(TM_A) BJ_CASE(TM_C) BJ_CASE(TM_RR1) BJ_CASE(TM_RR2) BJ_CASE(TM_INIT1)
    BJ_CASE(TM_INIT2) BJ_CASE(TM_AN) BJ_CASE(TM_CN) BJ_CASE(TM_RR1N) BJ_CASE(TM_RR2N)
    BJ_CASE(TM_INIT1N) BJ_CASE(TM_CL1) BJ_CASE(TM_CL2) BJ_CASE(TM_CL3) BJ_CASE(TM_PC)
    BJ_CASE(TM_PCI1) BJ_CASE(TM_PCI2)
#undef BJ_CASE
    default: return false;
  }
}

template <int DIM>
cudaError_t dispatch_attr(int mode, int smem, int* occ) {
  switch (mode) {
#define BJ_CASE(M) \
  case M: return attr_one<DIM, M>(smem, occ);
    BJ_CASE(TM_A) BJ_CASE(TM_C) BJ_CASE(TM_RR1) BJ_CASE(TM_RR2) BJ_CASE(TM_INIT1)
    BJ_CASE(TM_INIT2) BJ_CASE(TM_AN) BJ_CASE(TM_CN) BJ_CASE(TM_RR1N) BJ_CASE(TM_RR2N)
    BJ_CASE(TM_INIT1N) BJ_CASE(TM_CL1) BJ_CASE(TM_CL2) BJ_CASE(TM_CL3) BJ_CASE(TM_PC)
    BJ_CASE(TM_PCI1) BJ_CASE(TM_PCI2)
#undef BJ_CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

#define BJ_CAT2(a, b) a##b
#define BJ_CAT(a, b) BJ_CAT2(a, b)

bool BJ_CAT(tile_bj_launch_, PBICG_BJ_B)(int dim, int mode, int grid, size_t smem, cudaStream_t s,
                                          const TileGeo& g, const Vecs& V, Scal* sc, Dd* part,
                                          Hist h) {
  return dim == 3 ? dispatch<3>(mode, grid, smem, s, g, V, sc, part, h)
                  : dispatch<2>(mode, grid, smem, s, g, V, sc, part, h);
}

cudaError_t BJ_CAT(tile_bj_attr_, PBICG_BJ_B)(int dim, int mode, int smem, int* occ) {
  return dim == 3 ? dispatch_attr<3>(mode, smem, occ) : dispatch_attr<2>(mode, smem, occ);
}
