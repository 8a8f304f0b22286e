// tile_seg.cu -- the x-segmented instances of the stencil tile kernels (grids with
// nx > 1024, nx even: a tile is TY lines x sx columns, staged line segment by line
// segment with SEG_HX halo columns), compiled in parallel with pbicgstab.cu.
// pbicgstab.cu reaches them only through the two functions of tile_seg.h.
#include <cuda_runtime.h>

#include "tile_seg.h"
#include "tile_sweeps.cuh"

namespace {

template <int DIM, int MODE>
void launch_one(int grid, size_t smem, cudaStream_t s, const TileGeo& g, const Vecs& V, Scal* sc,
                Dd* part, Hist h) {
  if constexpr (HasPeer<MODE>::v) {
    if (g.peer) {  // peer-memory transport: the instance that stores the boundary planes
      tile_launch(t_tile<DIM, MODE, true, 0, true, true>, grid, smem, s, g, V, sc, part, h);
      return;
    }
  }
  tile_launch(t_tile<DIM, MODE, true, 0, true>, grid, smem, s, g, V, sc, part, h);
}

template <int DIM, int MODE>
cudaError_t attr_one(int smem, int* occ) {
  cudaError_t e = cudaFuncSetAttribute(t_tile<DIM, MODE, true, 0, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if constexpr (HasPeer<MODE>::v) {
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(t_tile<DIM, MODE, true, 0, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  }
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, t_tile<DIM, MODE, true, 0, true>, TNT,
                                                      smem);
  return e;
}

#define SEG_MODES(X)                                                                         \
  X(TM_A) X(TM_C) X(TM_RR1) X(TM_RR2) X(TM_GAP) X(TM_INIT1) X(TM_INIT2) X(TM_CL1) X(TM_CL2) \
  X(TM_CL3) X(TM_PC) X(TM_PCI1) X(TM_PCI2) X(TM_AN) X(TM_CN) X(TM_RR1N) X(TM_RR2N)         \
  X(TM_INIT1N) X(TM_SPB) X(TM_SPD)

template <int DIM>
bool dispatch(int mode, int grid, size_t smem, cudaStream_t s, const TileGeo& g, const Vecs& V,
              Scal* sc, Dd* part, Hist h) {
  switch (mode) {
#define SEG_CASE(M) \
  case M: launch_one<DIM, M>(grid, smem, s, g, V, sc, part, h); return true;
    SEG_MODES(SEG_CASE)
#undef SEG_CASE
    default: return false;
  }
}

template <int DIM>
cudaError_t dispatch_attr(int mode, int smem, int* occ) {
  switch (mode) {
#define SEG_CASE(M) \
  case M: return attr_one<DIM, M>(smem, occ);
    SEG_MODES(SEG_CASE)
#undef SEG_CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

bool tile_seg_launch(int dim, int mode, int grid, size_t smem, cudaStream_t s, const TileGeo& g,
                     const Vecs& V, Scal* sc, Dd* part, Hist h) {
  return dim == 3 ? dispatch<3>(mode, grid, smem, s, g, V, sc, part, h)
                  : dispatch<2>(mode, grid, smem, s, g, V, sc, part, h);
}

cudaError_t tile_seg_attr(int dim, int mode, int smem, int* occ) {
  return dim == 3 ? dispatch_attr<3>(mode, smem, occ) : dispatch_attr<2>(mode, smem, occ);
}
