// tile_jac.h -- entry points of the Jacobi full-line tile-kernel instances
// (tile_jac.cu; suffix 1 = paired 16-byte path, 0 = odd nx).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

struct TileGeo;
struct Vecs;
struct Scal;
struct Dd;
struct Hist;

#define PBICG_JAC_DECL(V)                                                                    \
  bool tile_jac_launch_##V(int dim, int mode, int grid, size_t smem, cudaStream_t s,         \
                           const TileGeo& g, const Vecs& V_, Scal* sc, Dd* part, Hist h);    \
  cudaError_t tile_jac_attr_##V(int dim, int mode, int smem, int* occ);
PBICG_JAC_DECL(0)
PBICG_JAC_DECL(1)
#undef PBICG_JAC_DECL
