// tile_bj.h -- entry points of the block-Jacobi tile-kernel instances (tile_bj.cu,
// one object per block size B = 2, 4, 8).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

struct TileGeo;
struct Vecs;
struct Scal;
struct Dd;
struct Hist;

#define PBICG_BJ_DECL(B)                                                                     \
  bool tile_bj_launch_##B(int dim, int mode, int grid, size_t smem, cudaStream_t s,          \
                          const TileGeo& g, const Vecs& V, Scal* sc, Dd* part, Hist h);      \
  cudaError_t tile_bj_attr_##B(int dim, int mode, int smem, int* occ);
PBICG_BJ_DECL(2)
PBICG_BJ_DECL(4)
PBICG_BJ_DECL(8)
#undef PBICG_BJ_DECL
