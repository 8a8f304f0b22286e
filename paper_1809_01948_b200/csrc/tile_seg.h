// tile_seg.h -- entry points of the x-segmented tile-kernel instances (tile_seg.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

struct TileGeo;
struct Vecs;
struct Scal;
struct Dd;
struct Hist;

bool tile_seg_launch(int dim, int mode, int grid, size_t smem, cudaStream_t s, const TileGeo& g,
                     const Vecs& V, Scal* sc, Dd* part, Hist h);
cudaError_t tile_seg_attr(int dim, int mode, int smem, int* occ);
