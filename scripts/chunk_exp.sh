#!/bin/bash
# chunk-count experiment on the per-rank slabs of the strong-scaling runs (cfg4 /
# cfg3 at 2, 4, 8 GPUs) measured on one GPU: it/s for PBICG_TILE_NCHUNKS overrides
for shape in "3 512 512 64" "3 512 512 128" "3 512 512 256" "3 256 256 32" "3 256 256 64" "3 256 256 128" "3 256 256 256"; do
  for nch in 0 1 2 3 4 5 6 8 12 16 24; do
    if [ $nch = 0 ]; then unset PBICG_TILE_NCHUNKS; else export PBICG_TILE_NCHUNKS=$nch; fi
    echo "NCH=$nch $(python scripts/measure_shape.py $shape 2>/dev/null | tail -1)"
  done
done
