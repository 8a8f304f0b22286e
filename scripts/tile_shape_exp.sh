#!/bin/bash
# tile-shape experiments for the latency regime (small grids): full-line tiles with
# fewer lines per tile (PBICG_TILE_TY) and x-segmented tiles (PBICG_TILE_SEG=sx)
for c in cfg2 cfg3/8 cfg3/4; do
  echo "== $c default"; python scripts/measure_persist.py $c
  for ty in 2 1; do echo "== $c TY=$ty"; PBICG_TILE_TY=$ty python scripts/measure_persist.py $c; done
  for sx in 512 256 128; do echo "== $c SEG=$sx"; PBICG_TILE_SEG=$sx python scripts/measure_persist.py $c; done
done
