#!/bin/bash
# tile-geometry experiment: cfg3 / cfg4 it/s for TY and chunk-count overrides
for cfg in cfg3 cfg4; do
  for ty in 0 1 2 3; do
    for nch in 0 2 4 8 16; do
      if [ $ty = 0 ]; then unset PBICG_TILE_TY; else export PBICG_TILE_TY=$ty; fi
      if [ $nch = 0 ]; then unset PBICG_TILE_NCHUNKS; else export PBICG_TILE_NCHUNKS=$nch; fi
      v=$(python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f %.3f' % (d['value'], d['roofline']['iteration_frac']))")
      echo "$cfg TY=$ty NCH=$nch $v"
    done
  done
done
