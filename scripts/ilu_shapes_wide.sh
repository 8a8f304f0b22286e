#!/bin/bash
# wide randomised sweep of the 3D ILU(0) wavefront sweeps: PBICG_ILU_SHAPES random grids per
# seed offset (single handle + loopback ranks), bitwise vs the oracle; first the odd-plane
# loopback reproduction (window SpMV alignment) and the suites that share the CSR schedule
O=gpurun_out/ilu_shapes_wide
mkdir -p $O
timeout 120 python scripts/repro_ilu_odd.py - ilu0 > $O/repro.txt 2>&1; cat $O/repro.txt
timeout 900 python -m pytest tests/test_gpu_ilu.py tests/test_gpu_regressions.py -q -x 2>&1 | tail -3 > $O/default.txt
cat $O/default.txt
for off in 1 2 3; do
  PBICG_FUZZ_OFFSET=$off PBICG_ILU_SHAPES=${1:-150} timeout 1200 python -m pytest tests/test_gpu_ilu.py -q \
      -k "random_shapes" 2>&1 | tail -3 > $O/offset_$off.txt
  cat $O/offset_$off.txt
done
