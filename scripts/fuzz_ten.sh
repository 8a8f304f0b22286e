#!/bin/bash
# ten independent 6,000-case randomised sweeps (PBICG_FUZZ_SCALE=100,
# seed offsets 1..10) of the current build
O=gpurun_out/fuzz_ten
mkdir -p $O
for j in 1 2 3 4 5 6 7 8 9 10; do
  PBICG_FUZZ_OFFSET=$j PBICG_FUZZ_SCALE=100 timeout 900 python -m pytest tests/test_gpu_fuzz.py -q 2>&1 | tail -4 > $O/sweep_$j.txt
  echo "sweep $j: $(tail -1 $O/sweep_$j.txt)"
done
