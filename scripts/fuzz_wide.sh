#!/bin/bash
# wide randomised sweep of the current build (PBICG_FUZZ_SCALE x the default cases)
O=gpurun_out/fuzz_r02
mkdir -p $O
PBICG_FUZZ_SCALE=${1:-25} timeout 2400 python -m pytest tests/test_gpu_fuzz.py -q -p no:randomly 2>&1 | tail -15 > $O/fuzz_scale${1:-25}.txt
cat $O/fuzz_scale${1:-25}.txt
