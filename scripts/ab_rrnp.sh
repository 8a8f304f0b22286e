#!/bin/bash
# replacement step: row pairs per thread NP = 2 (default) / 3 / 4, per-kernel A/B;
# randomised sweep of the stencil block-Jacobi comparison methods
O=gpurun_out/ab_rrnp
mkdir -p $O
python scripts/ab_kernels.py ablib/libR2.so ablib/libR4.so cfg4 cfg3 > $O/r2r4.txt 2>&1
python scripts/ab_kernels.py ablib/libR2.so ablib/libR3.so cfg4 cfg3 > $O/r2r3.txt 2>&1
grep -h "rr" $O/r2r4.txt $O/r2r3.txt
PBICG_FUZZ_SCALE=40 timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -k block_jacobi_methods 2>&1 | tail -3 > $O/fuzz_bjm.txt
cat $O/fuzz_bjm.txt
