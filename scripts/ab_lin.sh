#!/bin/bash
# balanced linear tile units (TileGeo::lin) vs (column, chunk) round-robin: A/B with
# graphs over the latency-regime cases, per-kernel A/B, parity suites with lin on
O=gpurun_out/ab_lin
mkdir -p $O
python scripts/ab_libs.py ablib/libL0.so ablib/libL1.so cfg3/8 cfg3/4 cfg3 cfg4/8 cfg2 cfg4 > $O/libs.txt 2>&1
cat $O/libs.txt
python scripts/ab_kernels.py ablib/libL0.so ablib/libL1.so cfg3 > $O/kernels.txt 2>&1
grep -h "sweep" $O/kernels.txt
PBICG_TILE_LIN=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_methods.py tests/test_gpu_blockjacobi.py tests/test_gpu_multirank.py tests/test_gpu_autorr.py -q -x 2>&1 | tail -3 > $O/tests_lin.txt
cat $O/tests_lin.txt
