#!/bin/bash
# deferred finalize: GPU suite, then iteration rates (graphs) and per-kernel times A/B
O=gpurun_out/ab_df
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > $O/tests.txt
cat $O/tests.txt
python scripts/ab_libs.py ablib/libD.so ablib/libE.so cfg2 cfg3/8 cfg3/4 cfg3 cfg4/8 cfg4 > $O/iter.txt 2>&1
cat $O/iter.txt
python scripts/ab_kernels.py ablib/libD.so ablib/libE.so cfg4 cfg2 > $O/kern.txt 2>&1
grep -h "sweep" $O/kern.txt
