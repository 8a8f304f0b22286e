#!/bin/bash
# host-parity fast start + acq_rel ticket: GPU suite, timeline, iteration-rate A/B
O=gpurun_out/ab_hp
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $O/tests.txt
cat $O/tests.txt
python scripts/timeline.py cfg2 cfg3/8 > $O/tl.txt 2>&1
python scripts/ab_libs.py ablib/libH.so ablib/libI.so cfg2 cfg3/8 cfg3/4 cfg3 cfg4 > $O/iter.txt 2>&1
cat $O/iter.txt
