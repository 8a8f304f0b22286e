#!/bin/bash
# acq_rel grid-reduction ticket: timeline and iteration-rate A/B (libH = before)
O=gpurun_out/ab_tk
mkdir -p $O
python scripts/timeline.py cfg2 cfg3/8 > $O/tl.txt 2>&1
python scripts/ab_libs.py ablib/libH.so ablib/libJ.so cfg2 cfg3/8 cfg3/4 cfg3 cfg4 > $O/iter.txt 2>&1
cat $O/iter.txt
