#!/bin/bash
# deferred finalize round 2: timelines with defer on / off, iteration-rate A/B
O=gpurun_out/ab_df2
mkdir -p $O
TL_OPTS=defer=0 python scripts/timeline.py cfg2 cfg3/8 > $O/tl_off.txt 2>&1
TL_OPTS=defer=1 python scripts/timeline.py cfg2 cfg3/8 > $O/tl_on.txt 2>&1
python scripts/ab_libs.py ablib/libD.so ablib/libF.so cfg2 cfg3/8 cfg4 > $O/iter.txt 2>&1
cat $O/iter.txt
