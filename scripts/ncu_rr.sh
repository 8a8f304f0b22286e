#!/bin/bash
# ncu --set full of the tile replacement step (RR1, RR2) on cfg4: one solve of 2
# iterations with a replacement in iteration 1 (launch order init1, init2, A, C, A, C,
# RR1, RR2)
TAG=${1:-r02b}
O=gpurun_out
P="python scripts/profile_solve.py --maxit 2 --rr 2"
$P > $O/${TAG}_rr_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:t_tile -s 6 -c 2 -o $O/${TAG}_rr $P > $O/${TAG}_rr_ncu.log 2>&1
echo "rr ncu=$?"
ncu -i $O/${TAG}_rr.ncu-rep --page raw --csv > $O/${TAG}_rr_raw.csv 2>/dev/null
