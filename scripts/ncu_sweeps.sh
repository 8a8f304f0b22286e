#!/bin/bash
# ncu --set full of the two cfg4 sweeps of iteration 0 (launches 3-4 of t_tile).
set -u
TAG=${1:-r01e}
O=gpurun_out
R=/tmp/ncu_$TAG
mkdir -p $R
P="python scripts/profile_solve.py --maxit 2 --rr 0"
$P > $O/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:t_tile -s 2 -c 2 -o $R/sw $P > $R/sw.log 2>&1
echo "sweeps=$?"
ncu -i $R/sw.ncu-rep --page raw --csv > $O/${TAG}_sweeps_raw.csv 2>/dev/null
ncu -i $R/sw.ncu-rep --page source --csv -c 1 > $O/${TAG}_sweepA_source.csv 2>/dev/null
du -sh $O
