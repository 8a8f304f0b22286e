#!/bin/bash
# split schedule (option schedule 2) on cfg4: per-kernel times (bench mode) and ncu
# --set full of the stand-alone SpMV tiles (t_tile launches: init1, init2, SPB, SPD, ...)
TAG=${1:-r02c}
O=gpurun_out
AB_SCHED=2 python scripts/ab_kernels.py ablib/libD.so ${2:-ablib/libD.so} cfg4 cfg3 cfg3/8 > $O/${TAG}_split_ab.txt 2>&1
P="python scripts/profile_solve.py --maxit 2 --rr 0 --schedule 2"
$P > $O/${TAG}_split_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:t_tile -s 2 -c 2 -o $O/${TAG}_split $P > $O/${TAG}_split_ncu.log 2>&1
echo "split ncu=$?"
ncu -i $O/${TAG}_split.ncu-rep --page raw --csv > $O/${TAG}_split_raw.csv 2>/dev/null
cat $O/${TAG}_split_ab.txt
