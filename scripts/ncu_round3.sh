#!/bin/bash
# ncu --set full of iteration 0 of: stencil block Jacobi b=2 and b=4 (cfg4 sweeps) and
# the split stencil schedule (sweeps + stand-alone SpMVs).  Raw pages come back as CSV.
set -u
TAG=${1:-r01f}
O=gpurun_out
R=/tmp/ncu_$TAG
mkdir -p $R
for b in 2 4; do
  P="python scripts/profile_solve.py --maxit 2 --rr 0 --block $b"
  $P > $O/${TAG}_bj$b.log 2>&1 && \
  ncu --set full --clock-control none -k regex:t_tile -s 2 -c 2 -o $R/bj$b $P > $R/bj$b.log 2>&1
  echo "bj$b=$?"
  ncu -i $R/bj$b.ncu-rep --page raw --csv > $O/${TAG}_bj${b}_raw.csv 2>/dev/null
done
P="python scripts/profile_solve.py --maxit 2 --rr 0 --schedule 2"
$P > $O/${TAG}_split.log 2>&1 && \
ncu --set full --clock-control none -s 3 -c 4 -o $R/split $P > $R/split.log 2>&1
echo "split=$?"
ncu -i $R/split.ncu-rep --page raw --csv > $O/${TAG}_split_raw.csv 2>/dev/null
du -sh $O
