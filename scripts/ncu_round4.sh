#!/bin/bash
# ncu --set full of iteration 0's sweeps of stencil block Jacobi b=4 and b=8 (cfg4,
# the transform-stage tile kernels).  Raw pages come back as CSV.
set -u
TAG=${1:-r01g}
O=gpurun_out
R=/tmp/ncu_$TAG
mkdir -p $R
for b in 4 8; do
  P="python scripts/profile_solve.py --maxit 2 --rr 0 --block $b"
  $P > $O/${TAG}_bj$b.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:t_tile -s 2 -c 2 -o $R/bj$b $P > $R/bj$b.log 2>&1
  echo "bj$b=$?"
  ncu -i $R/bj$b.ncu-rep --page raw --csv > $O/${TAG}_bj${b}_raw.csv 2>/dev/null
done
du -sh $O
