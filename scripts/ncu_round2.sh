#!/bin/bash
# ncu --set full of (1) the stencil sweeps after the sweep-A ring change (cfg4) and
# (2) the CSR path on cfg5 (window SpMVs + sweeps), Jacobi and block Jacobi b=4.
# The .ncu-rep files stay on the box; raw pages come back as CSV.
set -u
TAG=${1:-r01d}
O=gpurun_out
R=/tmp/ncu_$TAG
mkdir -p $R
P="python scripts/profile_solve.py --maxit 3 --rr 2"
$P > $O/${TAG}_cfg4_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:"t_tile<3, (0|1)," -c 4 -o $R/cfg4 $P > $R/cfg4.log 2>&1
echo "cfg4=$?"
ncu -i $R/cfg4.ncu-rep --page raw --csv > $O/${TAG}_cfg4_raw.csv 2>/dev/null
for b in 1 4; do
  P="python scripts/profile_solve.py --config cfg5 --maxit 3 --rr 0 --block $b"
  $P > $O/${TAG}_cfg5_b${b}_plain.log 2>&1 && \
  ncu --set full --clock-control none -k regex:"c_" -c 12 -o $R/cfg5_b$b $P > $R/cfg5_b$b.log 2>&1
  echo "cfg5 b$b=$?"
  ncu -i $R/cfg5_b$b.ncu-rep --page raw --csv > $O/${TAG}_cfg5_b${b}_raw.csv 2>/dev/null
done
du -sh $O
