#!/bin/bash
# Final-build evidence for the default bench (cfg4): ncu --set full of the two sweeps
# of iteration 0, and the launch list (gpu__time_duration) of `bench.py --steps 2`.
set -u
TAG=${1:-r01j}
O=gpurun_out
R=/tmp/ncu_$TAG
mkdir -p $R
P="python scripts/profile_solve.py --maxit 2 --rr 0"
$P > $O/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:t_tile -s 2 -c 2 -o $R/sw $P > $R/sw.log 2>&1
echo "sweeps=$?"
ncu -i $R/sw.ncu-rep --page raw --csv > $O/${TAG}_sweeps_raw.csv 2>/dev/null
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$B > $O/${TAG}_bench.json 2>$O/${TAG}_bench.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $O/${TAG}_launches_cfg4.csv $B > /dev/null 2>&1
echo "launches=$?"
du -sh $O
