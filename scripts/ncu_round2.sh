#!/bin/bash
# Round-2 ncu evidence (one gpurun call): the headline sweeps (cfg4, iteration 0),
# the launch list of the default bench, and the ILU(0) wavefront kernels (cfg1 ICC(0),
# 2D; cfg3 ILU(0), 3D).  Every ncu run follows the same command run plain.
set -u
TAG=${1:-r02a}
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
I1="python scripts/profile_ilu.py cfg1 3"
$I1 > $O/${TAG}_ilu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ilu -s 2 -c 2 -o $R/ilu1 $I1 > $R/ilu1.log 2>&1
echo "ilu1=$?"
ncu -i $R/ilu1.ncu-rep --page raw --csv > $O/${TAG}_ilu_cfg1_raw.csv 2>/dev/null
I3="python scripts/profile_ilu.py cfg3 2"
$I3 > $O/${TAG}_ilu3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ilu -s 2 -c 2 -o $R/ilu3 $I3 > $R/ilu3.log 2>&1
echo "ilu3=$?"
ncu -i $R/ilu3.ncu-rep --page raw --csv > $O/${TAG}_ilu_cfg3_raw.csv 2>/dev/null
du -sh $O
