#!/bin/bash
# ncu --set full of the cfg5 CSR path with the TMA-staged sweeps (Jacobi): init,
# window SpMVs, c_sweep_tma A/C.  Also the launch list (gpu__time_duration) of the
# default bench command.  Raw pages come back as CSV.
set -u
TAG=${1:-r01h}
O=gpurun_out
R=/tmp/ncu_$TAG
mkdir -p $R
P="python scripts/profile_solve.py --config cfg5 --maxit 3 --rr 0"
$P > $O/${TAG}_cfg5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"c_" -c 12 -o $R/cfg5 $P > $R/cfg5.log 2>&1
echo "cfg5=$?"
ncu -i $R/cfg5.ncu-rep --page raw --csv > $O/${TAG}_cfg5_raw.csv 2>/dev/null
B="python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu-baseline"
$B > $O/${TAG}_bench_cfg5.json 2>$O/${TAG}_bench_cfg5.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $O/${TAG}_launches_cfg5.csv $B > /dev/null 2>&1
echo "launches=$?"
du -sh $O
