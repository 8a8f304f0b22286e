#!/bin/bash
# One gpurun call: launch list of the default bench + `ncu --set full` of the tile
# kernels for p-BiCGStab (periodic and automated replacement), classic BiCGStab, p-CG.
# The .ncu-rep files stay on the box (gpurun_out is capped at 64 MiB): their raw
# pages come back as CSV, plus the source page of the p-BiCGStab capture.
# usage (under gpurun): bash scripts/ncu_round.sh TAG
set -u
TAG=${1:-r01}
O=gpurun_out
R=/tmp/ncu_$TAG
mkdir -p $R
BENCH="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$BENCH > $O/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 1240 -c 420 --csv \
    --log-file $O/${TAG}_launches.csv $BENCH > $R/launch.log 2>&1
echo launches=$?
for cfg in "0 0 14" "0 1 14" "1 0 8" "2 0 6"; do
  set -- $cfg
  P="python scripts/profile_solve.py --maxit 3 --rr 2 --method $1 --rr-auto $2"
  $P > $O/${TAG}_m$1a$2_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:t_tile -c $3 \
      -o $R/m$1a$2 $P > $R/m$1a$2_ncu.log 2>&1
  echo "full m$1 a$2=$?"
  ncu -i $R/m$1a$2.ncu-rep --page raw --csv > $O/${TAG}_m$1a$2_raw.csv 2>/dev/null
  if [ "$1$2" = "00" ]; then
    ncu -i $R/m$1a$2.ncu-rep --page source --csv -k regex:"t_tile<3, 1," -c 1 \
        > $O/${TAG}_m00_sweepC_source.csv 2>/dev/null
  fi
done
du -sh $O
