#!/bin/bash
# ncu --set full of the cfg4 3D ILU(0) sweeps with the per-instruction (source page) stall samples
O=gpurun_out/ncu_ilu_src
mkdir -p $O
R=/tmp/ncu_ilu_src
mkdir -p $R
I4="python scripts/profile_ilu.py ${1:-cfg4} 2"
$I4 > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -f -k regex:k_ilu -s 2 -c 2 -o $R/ilu4 $I4 > $O/ncu.log 2>&1
echo "ilu4=$?"
ncu -i $R/ilu4.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $R/ilu4.ncu-rep --page source --csv --print-source sass > $O/source_sass.csv 2>/dev/null
du -sh $O
