#!/bin/bash
# 3D ILU(0) sweeps: ILU_K = 4 (ablib/libI11.so) vs 8 (product build)
O=gpurun_out/ab_ilu_k
mkdir -p $O
L=paper_1809_01948_b200/libpbicgstab.so,ablib/libI11.so
for c in cfg3 cfg4; do timeout 600 python scripts/ilu_exp.py $c $L 16 > $O/$c.txt 2>&1; cat $O/$c.txt; done
