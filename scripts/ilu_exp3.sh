#!/bin/bash
# 2D ILU(0) line wavefront: CTAs per SM (PBICG_ILU_OCC); 3D with the new default
O=gpurun_out/ilu_exp
mkdir -p $O
for occ in 0 1 2 4; do
  PBICG_ILU_OCC=$occ timeout 600 python scripts/ilu_exp.py cfg2 ablib/libL.so 16 | sed "s/^/occ=$occ /"
  PBICG_ILU_OCC=$occ timeout 600 python scripts/ilu_exp.py cfg1 ablib/libL.so 16 | sed "s/^/occ=$occ /"
done > $O/2d_occ.txt 2>&1
timeout 600 python scripts/ilu_exp.py cfg3 ablib/libL.so 16 >> $O/2d_occ.txt 2>&1
cat $O/2d_occ.txt
