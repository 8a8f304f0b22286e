#!/bin/bash
# 3D ILU(0) sweeps (helper-warp kernel): register cap for 2 CTAs per SM (ablib/libI7.so,
# -DILU_MINB=2) at PBICG_ILU_OCC = 1, 2 vs the product build
O=gpurun_out/ab_ilu_occ2
mkdir -p $O
for occ in 1 2; do
  for c in cfg3 cfg4; do
    echo "occ=$occ" >> $O/$c.txt
    PBICG_ILU_OCC=$occ timeout 600 python scripts/ilu_exp.py $c paper_1809_01948_b200/libpbicgstab.so,ablib/libI7.so 16 >> $O/$c.txt 2>&1
  done
done
cat $O/cfg3.txt $O/cfg4.txt
