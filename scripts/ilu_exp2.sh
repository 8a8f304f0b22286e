#!/bin/bash
# ILU(0) stencil sweep tuning: CTAs per SM (PBICG_ILU_OCC) x tile widths
O=gpurun_out/ilu_exp
mkdir -p $O
L=$(ls ablib/libilu_*.so | tr '\n' ',' | sed 's/,$//')
for occ in 1 2; do
  PBICG_ILU_OCC=$occ timeout 900 python scripts/ilu_exp.py cfg3 $L 16,8 | sed "s/^/occ=$occ /"
done > $O/cfg3_occ.txt 2>&1
PBICG_ILU_OCC=1 timeout 900 python scripts/ilu_exp.py cfg4 $L 16,8 | sed "s/^/occ=1 /" >> $O/cfg3_occ.txt 2>&1
PBICG_ILU_OCC=2 timeout 900 python scripts/ilu_exp.py cfg4 ablib/libilu_T256_K8_B32.so 16 | sed "s/^/occ=2 /" >> $O/cfg3_occ.txt 2>&1
cat $O/cfg3_occ.txt
