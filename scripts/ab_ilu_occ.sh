#!/bin/bash
# 3D ILU(0) sweeps: zero-term steps (ablib/libI4.so) vs select steps (ablib/libI3.so),
# and 1 / 2 CTAs per SM (PBICG_ILU_OCC); M^-1 application time, parity suite at the
# product build's default
O=gpurun_out/ab_ilu_occ
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ilu.py -q -x 2>&1 | tail -3 > $O/tests.txt
cat $O/tests.txt
for occ in 1 2; do
  for c in cfg3 cfg4; do
    echo "occ=$occ" >> $O/$c.txt
    PBICG_ILU_OCC=$occ timeout 600 python scripts/ilu_exp.py $c ablib/libI3.so,ablib/libI4.so 16 >> $O/$c.txt 2>&1
  done
done
cat $O/cfg3.txt $O/cfg4.txt
PBICG_ILU_OCC=2 timeout 900 python -m pytest tests/test_gpu_ilu.py -q -x 2>&1 | tail -3 > $O/tests_occ2.txt
cat $O/tests_occ2.txt
