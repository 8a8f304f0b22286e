#!/bin/bash
# ILU(0) stencil sweep tuning: builds (ILU_T threads, ILU_K steps per publication,
# ILU_BMAX boundary slots) x tile widths (PBICG_ILU_TA)
O=gpurun_out/ilu_exp
mkdir -p $O
L=$(ls ablib/libilu_*.so | tr '\n' ',' | sed 's/,$//')
timeout 1500 python scripts/ilu_exp.py ${1:-cfg3} $L ${2:-16,8,4} > $O/${1:-cfg3}_2.txt 2>&1
cat $O/${1:-cfg3}_2.txt
