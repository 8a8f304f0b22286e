#!/bin/bash
# tall-tile stand-alone SpMVs of the split schedule: parity tests, per-kernel A/B, ncu
O=gpurun_out/ab_spt
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "split or schedule or tall" 2>&1 | tail -3 > $O/tests.txt
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_nccl.py -q -x 2>&1 | tail -3 >> $O/tests.txt
cat $O/tests.txt
AB_SCHED=2 python scripts/ab_kernels.py ablib/libF.so ablib/libG.so cfg4 cfg3 cfg3/8 > $O/np4.txt 2>&1
PBICG_SPT_NP=2 AB_SCHED=2 python scripts/ab_kernels.py ablib/libF.so ablib/libG.so cfg4 cfg3 cfg3/8 > $O/np2.txt 2>&1
grep -h spmv $O/np4.txt $O/np2.txt
P="python scripts/profile_solve.py --maxit 2 --rr 0 --schedule 2"
ncu --set full --clock-control none --import-source on -k regex:t_spmv3 -c 2 -o $O/spt $P > $O/ncu.log 2>&1
echo "ncu=$?"
ncu -i $O/spt.ncu-rep --page raw --csv > $O/spt_raw.csv 2>/dev/null
