#!/bin/bash
# replacement step on tall tiles: GPU suite, per-kernel A/B (libJ = t_tile RR), ncu
O=gpurun_out/ab_lrr
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $O/tests.txt
cat $O/tests.txt
python scripts/ab_kernels.py ablib/libJ.so ablib/libK.so cfg4 cfg3 > $O/jac.txt 2>&1
AB_SCHED=2 python scripts/ab_kernels.py ablib/libJ.so ablib/libK.so cfg4 > $O/split.txt 2>&1
grep -h "rr\|spmv" $O/jac.txt $O/split.txt
P="python scripts/profile_solve.py --maxit 2 --rr 2"
ncu --set full --clock-control none --import-source on -k regex:t_light3 -c 2 -o $O/lrr $P > $O/ncu.log 2>&1
echo "ncu=$?"
ncu -i $O/lrr.ncu-rep --page raw --csv > $O/lrr_raw.csv 2>/dev/null
