O=gpurun_out/ab_rr2
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > $O/tests.txt
python scripts/ab_kernels.py ablib/libB.so ablib/libD.so cfg4 cfg3 > $O/jac.txt 2>&1
bash scripts/ncu_rr.sh r02b
cat $O/tests.txt; grep -h "rr\|init" $O/jac.txt
