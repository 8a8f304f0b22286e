#!/bin/bash
# 3D ILU(0) sweeps: transposed (coalesced) operand copies and result stores vs one
# row per lane per instruction; M^-1 application time (ablib/libI1.so = before,
# product library = after), ILU parity suite, bench lines, ncu of the cfg4 sweeps
O=gpurun_out/ab_ilu_v2
mkdir -p $O
L=ablib/libI2.so,paper_1809_01948_b200/libpbicgstab.so
timeout 900 python -m pytest tests/test_gpu_ilu.py -q -x 2>&1 | tail -3 > $O/tests.txt
cat $O/tests.txt
for c in cfg3 cfg4; do timeout 600 python scripts/ilu_exp.py $c $L 16 > $O/$c.txt 2>&1; cat $O/$c.txt; done
for c in cfg3 cfg4; do timeout 300 python bench.py --config $c --block ilu0 --no-cpu-baseline > $O/bench_${c}_ilu0.json 2> $O/bench_${c}.err; done
timeout 300 python bench.py --config cfg3 --block icc0 --method pipecg --no-cpu-baseline > $O/bench_cfg3_icc0_pcg.json 2> /dev/null
tail -c 300 $O/bench_cfg3_ilu0.json; tail -c 300 $O/bench_cfg4_ilu0.json
R=/tmp/ncu_ilu_tr
mkdir -p $R
I4="python scripts/profile_ilu.py cfg4 2"
$I4 > $O/ilu4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ilu -s 2 -c 2 -o $R/ilu4 $I4 > $R/ilu4.log 2>&1
echo "ilu4=$?"
ncu -i $R/ilu4.ncu-rep --page raw --csv > $O/ilu_cfg4_raw.csv 2>/dev/null
ncu -i $R/ilu4.ncu-rep --page details --csv > $O/ilu_cfg4_details.csv 2>/dev/null
du -sh $O
