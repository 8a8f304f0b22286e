#!/bin/bash
# 3D ILU(0) sweeps: progress published as completed steps (tight hand-over) vs the
# all-lines x-count; M^-1 application time, ILU parity suite, bench lines
O=gpurun_out/ab_ilu_steps
mkdir -p $O
for c in cfg3 cfg4; do python scripts/ilu_exp.py $c ablib/libI0.so,ablib/libI1.so 16 > $O/$c.txt 2>&1; cat $O/$c.txt; done
timeout 900 python -m pytest tests/test_gpu_ilu.py -q -x 2>&1 | tail -3 > $O/tests.txt
cat $O/tests.txt
for c in cfg3 cfg4; do timeout 300 python bench.py --config $c --block ilu0 --no-cpu-baseline > $O/bench_${c}_ilu0.json 2> $O/bench_${c}.err; done
timeout 300 python bench.py --config cfg3 --block icc0 --method pipecg --no-cpu-baseline > $O/bench_cfg3_icc0_pcg.json 2> /dev/null
tail -c 400 $O/bench_cfg3_ilu0.json
