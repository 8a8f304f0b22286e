#!/bin/bash
# round-2 validation of the current build: GPU suite, smoke, bench lines (Jacobi and
# ILU(0)/ICC(0)), launch list
O=gpurun_out/r02v
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > $O/tests.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 >> $O/tests.txt
cat $O/tests.txt
timeout 400 python bench.py > $O/cfg4.json 2> $O/cfg4.err
for c in cfg3 cfg5 cfg2; do timeout 300 python bench.py --config $c --no-cpu-baseline > $O/$c.json 2> $O/$c.err; done
timeout 300 python bench.py --schedule 2 --no-cpu-baseline > $O/cfg4_split.json 2> $O/cfg4_split.err
timeout 300 python bench.py --rr-auto 1 --no-cpu-baseline > $O/cfg4_rrauto.json 2> $O/cfg4_rrauto.err
for c in cfg3 cfg4; do timeout 300 python bench.py --config $c --block ilu0 --no-cpu-baseline > $O/${c}_ilu0.json 2> $O/${c}_ilu0.err; done
timeout 300 python bench.py --config cfg3 --block icc0 --method pipecg --no-cpu-baseline > $O/cfg3_icc0_pcg.json 2> /dev/null
timeout 300 python bench.py --config cfg1 --block icc0 --no-cpu-baseline > $O/cfg1_icc0.json 2> /dev/null
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $O/launches_cfg4.csv $B > /dev/null 2>&1
echo "launches=$?"
