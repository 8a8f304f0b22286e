#!/bin/bash
# round-2 bench lines (one gpurun call): the headline and the ILU(0)/ICC(0) lines,
# each a separate bench.py process; JSON lines to gpurun_out/r02_bench/*.json
mkdir -p gpurun_out/r02_bench
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/r02_bench/$name.json 2> gpurun_out/r02_bench/$name.err; echo "$name exit=$?"; }
run cfg4 --steps 10 --warmup 3
run cfg4_ilu0 --block ilu0 --steps 3 --warmup 3 --no-cpu-baseline
run cfg3_ilu0 --config cfg3 --block ilu0 --steps 5 --warmup 3 --no-cpu-baseline
run cfg3 --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline
run cfg2_ilu0 --config cfg2 --block ilu0 --steps 5 --warmup 3 --no-cpu-baseline
run cfg1_icc0 --config cfg1 --block icc0 --steps 5 --warmup 3 --no-cpu-baseline
run cfg1 --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline
run cfg1_icc0_bicgstab --config cfg1 --block icc0 --method bicgstab --steps 5 --warmup 3 --no-cpu-baseline
run cfg1_icc0_pipecg --config cfg1 --block icc0 --method pipecg --steps 5 --warmup 3 --no-cpu-baseline
run cfg5 --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline
run reference --impl reference --steps 2 --warmup 1
