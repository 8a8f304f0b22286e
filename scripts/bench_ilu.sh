#!/bin/bash
# ILU(0)/ICC(0) bench lines (one gpurun call)
mkdir -p gpurun_out/r02_bench
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/r02_bench/$name.json 2> gpurun_out/r02_bench/$name.err; echo "$name exit=$?"; }
run cfg1_icc0 --config cfg1 --block icc0 --steps 5 --warmup 3 --no-cpu-baseline
run cfg1_icc0_bicgstab --config cfg1 --block icc0 --method bicgstab --steps 5 --warmup 3 --no-cpu-baseline
run cfg1_icc0_pipecg --config cfg1 --block icc0 --method pipecg --steps 5 --warmup 3 --no-cpu-baseline
run cfg2_ilu0 --config cfg2 --block ilu0 --steps 5 --warmup 3 --no-cpu-baseline
run cfg3_ilu0 --config cfg3 --block ilu0 --steps 5 --warmup 3 --no-cpu-baseline
run cfg4_ilu0 --block ilu0 --steps 3 --warmup 3 --no-cpu-baseline
