#!/bin/bash
# stencil block Jacobi for the comparison methods: parity suite + cfg4 bench lines
O=gpurun_out/bjm
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_blockjacobi.py tests/test_gpu_methods.py -q -x 2>&1 | tail -15 > $O/tests.txt
cat $O/tests.txt
for m in bicgstab pipecg; do for b in 1 2 4 8; do
  timeout 300 python bench.py --method $m --block $b --no-cpu-baseline > $O/cfg4_${m}_b$b.json 2> $O/cfg4_${m}_b$b.err
done; done
