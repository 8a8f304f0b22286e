#!/bin/bash
# 3D ILU(0) sweeps: helper warp (boundary loads, progress polling / publication off the
# compute warps' step barriers; product build) vs ablib/libI4.so; parity suite first
O=gpurun_out/ab_ilu_helper
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ilu.py -q -x 2>&1 | tail -3 > $O/tests.txt
cat $O/tests.txt
L=ablib/libI9p.so,paper_1809_01948_b200/libpbicgstab.so
for c in cfg3 cfg4; do timeout 600 python scripts/ilu_exp.py $c $L 16 > $O/$c.txt 2>&1; cat $O/$c.txt; done

