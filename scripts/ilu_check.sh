#!/bin/bash
# ILU(0) after the one-CTA-per-SM 3D sweep: parity tests and bench lines
O=gpurun_out/ilu_r02
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ilu.py -q 2>&1 | tail -3 > $O/tests.txt
cat $O/tests.txt
timeout 600 python bench.py --config cfg3 --block ilu0 --steps 5 --warmup 3 --no-cpu-baseline > $O/cfg3_ilu0.json 2> $O/cfg3_ilu0.err
timeout 900 python bench.py --block ilu0 --steps 3 --warmup 3 --no-cpu-baseline > $O/cfg4_ilu0.json 2> $O/cfg4_ilu0.err
for f in $O/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels'].get('prec',{})
print('$f', round(d['value'],2), d['unit'], 'prec_ms', k.get('avg_ms'))"; done
