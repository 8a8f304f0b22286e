#!/bin/bash
# full GPU validation + the bench lines DESIGN.md section 8 quotes (one B200)
O=gpurun_out/final
mkdir -p $O
python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > $O/cfg4.json 2> $O/cfg4.err
for c in cfg3 cfg5; do python bench.py --config $c --no-cpu-baseline > $O/$c.json 2> $O/$c.err; done
python bench.py --config cfg2 --no-cpu-baseline > $O/cfg2.json 2> $O/cfg2.err
python bench.py --rr-auto 1 --no-cpu-baseline > $O/cfg4_rrauto.json 2>/dev/null
python bench.py --method bicgstab --no-cpu-baseline > $O/cfg4_bicgstab.json 2>/dev/null
python bench.py --method pipecg --no-cpu-baseline > $O/cfg4_pipecg.json 2>/dev/null
python bench.py --schedule 2 --no-cpu-baseline > $O/cfg4_split.json 2>/dev/null
python bench.py --overlap 0 --no-cpu-baseline > $O/cfg4_overlap0.json 2>/dev/null
python bench.py --impl reference --steps 2 --warmup 3 > $O/reference.json 2>/dev/null
for f in $O/*.json; do python - "$f" <<'PY'
import json, sys
p = sys.argv[1]
try:
    d = json.loads(open(p).read().strip().splitlines()[-1])
except Exception as e:
    print(p, "FAILED", e); sys.exit()
r = d.get("roofline") or {}
print(p.split("/")[-1], round(d["value"], 2), d["unit"], "iter_frac", r.get("iteration_frac"),
      r.get("kernel"), r.get("frac"), "e2e", (d.get("e2e") or {}).get("value"),
      (d.get("clocks") or {}).get("sm_mhz"))
PY
done
