O=gpurun_out/v0
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $O/tests.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 >> $O/tests.txt
timeout 300 python bench.py > $O/cfg4.json 2> $O/cfg4.err
timeout 300 python bench.py --config cfg2 --no-cpu-baseline > $O/cfg2.json 2> $O/cfg2.err
timeout 300 python bench.py --config cfg3 --no-cpu-baseline > $O/cfg3.json 2> $O/cfg3.err
cat $O/tests.txt
