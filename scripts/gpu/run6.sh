python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r2_prof6.txt
: > $O
python scripts/profile_elementwise.py alg1 8 5 >> $O 2>&1
python scripts/profile_elementwise.py alg1 4 5 >> $O 2>&1
python scripts/profile_c5.py 4 8192 4 >> $O 2>&1
python scripts/profile_c5.py 8 8192 3 >> $O 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> $O
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench6.json 2> gpurun_out/r2_bench6.err
tail -2 gpurun_out/r2_bench6.err >> $O
cat $O
