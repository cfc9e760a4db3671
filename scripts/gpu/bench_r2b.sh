python -c "import __graft_entry__ as g; g.build()"
python bench.py > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err
tail -c 300 gpurun_out/bench_r2b.json
