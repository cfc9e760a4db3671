python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_suite.log 2>&1
tail -n 2 gpurun_out/gpu_suite.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
