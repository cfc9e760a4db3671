# round-2 third session re-entry: build, smoke, GPU suite, bench at HEAD
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_suite.log 2>&1
tail -5 gpurun_out/gpu_suite.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 600 gpurun_out/bench.json
