python -c "import __graft_entry__ as g; g.build()"
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_suite.log 2>&1
tail -3 gpurun_out/gpu_suite.log
python scripts/bench_layers.py --chain --reps 50 2>&1 | grep "chain of"
