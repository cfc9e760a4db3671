python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_suite_tma.log 2>&1; tail -2 gpurun_out/gpu_suite_tma.log
python scripts/bench_layers.py --chain --reps 50 2>&1 | grep "chain of" | cut -c1-60
python scripts/bench_layers.py --chain --reps 50 --model resnet50 --conv 2>&1 | grep "chain of" | cut -c1-80
