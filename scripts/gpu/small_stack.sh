python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_suite_small.log 2>&1; tail -2 gpurun_out/gpu_suite_small.log
python scripts/bench_layers.py --chain --reps 50 2>&1 | grep "chain of" | cut -c1-70
python scripts/bench_configs.py 2>/dev/null | grep -o '"C1": {[^}]*}' | head -2
