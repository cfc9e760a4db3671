python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for o in 1 0; do echo "occ=$o"; MPC_SPLIT2_OCC=$o python scripts/bench_layers.py --chain --reps 50 2>&1 | grep "chain of" | cut -c1-60; done
