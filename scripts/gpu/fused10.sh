python -c "import __graft_entry__ as g; g.build()"
MPC_FUSED_DEBUG=1 python scripts/bench_layers.py --model text --chain --reps 1 2>&1 | grep fused_small | head -2
