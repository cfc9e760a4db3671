python -c "import __graft_entry__ as g; g.build()"
for d in 1 2; do
MPC_FUSED_DEBUG=1 MPC_FUSED_DEPTH=$d MPC_FUSED_PF=1 MPC_FUSED_PFD=2 python scripts/bench_layers.py --model text --chain --reps 1 2>&1 | grep fused_small | tail -2
done
