python -c "import __graft_entry__ as g; g.build()"
for d in 1 2; do for pfd in 0 2 4; do
 echo "depth=$d pfd=$pfd"; MPC_FUSED_DEPTH=$d MPC_FUSED_PFD=$pfd python scripts/bench_layers.py --model text --chain --reps 50 2>&1 | grep "chain of"
done; done
for d in 1 2; do MPC_FUSED_DEPTH=$d MPC_FUSED_DEBUG=1 python scripts/bench_layers.py --model text --chain --reps 1 2>&1 | grep fused_small | head -2; done
