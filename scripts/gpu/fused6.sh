python -c "import __graft_entry__ as g; g.build()"
for d in 1 2; do for pfd in 2 4 6 8 12; do
 echo "depth=$d pfd=$pfd"; MPC_FUSED_DEPTH=$d MPC_FUSED_PF=1 MPC_FUSED_PFD=$pfd python scripts/bench_layers.py --model text --chain --reps 50 2>&1 | grep "chain of"
done; done
