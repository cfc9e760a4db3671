python -c "import __graft_entry__ as g; g.build()"
for nf in 0 1; do for d in 1 2; do
 echo "nofence=$nf depth=$d"; MPC_FUSED_NOFENCE=$nf MPC_FUSED_DEPTH=$d python scripts/bench_layers.py --model text --chain --reps 50 2>&1 | grep "chain of"
done; done
