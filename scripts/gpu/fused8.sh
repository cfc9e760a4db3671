python -c "import __graft_entry__ as g; g.build()"
for d in 1 2 3; do for pfd in 0 2; do
 echo "depth=$d pfd=$pfd"; MPC_FUSED_DEPTH=$d MPC_FUSED_PF=1 MPC_FUSED_PFD=$pfd python scripts/bench_layers.py --model text --chain --reps 50 2>&1 | grep "chain of"
done; done
MPC_FUSED_DEPTH=1 MPC_FUSED_PF=1 MPC_FUSED_PFD=0 MPC_GEMM_DEBUG=1 python scripts/bench_layers.py --model text --chain --reps 2 > /dev/null 2>&1
