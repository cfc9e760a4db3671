python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_fused_small.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for cyc in 1 0; do for d in 1 2; do for pfd in 0 2 4; do
 echo "cyc=$cyc depth=$d pfd=$pfd"; MPC_FUSED_CYCLIC=$cyc MPC_FUSED_DEPTH=$d MPC_FUSED_PF=1 MPC_FUSED_PFD=$pfd python scripts/bench_layers.py --model text --chain --reps 50 2>&1 | grep "chain of"
done; done; done
