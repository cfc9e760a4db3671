python -c "import __graft_entry__ as g; g.build()"
for rep in 1 2; do
for d in 1 2; do for pf in 1 3; do
 echo "depth=$d pf=$pf"; MPC_FUSED_DEPTH=$d MPC_FUSED_PF=$pf python scripts/bench_layers.py --model text --chain --reps 50 2>&1 | grep "chain of"
done; done; done
MPC_FUSED_DEPTH=2 MPC_FUSED_PF=3 ncu --set full --clock-control none -k regex:fused_small -c 1 -o gpurun_out/ncu_fused_text_d2p3 python scripts/bench_layers.py --model text --chain --reps 2 > /dev/null 2>&1
