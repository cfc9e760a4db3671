python -c "import __graft_entry__ as g; g.build()"
for d in 1 2; do for pf in 0 1; do
 echo "depth=$d pf=$pf"; MPC_FUSED_DEPTH=$d MPC_FUSED_PF=$pf python scripts/bench_layers.py --model text --chain --reps 50 2>&1 | grep "chain of"
done; done
MPC_FUSED_DEPTH=1 MPC_FUSED_PF=1 ncu --set full --clock-control none -k regex:fused_small -c 1 -o gpurun_out/ncu_fused_text_d1 python scripts/bench_layers.py --model text --chain --reps 2 > /dev/null 2>&1
