python -c "import __graft_entry__ as g; g.build()"
for pf in 0 1 2; do
 echo "pf=$pf"; MPC_FUSED_PF=$pf python scripts/bench_layers.py --model text --chain --reps 50 2>&1 | grep "chain of"
done
MPC_FUSED_PF=1 ncu --set full --clock-control none -k regex:fused_small -c 1 -o gpurun_out/ncu_fused_text_pf1 python scripts/bench_layers.py --model text --chain --reps 2 > /dev/null 2>&1
MPC_FUSED_PF=2 ncu --set full --clock-control none -k regex:fused_small -c 1 -o gpurun_out/ncu_fused_text_pf2 python scripts/bench_layers.py --model text --chain --reps 2 > /dev/null 2>&1
