python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_fused_small.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for pf in 0 1 2; do
 echo "pf=$pf"; MPC_FUSED_PF=$pf python scripts/bench_layers.py --model text --chain --reps 50 2>&1 | grep "chain of"
done
MPC_FUSED_PF=1 ncu --set full --clock-control none -k regex:fused_small -c 1 -o gpurun_out/ncu_fused_text_v3 python scripts/bench_layers.py --model text --chain --reps 2 > /dev/null 2>&1
