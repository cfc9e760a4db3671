python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_fused_small.py tests/test_gpu_configs.py -k "fused or text" -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for t in 1 0; do echo "tma=$t"; for r in 1 2; do MPC_FUSED_TMA=$t python scripts/bench_layers.py --model text --chain --reps 100 2>&1 | grep "chain of"; done; done
ncu --set full --clock-control none -k regex:fused_small -c 1 -o gpurun_out/ncu_fused_text_tma python scripts/bench_layers.py --model text --chain --reps 2 > /dev/null 2>&1
