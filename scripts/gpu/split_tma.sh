python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_determinism.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for t in 1 0; do echo "tma=$t"; MPC_SPLIT_TMA=$t python scripts/bench_layers.py --chain --reps 50 2>&1 | grep "chain of" | cut -c1-60; MPC_SPLIT_TMA=$t python scripts/profile_c5.py 2 4096 50; done
ncu --set full --clock-control none -k regex:split2_tma --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_splittma_vitfc1 python scripts/profile_layer.py 197 768 3072 > /dev/null 2>&1
