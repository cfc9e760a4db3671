python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_conv.py tests/test_gpu_configs.py tests/test_gpu_determinism.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for s2 in 1 0; do echo "split2=$s2"; MPC_SPLIT2=$s2 python scripts/bench_layers.py --chain --reps 50 2>&1 | grep "chain of" | cut -c1-60; done
MPC_SPLIT2=1 python scripts/chain_timeline.py --model vit --out gpurun_out/tl_vit_s2.json > /dev/null 2>&1
MPC_SPLIT2=1 python scripts/chain_timeline.py --model resnet50 --out gpurun_out/tl_r50_s2.json > /dev/null 2>&1
