python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_conv.py tests/test_gpu_local_group.py -m gpu -x -q -p no:cacheprovider > gpurun_out/splitk_tests.log 2>&1
tail -3 gpurun_out/splitk_tests.log
for m in resnet50 vit; do
  python scripts/chain_timeline.py --model $m --per-kernel --out gpurun_out/tl2_$m.json > /dev/null 2>> gpurun_out/tl2.err
  MPC_GEMM_REDUCE=0 python scripts/chain_timeline.py --model $m --per-kernel --out gpurun_out/tl2_${m}_fin.json > /dev/null 2>> gpurun_out/tl2.err
done
python scripts/bench_layers.py --chain --reps 50 > gpurun_out/chain2.txt 2>&1
MPC_GEMM_REDUCE=0 python scripts/bench_layers.py --chain --reps 50 > gpurun_out/chain2_fin.txt 2>&1
grep chain gpurun_out/chain2.txt gpurun_out/chain2_fin.txt
