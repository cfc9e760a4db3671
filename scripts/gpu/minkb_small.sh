# split-K items of 4 blocks allowed only for reductions under 16 blocks: chains A/B (MPC_GEMM_MINKB=8 = before)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for env in "X=1" "MPC_GEMM_MINKB=8" "X=1" "MPC_GEMM_MINKB=8"; do
  echo "== $env"
  for m in resnet50 resnet18 vit wav2letter; do env $env python scripts/bench_layers.py --model $m --chain 2>&1 | grep "chain of" | cut -c1-70; done
done > gpurun_out/minkb_small.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_conv.py -x -q -p no:cacheprovider > gpurun_out/minkb_small_tests.txt 2>&1
tail -n 2 gpurun_out/minkb_small_tests.txt
