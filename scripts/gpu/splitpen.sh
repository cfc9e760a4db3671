# GEMM chooser with a split-K cost term (MPC_SPLIT_PENALTY cycles): chains and per-layer, A/B with 0
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for pen in 12000 0 12000 0; do
  echo "== MPC_SPLIT_PENALTY=$pen"
  for m in resnet50 resnet18 vit wav2letter; do MPC_SPLIT_PENALTY=$pen python scripts/bench_layers.py --model $m --chain 2>&1 | grep "chain of" | cut -c1-70; done
  MPC_SPLIT_PENALTY=$pen python scripts/bench_layers.py --model resnet50 --conv 2>&1 | grep "true convs" | cut -c1-90
  MPC_SPLIT_PENALTY=$pen python scripts/bench_layers.py --model wav2letter --conv 2>&1 | grep "b1 " | cut -c1-90
  MPC_SPLIT_PENALTY=$pen python scripts/bench_layers.py --model vit --chain --prepared 2>&1 | grep "chain of" | cut -c1-70
done > gpurun_out/splitpen.txt 2>&1
MPC_SPLIT_PENALTY=12000 python scripts/bench_layers.py --model resnet50 --graph --reps 50 2>&1 | grep -v "^{" >> gpurun_out/splitpen.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_conv.py tests/test_gpu_determinism.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > gpurun_out/splitpen_tests.txt 2>&1
tail -n 2 gpurun_out/splitpen_tests.txt
