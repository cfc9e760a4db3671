# split-K minimum item length 4 vs 8 blocks with the corrected chooser: chains
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for mk in 8 4 6 8 4; do
  echo "== MPC_GEMM_MINKB=$mk"
  for m in resnet50 resnet18 vit wav2letter; do MPC_GEMM_MINKB=$mk python scripts/bench_layers.py --model $m --chain 2>&1 | grep "chain of" | cut -c1-70; done
done > gpurun_out/minkb.txt 2>&1
