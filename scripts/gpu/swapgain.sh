# chooser: transposed GEMM only when it promises >= 1/gain of the modelled tensor time; chains per gain
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for g in 1.0 0.5 0.45 1.0 0.5; do
  echo "== MPC_SWAP_GAIN=$g"
  for m in resnet50 resnet18 vit wav2letter text; do MPC_SWAP_GAIN=$g python scripts/bench_layers.py --model $m --chain 2>&1 | grep "chain of" | cut -c1-60; done
done > gpurun_out/swapgain.txt 2>&1
