# chains with and without programmatic dependent launch, transposition factor 0.5 / 1.0
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for env in "X=1" "MPC_NO_PDL=1" "MPC_SWAP_GAIN=1.0 MPC_NO_PDL=1" "MPC_SWAP_GAIN=1.0"; do
  echo "== $env"
  for m in resnet50 resnet18 vit wav2letter; do env $env python scripts/bench_layers.py --model $m --chain 2>&1 | grep "chain of" | cut -c1-70; done
done > gpurun_out/pdl.txt 2>&1
