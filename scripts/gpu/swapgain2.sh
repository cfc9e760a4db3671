# per-layer (graph) times of Wav2Letter and ResNet-18 under the transposition gain 1.0 / 0.5
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for g in 1.0 0.5; do
  echo "== MPC_SWAP_GAIN=$g"
  for m in wav2letter resnet18; do MPC_SWAP_GAIN=$g python scripts/bench_layers.py --model $m --graph --reps 50 2>&1 | grep -v "^{"; done
done > gpurun_out/swapgain2.txt 2>&1
