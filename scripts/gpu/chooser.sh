# per-layer times (CUDA graph) under the GEMM-choice knobs: default, no transposition, stacked kernel forced, split-K granularity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for env in "X=1" "MPC_NO_SWAP=1" "MPC_GEMM_SMALL=1" "MPC_GEMM_MINKB=4" "MPC_GEMM_MINKB=16"; do
  echo "== $env"
  env $env python scripts/bench_layers.py --model resnet50 --graph --reps 50 2>&1 | grep -v "^{" | head -30
done > gpurun_out/chooser.txt 2>&1
