python -c "import __graft_entry__ as g; g.build()"
MPC_GEMM_VERBOSE=1 timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/splitk_tests.log 2>&1
tail -3 gpurun_out/splitk_tests.log; grep "max active" gpurun_out/splitk_tests.log | head -2
for m in resnet50 vit; do
  python scripts/chain_timeline.py --model $m --per-kernel --out gpurun_out/tl3_$m.json > /dev/null 2>> gpurun_out/tl3.err
done
python scripts/bench_layers.py --chain --reps 50 > gpurun_out/chain3.txt 2>&1
MPC_GEMM_REDUCE=0 python scripts/bench_layers.py --chain --reps 50 > gpurun_out/chain3_fin.txt 2>&1
grep "chain of" gpurun_out/chain3.txt gpurun_out/chain3_fin.txt
