python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/splitk_tests.log 2>&1
tail -2 gpurun_out/splitk_tests.log
python scripts/chain_timeline.py --model resnet50 --per-kernel --out gpurun_out/tl4_resnet50.json > /dev/null 2>> gpurun_out/tl4.err
python scripts/bench_layers.py --chain --reps 50 > gpurun_out/chain4.txt 2>&1
MPC_GEMM_REDUCE=0 python scripts/bench_layers.py --chain --reps 50 > gpurun_out/chain4_fin.txt 2>&1
grep "chain of" gpurun_out/chain4.txt gpurun_out/chain4_fin.txt
