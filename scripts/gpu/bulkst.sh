# bulk-copy store of each CTA's last tile: small-layer timelines, chains, GEMM parity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MPC_GEMM_DEBUG=1 python scripts/small_gemm_debug.py > gpurun_out/smalldbg3.txt 2>&1
python scripts/bench_layers.py --model resnet50 --chain > gpurun_out/chain3.txt 2>&1
python scripts/bench_layers.py --model vit --chain >> gpurun_out/chain3.txt 2>&1
python scripts/bench_layers.py --model resnet18 --chain >> gpurun_out/chain3.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_conv.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > gpurun_out/par3.txt 2>&1
tail -3 gpurun_out/par3.txt
python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-next-rows --no-multi-party > gpurun_out/bench3.json 2>/dev/null
