# tensor-map descriptors prefetched before griddepcontrol.wait (ring GEMM TMA producer, TMA split)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MPC_GEMM_DEBUG=1 python scripts/small_gemm_debug.py > gpurun_out/smalldbg5.txt 2>&1
for m in resnet50 vit resnet18; do python scripts/bench_layers.py --model $m --chain; done > gpurun_out/chain5.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/par5.txt 2>&1
tail -n 2 gpurun_out/par5.txt
python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-next-rows --no-multi-party > gpurun_out/bench5.json 2>/dev/null
