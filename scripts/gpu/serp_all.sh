# K-serpentine as the default for every 2-CTA launch: determinism + parity + chains + headline
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for m in resnet50 vit resnet18; do python scripts/bench_layers.py --model $m --chain 2>&1 | grep "chain of"; done > gpurun_out/serp_all.txt 2>&1
python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-next-rows --no-multi-party 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('headline', d['ms_per_step'], d['roofline']['gemm_ms_per_launch'], d['clocks']['sm_mhz'], d['check']['bit_exact_vs_oracle']['bit_exact'])" >> gpurun_out/serp_all.txt 2>&1
timeout 2000 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_conv.py tests/test_gpu_local_group.py -x -q -p no:cacheprovider > gpurun_out/serp_all_tests.txt 2>&1
tail -n 2 gpurun_out/serp_all_tests.txt
