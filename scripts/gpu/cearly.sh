# c_p added after the item's first drain (MPC_GEMM_C_EARLY=1) vs at the tile end (0): timelines, chains, headline, parity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for ce in 1 0; do
  echo "C_EARLY=$ce"
  MPC_GEMM_C_EARLY=$ce MPC_GEMM_DEBUG=1 python scripts/small_gemm_debug.py 2>&1 | grep -A1 -- "--- " | grep ring_gemm | sed 's/.*M=\([0-9]*\) N=\([0-9]*\) kb=\([0-9]*\).*splits=\([0-9]*\).*timeline us: /\1x\2 kb\3 s\4: /'
  for m in resnet50 vit resnet18; do MPC_GEMM_C_EARLY=$ce python scripts/bench_layers.py --model $m --chain 2>&1 | grep "chain of"; done
  MPC_GEMM_C_EARLY=$ce python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-next-rows --no-multi-party 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('headline', d['ms_per_step'], d['roofline']['gemm_ms_per_launch'], d['clocks']['sm_mhz'])"
done > gpurun_out/cearly.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_conv.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > gpurun_out/cearly_tests.txt 2>&1
tail -n 2 gpurun_out/cearly_tests.txt
