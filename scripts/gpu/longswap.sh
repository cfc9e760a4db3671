# transposition factor only for short GEMMs (< 200k modelled cycles): chains + determinism + parity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do for m in resnet50 resnet18 vit wav2letter; do python scripts/bench_layers.py --model $m --chain 2>&1 | grep "chain of" | cut -c1-70; done; done > gpurun_out/longswap.txt 2>&1
python scripts/bench_layers.py --model wav2letter --conv 2>&1 | grep "b1 \|b32" | cut -c1-90 >> gpurun_out/longswap.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_conv.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > gpurun_out/longswap_tests.txt 2>&1
tail -n 2 gpurun_out/longswap_tests.txt
