# transposition factor for plain matmuls only (convolutions keep the plain model): conv chains, matmul chains, conv tests
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for m in resnet50 resnet18 wav2letter; do python scripts/bench_layers.py --model $m --chain 2>&1 | grep "chain of" | cut -c1-70; done > gpurun_out/sg4_chains.txt 2>&1
python scripts/bench_layers.py --model resnet50 --conv 2>&1 | grep -v "^{" >> gpurun_out/sg4_chains.txt
python scripts/bench_layers.py --model wav2letter --conv 2>&1 | grep -v "^{" >> gpurun_out/sg4_chains.txt
timeout 1200 python -m pytest tests/test_gpu_conv.py tests/test_gpu_determinism.py -x -q -p no:cacheprovider > gpurun_out/sg4_tests.txt 2>&1
tail -n 2 gpurun_out/sg4_tests.txt
