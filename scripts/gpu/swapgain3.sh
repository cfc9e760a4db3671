# transposition factor 0.5 as the default: GPU suite, conv + parity under the plain model too, chains
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/sg3_suite.txt 2>&1
tail -n 2 gpurun_out/sg3_suite.txt
MPC_SWAP_GAIN=1.0 timeout 1200 python -m pytest tests/test_gpu_conv.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/sg3_plain.txt 2>&1
tail -n 2 gpurun_out/sg3_plain.txt
for m in resnet50 resnet18 vit wav2letter; do python scripts/bench_layers.py --model $m --chain 2>&1 | grep "chain of" | cut -c1-70; done > gpurun_out/sg3_chains.txt 2>&1
python scripts/bench_layers.py --model resnet50 --conv 2>&1 | grep -v "^{" >> gpurun_out/sg3_chains.txt
python scripts/bench_layers.py --model wav2letter --conv 2>&1 | grep -v "^{" >> gpurun_out/sg3_chains.txt
