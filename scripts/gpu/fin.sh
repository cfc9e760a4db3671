# split-K finalize: element pairs (16-byte accesses), 4 slabs' loads in flight; chains + timelines + parity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for m in resnet50 vit resnet18 wav2letter; do python scripts/bench_layers.py --model $m --chain; done > gpurun_out/chain_fin.txt 2>&1
python scripts/chain_timeline.py --model resnet50 --per-kernel --out gpurun_out/tl_resnet50_fin.json > /dev/null 2> gpurun_out/tl_fin.err
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_conv.py -x -q -p no:cacheprovider > gpurun_out/fin_tests.txt 2>&1
tail -n 2 gpurun_out/fin_tests.txt
