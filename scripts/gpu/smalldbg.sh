# small-layer GEMM timelines (debug mode: no PDL, standalone launches) + chain timeline
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MPC_GEMM_DEBUG=1 python scripts/small_gemm_debug.py > gpurun_out/smalldbg.txt 2>&1
python scripts/chain_timeline.py --model resnet50 --offline --per-kernel --out gpurun_out/tl_resnet50_off.json > /dev/null 2> gpurun_out/tl.err
python scripts/chain_timeline.py --model resnet50 --per-kernel --out gpurun_out/tl_resnet50.json > /dev/null 2>> gpurun_out/tl.err
python scripts/bench_layers.py --model resnet50 --chain > gpurun_out/chain_r50.txt 2>&1
python scripts/bench_layers.py --model vit --chain >> gpurun_out/chain_r50.txt 2>&1
