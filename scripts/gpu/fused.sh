python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_fused_small.py tests/test_gpu_configs.py -k "fused or text" -m gpu -x -q -p no:cacheprovider > gpurun_out/fused_tests.log 2>&1
tail -15 gpurun_out/fused_tests.log
python scripts/bench_layers.py --model text --chain --reps 50 2>&1 | grep "chain of"
MPC_FUSED_SMALL=0 python scripts/bench_layers.py --model text --chain --reps 50 2>&1 | grep "chain of"
python scripts/chain_timeline.py --model text --per-kernel --out gpurun_out/tl_text_fused.json > /dev/null 2>&1
ncu --set full --clock-control none -k regex:fused_small -c 1 -o gpurun_out/ncu_fused_text python scripts/bench_layers.py --model text --chain --reps 2 > /dev/null 2>&1
ncu -i gpurun_out/ncu_fused_text.ncu-rep --page details --csv > gpurun_out/ncu_fused_text_details.csv 2>&1
