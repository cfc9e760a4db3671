python -c "import __graft_entry__ as g; g.build()"
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -c 200 gpurun_out/bench_final.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-next-rows --no-multi-party > /dev/null 2>&1
python scripts/bench_layers.py --chain --reps 50 > gpurun_out/chains_final.txt 2>&1
python scripts/bench_layers.py --chain --reps 50 --model resnet50 --conv > gpurun_out/chains_conv_final.txt 2>&1
