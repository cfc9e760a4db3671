# sustained headline at the final HEAD: 500 timed steps
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python bench.py --steps 500 --warmup 5 --no-next-rows --no-multi-party --no-cpu-baseline > gpurun_out/bench_steady.json 2> gpurun_out/bench_steady.err
