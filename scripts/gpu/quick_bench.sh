python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python bench.py --steps 20 --warmup 3 --no-next-rows --no-multi-party --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
