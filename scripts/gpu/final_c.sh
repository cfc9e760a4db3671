# final HEAD check: smoke, full GPU suite, bench line, launch list
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_suite.log 2>&1
tail -n 2 gpurun_out/gpu_suite.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-next-rows --no-multi-party > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/ncu_gemm_4096_final python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-next-rows --no-multi-party > /dev/null 2>&1
