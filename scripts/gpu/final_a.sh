# end-of-session evidence: GPU suite, smoke, bench line, launch list, ncu of Alg. 1 / ReLU / GEMM
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -c 300 gpurun_out/bench_final.json
M="sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.avg.per_cycle_active,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second"
ncu --metrics $M --clock-control none -k regex:trunc_alg1_all_w32 --launch-skip 1 --launch-count 1 --csv python scripts/profile_elementwise.py alg1 8 2 > gpurun_out/ncu_alg1_pipes.csv 2> gpurun_out/ncu_alg1.err
ncu --metrics $M --clock-control none -k regex:relu_all_kernel --launch-skip 1 --launch-count 1 --csv python scripts/profile_elementwise.py relu 2 2 > gpurun_out/ncu_relu_pipes.csv 2> gpurun_out/ncu_relu.err
ncu --set full --import-source on --clock-control none -k regex:trunc_alg1_all_w32 --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_alg1_p8_pf python scripts/profile_elementwise.py alg1 8 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-next-rows --no-multi-party > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_suite.log 2>&1
tail -3 gpurun_out/gpu_suite.log
