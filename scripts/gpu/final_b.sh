# end of round 2: sanitizers over this session's changes, GPU suite, smoke, bench line, launch list
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
O=gpurun_out/memcheck_r2c.log
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_truncation.py -m gpu -q -p no:cacheprovider -k "not contract_check" > gpurun_out/memcheck_r2c_trunc.log 2>&1; echo "truncation (Alg. 1 cp.async prefetch) memcheck rc=$?" > $O
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "null_workspace or beaver_matmul_parity or ttp" > gpurun_out/memcheck_r2c_parity.log 2>&1; echo "parity (null workspace, tensormap prefetch) memcheck rc=$?" >> $O
MPC_GEMM_SERPENTINE=1 MPC_GEMM_TMA=0 MPC_GEMM_SPLITS=7 MPC_GEMM_KC=5 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "beaver_matmul_parity_untruncated and 300-100-260" > gpurun_out/memcheck_r2c_serp.log 2>&1; echo "serpentine memcheck rc=$?" >> $O
compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_truncation.py -m gpu -q -p no:cacheprovider -k "all_parties" > gpurun_out/racecheck_r2c.log 2>&1; echo "truncation racecheck rc=$?" >> $O
for f in trunc parity serp; do tail -n 3 gpurun_out/memcheck_r2c_$f.log >> $O; done
tail -n 3 gpurun_out/racecheck_r2c.log >> $O
cat $O
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_suite.log 2>&1
tail -n 2 gpurun_out/gpu_suite.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-next-rows --no-multi-party > /dev/null 2>&1
