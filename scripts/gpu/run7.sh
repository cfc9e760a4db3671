python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2p
B="python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-next-rows --no-multi-party"
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r2p/ncu_launches.csv $B > gpurun_out/r2p/launches_bench.json 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:ring_gemm_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/r2p/gemm_4096 -f $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:split_both --launch-skip 2 --launch-count 1 -o gpurun_out/r2p/split_4096 -f $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:trunc_alg1_all --launch-skip 1 --launch-count 1 -o gpurun_out/r2p/alg1_p8_id -f python scripts/profile_elementwise.py alg1 8 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:share_all --launch-skip 1 --launch-count 1 -o gpurun_out/r2p/share_p2 -f python scripts/profile_elementwise.py share 2 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/r2p/gemm_c5_p4 -f python scripts/profile_c5.py 4 8192 2 > /dev/null 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_truncation.py tests/test_gpu_local_group.py -q -x -k "not xor_reveal" -p no:cacheprovider > gpurun_out/r2p/memcheck.log 2>&1
tail -5 gpurun_out/r2p/memcheck.log
ls -la gpurun_out/r2p
