# K-serpentine tile walk for launches over 2 GiB of planes: DRAM bytes + time A/B (4- and 8-party 8192^3), determinism
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for P in 4 8; do for s in 0 1; do
echo "P=$P serpentine=$s"
MPC_GEMM_SERPENTINE=$s ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 python scripts/profile_c5.py $P 8192 2 2>&1 | grep -E "dram__bytes|gpu__time"
MPC_GEMM_SERPENTINE=$s python scripts/profile_c5.py $P 8192 4
done; done > gpurun_out/serp.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_determinism.py -x -q -p no:cacheprovider -k "SERPENTINE or default" > gpurun_out/serp_tests.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -p no:cacheprovider -k "8192" > gpurun_out/serp_c5.txt 2>&1
tail -2 gpurun_out/serp_tests.txt gpurun_out/serp_c5.txt
