python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r2_prof10.txt
: > $O
for i in 1 2; do python scripts/profile_c5.py 2 4096 40 >> $O 2>&1; done
MPC_GEMM_TMA=0 python scripts/profile_c5.py 2 4096 40 >> $O 2>&1
MPC_GEMM_DEBUG=1 python scripts/profile_c5.py 2 4096 2 2>&1 | tail -1 >> $O
python scripts/profile_c5.py 4 8192 3 >> $O 2>&1
ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 python scripts/profile_c5.py 2 4096 2 2>&1 | grep -E "dram__|gpu__time|tensor" >> $O
timeout 1500 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_conv.py tests/test_gpu_local_group.py -x -q 2>&1 | tail -3 >> $O
cat $O
