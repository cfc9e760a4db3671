python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r2_prof8.txt
: > $O
timeout 1200 python -m pytest tests/test_gpu_boundary_swap.py tests/test_gpu_parity.py tests/test_gpu_local_group.py tests/test_gpu_conv.py tests/test_gpu_elementwise.py tests/test_gpu_relu.py tests/test_gpu_truncation.py -x -q 2>&1 | tail -3 >> $O
MPC_GEMM_DEBUG=1 python scripts/profile_c5.py 2 4096 3 >> $O 2>&1
MPC_GEMM_DEBUG=1 python scripts/profile_c5.py 1 4096 3 >> $O 2>&1
MPC_GEMM_TMA=0 python scripts/profile_c5.py 2 4096 30 >> $O 2>&1
MPC_GEMM_TMA=1 python scripts/profile_c5.py 2 4096 30 >> $O 2>&1
cat $O
