# debug-timeline atomics removed from the production kernels (they made ptxas spill 336 B in the bulk-copy variants)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for P in 4 8; do python scripts/profile_c5.py $P 8192 4; done > gpurun_out/nospill.txt 2>&1
MPC_GEMM_DEBUG=1 python scripts/small_gemm_debug.py 2>&1 | grep -c ring_gemm >> gpurun_out/nospill.txt
timeout 1500 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > gpurun_out/nospill_tests.txt 2>&1
tail -n 2 gpurun_out/nospill_tests.txt
