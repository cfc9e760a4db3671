python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
python scripts/profile_c5.py 4 8192 6
python scripts/profile_c5.py 8 8192 3
MPC_GEMM_PARTY_MAJOR=0 MPC_GEMM_GROUPM=4 python scripts/profile_c5.py 8 8192 3
ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 python scripts/profile_c5.py 8 8192 3 2>&1 | grep -E "dram__bytes_read|gpu__time"
