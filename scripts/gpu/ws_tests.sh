# null-workspace entry points, tensor-map prefetch, debug-mode producer: parity + determinism suites
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_local_group.py tests/test_gpu_fused_small.py -x -q -p no:cacheprovider > gpurun_out/ws_tests.txt 2>&1
tail -n 2 gpurun_out/ws_tests.txt
