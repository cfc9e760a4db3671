python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests/test_gpu_parity.py::test_c2_4096_sampled_rows_and_identity tests/test_gpu_configs.py -x -q -s -k "c2_4096 or c5" 2>&1 | grep -v "^$" | tail -30 > gpurun_out/r2_full.log
cat gpurun_out/r2_full.log
