# small-layer GEMM phase timeline (debug mode, standalone launches): fill / issue / completion / epilogue
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MPC_GEMM_DEBUG=1 python scripts/small_gemm_debug.py > gpurun_out/smalldbg4.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "null_workspace" > gpurun_out/nullws.txt 2>&1
tail -n 2 gpurun_out/nullws.txt
