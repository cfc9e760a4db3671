# small-layer GEMM phase timeline with the production producer (TMA) in debug mode
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MPC_GEMM_DEBUG=1 python scripts/small_gemm_debug.py > gpurun_out/smalldbg6.txt 2>&1
MPC_GEMM_DEBUG=1 MPC_GEMM_TMA=0 python scripts/small_gemm_debug.py > gpurun_out/smalldbg6_bulk.txt 2>&1
