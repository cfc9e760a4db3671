python -c "import __graft_entry__ as g; g.build()"
for c in 1 0; do echo "cpf=$c"; MPC_GEMM_C_PREFETCH=$c python scripts/bench_layers.py --chain --reps 50 2>&1 | grep "chain of" | cut -c1-60; MPC_GEMM_C_PREFETCH=$c python scripts/profile_c5.py 2 4096 100; done
