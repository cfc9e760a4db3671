python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r2_prof9.txt
: > $O
python scripts/probe_pcie.py >> $O 2>&1
for gm in 1 2 4 8; do for kc in 32 48 64; do
  MPC_GEMM_GROUPM=$gm MPC_GEMM_KC=$kc python scripts/profile_c5.py 2 4096 40 >> $O 2>&1
done; done
cat $O
