python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/order.txt; : > $O
for pm in 0 1; do for gm in 4 8; do
  echo "pm=$pm gm=$gm" >> $O
  MPC_GEMM_PARTY_MAJOR=$pm MPC_GEMM_GROUPM=$gm python scripts/profile_c5.py 4 8192 6 >> $O 2>&1
  MPC_GEMM_PARTY_MAJOR=$pm MPC_GEMM_GROUPM=$gm ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 python scripts/profile_c5.py 4 8192 3 2>&1 | grep -E "dram__bytes_read|gpu__time" >> $O
  MPC_GEMM_PARTY_MAJOR=$pm MPC_GEMM_GROUPM=$gm python scripts/profile_c5.py 2 4096 40 >> $O 2>&1
done; done
cat $O
