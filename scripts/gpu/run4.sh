python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r2_prof4.txt
: > $O
python scripts/profile_elementwise.py alg1 8 5 >> $O 2>&1
python scripts/profile_elementwise.py alg1 4 5 >> $O 2>&1
MPC_ALG1_INT128=1 python scripts/profile_elementwise.py alg1 8 5 >> $O 2>&1
python scripts/profile_elementwise.py share 2 10 >> $O 2>&1
python scripts/profile_elementwise.py share 8 10 >> $O 2>&1
for kc in 64 32; do for gm in 4 2 8; do
  MPC_GEMM_KC=$kc MPC_GEMM_GROUPM=$gm python scripts/profile_c5.py 4 8192 4 >> $O 2>&1
  MPC_GEMM_KC=$kc MPC_GEMM_GROUPM=$gm ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 python scripts/profile_c5.py 4 8192 2 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/kc=$kc gm=$gm /" >> $O
done; done
ncu --set full --import-source on --clock-control none -k regex:trunc_alg1_all --launch-skip 1 --launch-count 1 -o gpurun_out/r2_alg1_p8_w32 -f python scripts/profile_elementwise.py alg1 8 1 > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "truncat or share or parity or alg1 or local_group" 2>&1 | tail -3 >> $O
cat $O
