python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r2_prof5.txt
: > $O
python scripts/profile_elementwise.py alg1 8 5 >> $O 2>&1
python scripts/profile_elementwise.py alg1 4 5 >> $O 2>&1
for kc in 64 32 24 16; do
  MPC_GEMM_KC=$kc python scripts/profile_c5.py 2 4096 30 >> $O 2>&1
done
for kc in 24 16; do
  MPC_GEMM_KC=$kc python scripts/profile_c5.py 4 8192 4 >> $O 2>&1
  MPC_GEMM_KC=$kc ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 python scripts/profile_c5.py 4 8192 2 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/P4 kc=$kc /" >> $O
done
for kc in 64 32; do
  MPC_GEMM_KC=$kc ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 python scripts/profile_c5.py 2 4096 2 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/P2-4096 kc=$kc /" >> $O
done
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_conv.py tests/test_gpu_determinism.py tests/test_gpu_parity.py -x -q -k "not c5 and not c2_4096" 2>&1 | tail -3 >> $O
for f in 1 0; do
  MPC_GEMM_FUSED_SPLITK=$f python scripts/bench_layers.py --model resnet50 --chain 2>&1 | grep chain | sed "s/^/fused=$f /" >> $O
  MPC_GEMM_FUSED_SPLITK=$f python scripts/bench_layers.py --model vit --chain 2>&1 | grep chain | sed "s/^/fused=$f /" >> $O
done
python scripts/bench_layers.py --model wav2letter --conv 2>&1 | grep wav2letter >> $O
cat $O
