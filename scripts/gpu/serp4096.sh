# K-serpentine on the TMA-fed kernel at 4096^3 (MPC_GEMM_SERPENTINE=1 forces it): DRAM bytes + headline A/B
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for s in 0 1 0 1; do
echo "serpentine=$s"
MPC_GEMM_SERPENTINE=$s ncu --clock-control none --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 python scripts/profile_c5.py 2 4096 2 2>&1 | grep -E "dram__bytes|gpu__time"
MPC_GEMM_SERPENTINE=$s python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-next-rows --no-multi-party 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('headline', d['ms_per_step'], d['roofline']['gemm_ms_per_launch'], d['clocks']['sm_mhz'])"
done > gpurun_out/serp4096.txt 2>&1
MPC_GEMM_SERPENTINE=1 timeout 900 python -m pytest tests/test_gpu_determinism.py -x -q -p no:cacheprovider -k "default or TMA=1" > gpurun_out/serp4096_tests.txt 2>&1
tail -n 2 gpurun_out/serp4096_tests.txt
