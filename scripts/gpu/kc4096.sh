# 4096^3 unit length sweep with the serpentine walk: DRAM bytes per launch + 100-step bench
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for kc in 64 32 48 96 64 48; do
echo "KC=$kc"
MPC_GEMM_KC=$kc ncu --clock-control none --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 python scripts/profile_c5.py 2 4096 2 2>&1 | grep -E "dram__bytes|gpu__time"
MPC_GEMM_KC=$kc python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-next-rows --no-multi-party 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('headline', d['ms_per_step'], d['roofline']['gemm_ms_per_launch'], d['clocks']['sm_mhz'])"
done > gpurun_out/kc4096.txt 2>&1
