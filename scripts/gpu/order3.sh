python -c "import __graft_entry__ as g; g.build()"
for v in "1 8" "0 4"; do set -- $v
echo "pm=$1 gm=$2"
MPC_GEMM_PARTY_MAJOR=$1 MPC_GEMM_GROUPM=$2 ncu --clock-control none --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 python scripts/profile_c5.py 8 8192 3 2>&1 | grep -E "dram__bytes_read|gpu__time"
MPC_GEMM_PARTY_MAJOR=$1 MPC_GEMM_GROUPM=$2 ncu --clock-control none --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 python scripts/profile_c5.py 4 8192 3 2>&1 | grep -E "dram__bytes_read|gpu__time"
done
