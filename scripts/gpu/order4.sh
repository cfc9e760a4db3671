python -c "import __graft_entry__ as g; g.build()"
for v in "0 4" "1 4" "1 8" "1 2"; do set -- $v
echo "pm=$1 gm=$2"
MPC_GEMM_PARTY_MAJOR=$1 MPC_GEMM_GROUPM=$2 ncu --clock-control none --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 python scripts/profile_c5.py 2 4096 3 2>&1 | grep -E "dram__bytes_read|gpu__time"
MPC_GEMM_PARTY_MAJOR=$1 MPC_GEMM_GROUPM=$2 python scripts/profile_c5.py 2 4096 200
done
