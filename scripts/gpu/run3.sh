python -c "import __graft_entry__ as g; g.build()"
python scripts/profile_elementwise.py alg1 8 5 > gpurun_out/r2_alg1_times.txt 2>&1
python scripts/profile_elementwise.py alg1 4 5 >> gpurun_out/r2_alg1_times.txt 2>&1
python scripts/profile_elementwise.py share 2 10 >> gpurun_out/r2_alg1_times.txt 2>&1
python scripts/profile_elementwise.py share 8 10 >> gpurun_out/r2_alg1_times.txt 2>&1
ncu --set full --import-source on -k regex:trunc_alg1_all --launch-skip 1 --launch-count 1 -o gpurun_out/r2_alg1_p8_id -f python scripts/profile_elementwise.py alg1 8 1 > /dev/null 2>&1
ncu --set full --import-source on -k regex:share_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/r2_share_p2 -f python scripts/profile_elementwise.py share 2 1 > /dev/null 2>&1
cat gpurun_out/r2_alg1_times.txt
