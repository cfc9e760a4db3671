# Alg. 1 prefetching kernel at 3 blocks per SM (P <= 8, 80 registers) vs the committed 2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for P in 3 4 8; do python scripts/profile_elementwise.py alg1 $P 10; done > gpurun_out/alg1occ3.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_truncation.py -x -q -p no:cacheprovider > gpurun_out/alg1occ3_tests.txt 2>&1
tail -n 2 gpurun_out/alg1occ3_tests.txt
