# Alg. 1 with the next iteration's x pairs prefetched into shared memory (cp.async): A/B + parity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for pf in 1 0; do for P in 3 4 8 16; do echo "prefetch=$pf"; MPC_ALG1_PREFETCH=$pf python scripts/profile_elementwise.py alg1 $P 10; done; done > gpurun_out/alg1pf.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_truncation.py tests/test_gpu_local_group.py -x -q -p no:cacheprovider > gpurun_out/alg1pf_tests.txt 2>&1
tail -3 gpurun_out/alg1pf_tests.txt
