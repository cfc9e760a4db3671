python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/memcheck_r2b.log
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_fused_small.py -m gpu -q -p no:cacheprovider -k "parity or carries" > $O 2>&1; echo "fused memcheck rc=$?" >> $O
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "share or beaver" > gpurun_out/memcheck_r2b_parity.log 2>&1; echo "parity memcheck rc=$?" >> $O
compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_fused_small.py -m gpu -q -p no:cacheprovider -k "parity and 17-4099" > gpurun_out/racecheck_r2b.log 2>&1; echo "fused racecheck rc=$?" >> $O
tail -3 gpurun_out/memcheck_r2b_parity.log >> $O
tail -3 gpurun_out/racecheck_r2b.log >> $O
cat $O | tail -20
