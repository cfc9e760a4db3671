python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -k share -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for P in 2 8; do python scripts/profile_elementwise.py share $P 20; done
ncu --set full --clock-control none -k regex:share_all --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_share_quad python scripts/profile_elementwise.py share 2 > /dev/null 2>&1
