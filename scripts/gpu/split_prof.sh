python -c "import __graft_entry__ as g; g.build()"
ncu --set full --clock-control none -k regex:split_both --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_split_vitfc1 python scripts/profile_layer.py 197 768 3072 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:split_both --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_split_r50l2c2 python scripts/profile_layer.py 784 1152 128 > /dev/null 2>&1
