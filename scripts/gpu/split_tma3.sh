python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_local_group.py tests/test_gpu_conv.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
python scripts/bench_configs.py > gpurun_out/configs_r2c.json 2>/dev/null; python - <<'PY'
import json
d=json.loads(open('gpurun_out/configs_r2c.json').read().strip().splitlines()[-1])
for k in ('C3_resnet50','C4_vit_b16'):
    v=d[k]; print(k, v['chain_ms'], v['roofline_tensor_or_hbm_frac'], v.get('weights_prepared_offline',{}).get('chain_ms'), v.get('weights_prepared_offline',{}).get('roofline_tensor_or_hbm_frac'))
PY
