python -c "import __graft_entry__ as g; g.build()"
for m in resnet50 vit text; do
  python scripts/chain_timeline.py --model $m --per-kernel --out gpurun_out/tl_$m.json > /dev/null 2> gpurun_out/tl_$m.err
  python scripts/chain_timeline.py --model $m --offline --per-kernel --out gpurun_out/tl_${m}_off.json > /dev/null 2>> gpurun_out/tl_$m.err
done
ls -la gpurun_out
