python -c "import __graft_entry__ as g; g.build()"
python scripts/e2e_breakdown.py > gpurun_out/r2_e2e_breakdown.json 2>&1
cat gpurun_out/r2_e2e_breakdown.json
