python -c "import __graft_entry__ as g; g.build()"
for o in 0 3; do for P in 3 4 8; do echo "occ=$o"; MPC_ALG1_OCC=$o python scripts/profile_elementwise.py alg1 $P 10; done; done
