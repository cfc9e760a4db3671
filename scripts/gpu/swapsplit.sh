# split vs GEMM time per orientation without PDL (profile classes), small-M shapes
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cat > /tmp/ss.py <<'PY'
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth, paper_2109_00984_b200 as m
c = m.Context(2, m.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
for (M, K, N) in [(49, 4608, 512), (51, 8000, 2000), (49, 512, 2048), (50, 12000, 250)]:
    dev = lambda a: torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
    x = c.share(dev(synth.uniform_fixed((M, K), 31)), 0, 1); y = c.share(dev(synth.uniform_fixed((K, N), 32)), 1, 2)
    a, b, cc = c.ttp_triples(4, M, K, N)
    z = c.beaver_matmul(x, y, a, b, cc, truncate=True); torch.cuda.synchronize()
    c.profile_enable(True)
    for k in ("gemm", "split"): c.profile_read(k)
    for _ in range(10): z = c.beaver_matmul(x, y, a, b, cc, truncate=True)
    torch.cuda.synchronize()
    g, _ = c.profile_read("gemm"); s, _ = c.profile_read("split")
    c.profile_enable(False)
    print(f"{M}x{K}x{N}: split {s/10*1e3:.1f} us, gemm+finalize {g/10*1e3:.1f} us")
PY
for env in "MPC_SWAP_GAIN=100" "MPC_GEMM_SMALL=0 MPC_NO_SWAP=1" "X=1"; do
  echo "== $env"; env $env MPC_NO_PDL=1 python /tmp/ss.py
done > gpurun_out/swapsplit.txt 2>&1
