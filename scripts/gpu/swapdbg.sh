# 49 x 4608 x 512 and 51 x 8000 x 2000: 2-CTA GEMM timelines transposed (MPC_SWAP_GAIN=100) vs not (MPC_GEMM_SMALL=0, MPC_NO_SWAP=1)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cat > /tmp/sd.py <<'PY'
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth, paper_2109_00984_b200 as m
c = m.Context(2, m.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
for (M, K, N) in [(49, 4608, 512), (51, 8000, 2000), (49, 512, 2048)]:
    dev = lambda a: torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
    x = c.share(dev(synth.uniform_fixed((M, K), 31)), 0, 1); y = c.share(dev(synth.uniform_fixed((K, N), 32)), 1, 2)
    a, b, cc = c.ttp_triples(4, M, K, N)
    for _ in range(3): z = c.beaver_matmul(x, y, a, b, cc, truncate=True)
    torch.cuda.synchronize()
PY
for env in "MPC_SWAP_GAIN=100" "MPC_GEMM_SMALL=0 MPC_NO_SWAP=1" "MPC_SWAP_GAIN=100 MPC_GEMM_TMA=0" "MPC_GEMM_SMALL=0 MPC_NO_SWAP=1 MPC_GEMM_TMA=0"; do
  echo "== $env"
  env $env MPC_GEMM_DEBUG=1 python /tmp/sd.py 2>&1 | grep ring_gemm | sed 's/per MMA thread//'
done > gpurun_out/swapdbg.txt 2>&1
