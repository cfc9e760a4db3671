# transposed vs not for the M = 49 ResNet-50 layers: per-layer GEMM share (eager, profiled) + debug timelines
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for env in "X=1" "MPC_NO_SWAP=1"; do
  echo "== $env"
  env $env python scripts/bench_layers.py --model resnet50 --reps 30 2>&1 | grep -E "l4|l3.c1b|l1.c2|l3.c3" 
  env $env MPC_GEMM_DEBUG=1 python - <<'PY' 2>&1 | grep ring_gemm
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth, paper_2109_00984_b200 as m
c = m.Context(2, m.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
for (M, K, N) in [(49, 4608, 512), (49, 512, 2048)]:
    dev = lambda a: torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
    x = c.share(dev(synth.uniform_fixed((M, K), 31)), 0, 1); y = c.share(dev(synth.uniform_fixed((K, N), 32)), 1, 2)
    a, b, cc = c.ttp_triples(4, M, K, N)
    for _ in range(2): z = c.beaver_matmul(x, y, a, b, cc, truncate=True)
    torch.cuda.synchronize()
PY
done > gpurun_out/swapprobe.txt 2>&1
