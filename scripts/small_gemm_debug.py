import sys, numpy as np, torch
sys.path.insert(0, '.')
import synth, paper_2109_00984_b200 as m
c = m.Context(2, m.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
for (M,K,N) in [(3136,64,64),(197,768,768),(49,4608,512),(1,2048,1000),(12544,147,64)]:
    dev = lambda a: torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
    x = c.share(dev(synth.uniform_fixed((M, K), 31)), 0, 1)
    y = c.share(dev(synth.uniform_fixed((K, N), 32)), 1, 2)
    a, b, cc = c.ttp_triples(4, M, K, N)
    for _ in range(3):
        z = c.beaver_matmul(x, y, a, b, cc, truncate=True)
    torch.cuda.synchronize()
