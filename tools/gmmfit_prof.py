import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07630_b200 as sk
from workloads import gen
p = gen.c3()
ctx = sk.Context(0)
x = torch.from_numpy(p.x).cuda()
idx = gen.gmm_start_idx(p.n, 8, 3)
for it in (1, 10, 50):
    sk.sinkhorn_fit_gmm(ctx, x, 8, idx, iters=it)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sk.sinkhorn_fit_gmm(ctx, x, 8, idx, iters=it)
    torch.cuda.synchronize(); print("iters", it, "%.2f ms" % (1e3 * (time.perf_counter() - t0)))
