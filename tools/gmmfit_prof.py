"""Time the device GMM fit (K16) at C3 (16384 x 16, K = 8) for several EM iteration counts,
with and without the k-means start; under ncu it gives the per-kernel launch list."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07630_b200 as sk
from workloads import gen
p = gen.c3()
ctx = sk.Context(0)
x = torch.from_numpy(p.x).cuda()
idx = gen.gmm_start_idx(p.n, 8, 3)
quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
for km, it in ((0, 1), (0, 10), (0, 50), (10, 50)) if not quick else ((10, 3),):
    sk.sinkhorn_fit_gmm(ctx, x, 8, idx, iters=it, kmeans_iters=km)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sk.sinkhorn_fit_gmm(ctx, x, 8, idx, iters=it, kmeans_iters=km)
    torch.cuda.synchronize(); print("kmeans", km, "iters", it, "%.2f ms" % (1e3 * (time.perf_counter() - t0)))
