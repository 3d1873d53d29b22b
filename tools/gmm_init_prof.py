"""C3 GMM-initializer breakdown: device fits of both mixtures, then sinkhorn_init_gmm (Bures
costs, the K x K solve, responsibilities, the n-point potential), each timed with CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07630_b200 as sk
from workloads import gen
p = gen.c3()
ctx = sk.Context(0)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
ix, iy = gen.gmm_start_idx(p.n, 8, 3), gen.gmm_start_idx(p.m, 8, 4)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for rep in range(3):
    ev[0].record()
    gx, _ = sk.sinkhorn_fit_gmm(ctx, x, 8, ix, iters=100, kmeans_iters=10, tol=1e-3)
    ev[1].record()
    gy, _ = sk.sinkhorn_fit_gmm(ctx, y, 8, iy, iters=100, kmeans_iters=10, tol=1e-3)
    ev[2].record()
    f0, side = sk.sinkhorn_init_gmm(ctx, x, y, gx, gy, p.eps)
    ev[3].record()
    torch.cuda.synchronize()
    print("fit x %.3f ms  fit y %.3f ms  init_gmm %.3f ms" % (ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]),
                                                            ev[2].elapsed_time(ev[3])))
