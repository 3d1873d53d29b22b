"""Time the GMM initializer (C3) and its kernels."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07630_b200 as sk
from workloads import gen
p = gen.c3(eps_factor=0.01)
ctx = sk.Context(0)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
gx = {k: torch.from_numpy(v).cuda() for k, v in p.extra["gmm_x"].items()}
gy = {k: torch.from_numpy(v).cuda() for k, v in p.extra["gmm_y"].items()}
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f0, _ = sk.sinkhorn_init_gmm(ctx, x, y, gx, gy, p.eps)
    torch.cuda.synchronize()
    print("gmm init ms", 1e3 * (time.perf_counter() - t0))
for mi in (10, 100, 1000, 3000, 10000, 100000):
    for tol in (1e-4, 1e-6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f0, _ = sk.sinkhorn_init_gmm(ctx, x, y, gx, gy, p.eps, inner_tol=tol, inner_max_iter=mi)
        torch.cuda.synchronize()
        print("max_iter", mi, "tol", tol, "ms %.3f" % (1e3 * (time.perf_counter() - t0)), float(f0[:3].sum()))
