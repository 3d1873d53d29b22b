"""Host-side fixed cost of a sinkhorn_solve call (C2 shapes): wall time of calls whose device
work is tiny (max_iter = 1), split by the binding's pieces."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07630_b200 as sk
from workloads import gen
p = gen.c2()
ctx = sk.Context(0)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
B, n, m = p.batch, p.n, p.m
f0 = sk.sinkhorn_init_sort1d(ctx, x.view(B, n), y.view(m), y_shared=True)
def t(fn, k=20):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    ts.sort()
    return 1e3 * ts[len(ts) // 2]
print("solve B=1024 max_iter=1: %.3f ms" % t(lambda: sk.sinkhorn_solve(ctx, x, y, p.eps, y_shared=True, f_init=f0, max_iter=1, tol=1e-30)))
x8, f8 = x[:8].contiguous(), f0[:8].contiguous()
print("solve B=8 max_iter=1:    %.3f ms" % t(lambda: sk.sinkhorn_solve(ctx, x8, y, p.eps, y_shared=True, f_init=f8, max_iter=1, tol=1e-30)))
for park in (0, 12):
    ctx.set_tuning("batched_park", park)
    print("park %d solve B=1024 max_iter=1: %.3f ms" % (park, t(lambda: sk.sinkhorn_solve(ctx, x, y, p.eps, y_shared=True, f_init=f0, max_iter=1, tol=1e-30))))
print("sort1d init: %.3f ms" % t(lambda: sk.sinkhorn_init_sort1d(ctx, x.view(B, n), y.view(m), y_shared=True)))
print("empty torch sync: %.3f ms" % t(lambda: None))
