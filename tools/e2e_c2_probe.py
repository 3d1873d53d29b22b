"""Where the C2 end-to-end step (host buffers through the C ABI) spends its time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2206_07630_b200 as sk
from workloads import gen
p = gen.c2()
ctx = sk.Context(0)
xd, yd = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
xh, yh = torch.from_numpy(p.x).pin_memory(), torch.from_numpy(p.y).pin_memory()
B, n, m = p.batch, p.n, p.m
def t(fn, k=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts)
f0d = sk.sinkhorn_init_sort1d(ctx, xd.view(B, n), yd.view(m), y_shared=True)
f0h = f0d.cpu().pin_memory()
print("init dev  %.2f ms" % t(lambda: sk.sinkhorn_init_sort1d(ctx, xd.view(B, n), yd.view(m), y_shared=True)))
print("init host %.2f ms" % t(lambda: sk.sinkhorn_init_sort1d(ctx, xh.view(B, n), yh.view(m), y_shared=True)))
print("solve dev  %.2f ms" % t(lambda: sk.sinkhorn_solve(ctx, xd, yd, p.eps, y_shared=True, f_init=f0d)))
print("solve host %.2f ms" % t(lambda: sk.sinkhorn_solve(ctx, xh, yh, p.eps, y_shared=True, f_init=f0h)))
print("copy x h2d %.2f ms" % t(lambda: xh.cuda(non_blocking=True)))
fo = torch.empty(B * n, pin_memory=True)
print("copy f d2h %.2f ms" % t(lambda: fo.copy_(f0d.view(-1), non_blocking=True)))
