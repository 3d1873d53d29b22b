"""Per-sweep cost of the on-chip solver with and without Anderson (C1 and a C2 batch):
solve_ms from the report at fixed sweep counts (tol unreachable)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2206_07630_b200 as sk
from workloads import gen

ctx = sk.Context(0)
p = gen.c1()
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
for mem in (0, 2, 5):
    out = []
    for L in (10, 40, 160):
        ts = []
        for _ in range(5):
            _, _, r = sk.sinkhorn_solve(ctx, x, y, p.eps, tol=1e-30, max_iter=L, anderson=mem)
            ts.append(r["solve_ms"])
        out.append((L, r["iterations"], min(ts)))
    print("c1 mem", mem, out, "us/sweep %.2f" % (1e3 * (out[2][2] - out[1][2]) / 120))
c2 = gen.c2(B=1024, n=1024)
xb, yb = torch.from_numpy(c2.x).cuda(), torch.from_numpy(c2.y).cuda()
for mem in (0, 5):
    ts = {}
    for L in (10, 30):
        _, _, r = sk.sinkhorn_solve(ctx, xb, yb, c2.eps, y_shared=True, tol=1e-30, max_iter=L, anderson=mem)
        _, _, r = sk.sinkhorn_solve(ctx, xb, yb, c2.eps, y_shared=True, tol=1e-30, max_iter=L, anderson=mem)
        ts[L] = r[0]["solve_ms"]
    print("c2 mem", mem, ts, "ms/sweep %.3f" % ((ts[30] - ts[10]) / 20))
