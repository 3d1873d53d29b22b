"""C2: per-problem iteration counts (sort1d init) -> FIFO vs longest-first makespan on 296 slots."""
import os, sys, heapq
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2206_07630_b200 as sk
from workloads import gen
p = gen.c2()
ctx = sk.Context(0)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
f0 = sk.sinkhorn_init_sort1d(ctx, x.view(1024, 1024), y.view(1024), y_shared=True)
_, _, reps = sk.sinkhorn_solve(ctx, x, y, p.eps, y_shared=True, f_init=f0)
L = np.array([r["iterations"] for r in reps])
np.save("gpurun_out/c2_L.npy", L)
def makespan(order, slots=296):
    h = [0.0] * slots
    for i in order:
        t = heapq.heappop(h); heapq.heappush(h, t + 2 * L[i] + 1)
    return max(h)
ideal = (2 * L + 1).sum() / 296
print("L mean %.1f max %d; ideal %.1f fifo %.1f (eff %.3f) lpt %.1f (eff %.3f)" % (L.mean(), L.max(), ideal,
      makespan(range(1024)), ideal / makespan(range(1024)), makespan(np.argsort(-L)), ideal / makespan(np.argsort(-L))))
# proxy: the marginal error after one sweep (one batched sweep)
_, _, r1 = sk.sinkhorn_solve(ctx, x, y, p.eps, y_shared=True, f_init=f0, tol=1e-30, max_iter=1)
e1 = np.array([r["marginal_error"] for r in r1])
_, _, r2 = sk.sinkhorn_solve(ctx, x, y, p.eps, y_shared=True, f_init=f0, tol=1e-30, max_iter=3)
e3 = np.array([r["marginal_error"] for r in r2])
np.save("gpurun_out/c2_e1.npy", e1); np.save("gpurun_out/c2_e3.npy", e3)
for nm, e in (("err1", e1), ("err3", e3), ("rate", e3 / e1)):
    print(nm, "corr(log, L) %.3f" % np.corrcoef(np.log(e), L)[0, 1], "lpt-by-proxy eff %.3f" % (ideal / makespan(np.argsort(-np.log(e)))))
