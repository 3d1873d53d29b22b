import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch
import paper_2206_07630_b200 as sk
from workloads import gen
from oracle import oracle as O
ctx = sk.Context(0)
n,m,d = 6000,2100,40
rng = np.random.default_rng(n + d)
x = rng.random((n, d)).astype(np.float32); y = rng.random((m, d)).astype(np.float32)
a = gen.random_weights(n, rng)
eps = float(np.float32(0.04 * gen.mean_sq_cost(x, y)))
c = lambda v: torch.from_numpy(v).cuda()
outs = {W: sk.sinkhorn_solve_sharded_emulated(ctx, W, c(x), c(y), eps, a=c(a), mode="online") for W in (1,2)}
f1,g1,r1 = outs[1]; f2,g2,r2 = outs[2]
print("W1 vs W2 equal:", torch.equal(f1,f2), torch.equal(g1,g2), r1["iterations"], r2["iterations"], (f1-f2).abs().max().item())
fu,gu,ru = sk.sinkhorn_solve(ctx, c(x), c(y), eps, a=c(a), mode="online")
print("unsharded its", ru["iterations"], "sharded", r1["iterations"])
def rel(u, v):
    u = u - u.mean(); v = v - v.mean(); return np.abs(u-v).max()/max(np.abs(v).max(), eps)
print("unsharded vs sharded f rel", rel(fu.cpu().numpy().astype(np.float64), f1.cpu().numpy().astype(np.float64)))
L = r1["iterations"]
lock = O.sinkhorn(x, y, eps, a=a, tol=0, max_iter=L)
print("sharded vs oracle", rel(f1.cpu().numpy().astype(np.float64), lock.f), rel(g1.cpu().numpy().astype(np.float64), lock.g))
lock2 = O.sinkhorn(x, y, eps, a=a, tol=0, max_iter=ru["iterations"])
print("unsharded vs oracle", rel(fu.cpu().numpy().astype(np.float64), lock2.f), rel(gu.cpu().numpy().astype(np.float64), lock2.g))
