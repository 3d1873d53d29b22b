"""One sweep of the wide FFMA pass (tc = 0) against the tensor-core pass and the oracle (debug)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2206_07630_b200 as sk
from oracle import oracle as O
from workloads import gen
d, n, m = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
p = gen.c5(n=max(n, m), d=d, eps_factor=3e-2)
x, y = p.x[:n].copy(), p.y[:m].copy()
eps = float(np.float32(3e-2 * gen.mean_sq_cost(x, y)))
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
out = {}
for tc in (0, 1):
    c = sk.Context(0); c.set_tuning("tc", tc)
    f, g, r = sk.sinkhorn_solve(c, xd, yd, eps, mode="online", max_iter=1, tol=1e-12)
    out[tc] = (f.cpu().numpy().astype(np.float64), g.cpu().numpy().astype(np.float64))
    c.close()
ref = O.sinkhorn(x, y, eps, tol=0, max_iter=1)
for tc in (0, 1):
    f, g = out[tc]
    print(d, n, m, "tc", tc, "g err %.3e" % np.abs(g - ref.g).max(), "f err %.3e" % np.abs(f - ref.f).max(),
          "worst g col", int(np.argmax(np.abs(g - ref.g))), "worst f row", int(np.argmax(np.abs(f - ref.f))), flush=True)
