"""A short d = 256 (or argv d) online solve at n = m = 65536 for ncu: K3 with KC = ceil(d/64) K chunks.
    python tools/wide_prof.py [d] [tc]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_07630_b200 as sk  # noqa: E402
from workloads import gen  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 256
tc = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n = 65536 if tc else 16384
p = gen.c5(n=n, d=d)
ctx = sk.Context(0)
ctx.set_tuning("tc", tc)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
f, g, rep = sk.sinkhorn_solve(ctx, x, y, p.eps, tol=1e-12, max_iter=4, mode="online")
torch.cuda.synchronize()
print(rep)
