"""Short C4 run for ncu: full-size online passes (2 sweeps, zero init)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_07630_b200 as sk  # noqa: E402
from workloads import gen  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c4"
p = {"c4": gen.c4, "c5": gen.c5, "c3": gen.c3}[w]()
ctx = sk.Context(0)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
mode = "stored" if w == "c3" else "online"
for _ in range(2):
    f, g, rep = sk.sinkhorn_solve(ctx, x, y, p.eps, tol=1e-9, max_iter=3, mode=mode)
torch.cuda.synchronize()
print(rep)
