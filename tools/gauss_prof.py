"""The Gaussian initializer alone at a C5 / C3 shape (for ncu launch lists and timing).
    python tools/gauss_prof.py [c5|c3] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_07630_b200 as sk  # noqa: E402
from workloads import gen  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
p = {"c5": gen.c5, "c3": gen.c3}[w]()
ctx = sk.Context(0)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f0, side = sk.sinkhorn_init_gaussian(ctx, x, y)
    torch.cuda.synchronize()
    print("gaussian init %s %.3f ms" % (w, 1e3 * (time.perf_counter() - t0)), flush=True)
