"""The C4 subsample initializer alone (for ncu launch lists / timing): 4096 points per side,
inner solve to tol/10, Eq. (8) over all 262144 rows."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07630_b200 as sk
from workloads import gen
p = gen.c4()
ctx = sk.Context(0)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
ix, iy = torch.from_numpy(p.extra["idx_x"]).cuda(), torch.from_numpy(p.extra["idx_y"]).cuda()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f0, _, inner = sk.sinkhorn_init_subsample(ctx, x, y, ix, iy, p.eps, p.tol / 10)
    torch.cuda.synchronize()
    print("subsample init %.3f ms, inner %d sweeps, inner solve_ms %.3f" % (1e3 * (time.perf_counter() - t0),
                                                                           inner["iterations"], inner["solve_ms"]))
