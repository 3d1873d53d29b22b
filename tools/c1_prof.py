"""C1 (256 x 256, d = 2): the Gaussian initializer and the on-chip solve, for an ncu launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07630_b200 as sk
from workloads import gen
p = gen.c1()
ctx = sk.Context(0)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
for _ in range(3):
    f0, _ = sk.sinkhorn_init_gaussian(ctx, x, y)
    sk.sinkhorn_solve(ctx, x, y, p.eps, f_init=f0)
torch.cuda.synchronize()
