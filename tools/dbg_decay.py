import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, 'tests')
import numpy as np, torch
import paper_2206_07630_b200 as sk
from workloads import gen
from oracle import oracle as O
from parity import centred, rel_inf
ctx = sk.Context(0)
c2 = gen.c2(B=4, n=256)
xb, yb = torch.from_numpy(c2.x).cuda(), torch.from_numpy(c2.y).cuda()
pot = sk.sinkhorn_init_sort1d(ctx, xb.view(4, 256), yb.view(-1))
k = 2
f0 = pot[k].cpu().numpy()
for dec in [None, (5.0, 0.8)]:
    for L in [1, 4, 8, 9, 12, 20, 50, 100, 200]:
        f, g, reps = sk.sinkhorn_solve(ctx, xb, yb, c2.eps, y_shared=True, f_init=pot, tol=1e-12, max_iter=L, eps_decay=dec)
        lock = O.sinkhorn(c2.x[k], c2.y, c2.eps, tol=0, max_iter=L, f0=f0, eps_decay=dec)
        fc, gc = centred(f[k].cpu().numpy(), g[k].cpu().numpy()); foc, goc = centred(lock.f, lock.g)
        print(dec, L, reps[k]["iterations"], "f %.2e g %.2e" % (rel_inf(fc, foc, c2.eps), rel_inf(gc, goc, c2.eps)), "maxf %.3g" % np.abs(foc).max())
