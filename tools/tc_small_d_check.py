"""Accuracy of the tensor-core cross term (K3) at small d (sk_set_tuning tc_min_d): C4-recipe
problems solved on K3 vs the fp64 oracle - lockstep rel-inf of the centred potentials and E, at
reduced n and on sampled columns of the full-size first sweep."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import paper_2206_07630_b200 as sk
from oracle import oracle as O
from parity import centred, rel_inf
from workloads import gen

for tmd in (17, 1):
    ctx = sk.Context(0)
    ctx.set_tuning("tc_min_d", tmd)
    p = gen.c4(n=6000, ns=600)
    x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
    f, g, rep = sk.sinkhorn_solve(ctx, x, y, p.eps, mode="online")
    ref = O.sinkhorn(p.x, p.y, p.eps)
    lock = O.sinkhorn(p.x, p.y, p.eps, tol=0, max_iter=rep["iterations"])
    fc, gc = centred(f.cpu().numpy(), g.cpu().numpy())
    fo, go = centred(lock.f, lock.g)
    print(f"tc_min_d {tmd}: n=6000 L {rep['iterations']} (oracle {ref.iterations}) f {rel_inf(fc, fo, p.eps):.2e} "
          f"g {rel_inf(gc, go, p.eps):.2e} E {abs(rep['dual_objective'] - lock.E) / max(abs(lock.E), p.eps):.2e}", flush=True)
    p = gen.c4()
    x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
    f, g, rep = sk.sinkhorn_solve(ctx, x, y, p.eps, tol=1e-9, max_iter=3, mode="online")
    cols = np.sort(np.random.default_rng(0).choice(p.m, 64, replace=False))
    f3 = O.sinkhorn(p.x[:1], p.y[:1], p.eps, tol=0, max_iter=1)   # (warm the oracle)
    g_ref = O.g_update(p.x, p.y, f.cpu().numpy().astype(np.float64), p.eps, cols=cols)
    # g^3 from the GPU's f^2?  Instead: one more column pass of the GPU's f^3 by the oracle vs the GPU's
    # next g: compare the g-update the oracle computes from the GPU's f with the GPU's g of a 4th sweep
    f4, g4, rep4 = sk.sinkhorn_solve(ctx, x, y, p.eps, tol=1e-9, max_iter=4, mode="online")
    g_ref = O.g_update(p.x, p.y, f.cpu().numpy().astype(np.float64), p.eps, cols=cols)
    err = np.abs(g4.cpu().numpy()[cols] - g_ref).max() / max(np.abs(g_ref).max(), p.eps)
    print(f"tc_min_d {tmd}: full-size C4 g^4 = g_sk(f^3) on 64 sampled columns rel {err:.2e}", flush=True)
    ctx.close()
