"""A/B of K3 variants on the C5 solve (Gaussian init, eps = 0.01 mean(C)), alternating runs.
    python tools/c5_epi_ab.py epi,emu[,pipe] ...   (default: 162,2 16,2)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07630_b200 as sk
from workloads import gen
p = gen.c5()
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
specs = sys.argv[1:] or ["162,2", "16,2"]
ctxs = {}
for spec in specs:
    v = [int(t) for t in spec.split(",")]
    c = sk.Context(0)
    c.set_tuning("tc_epi", v[0]); c.set_tuning("tc_emu", v[1])
    if len(v) > 2:
        c.set_tuning("tc_pipe", v[2])
    ctxs[spec] = c
f0, _ = sk.sinkhorn_init_gaussian(ctxs[specs[0]], x, y)
res = {s: [] for s in specs}
for rnd in range(int(os.environ.get("ROUNDS", "4"))):
    for s in specs:
        f, g, r = sk.sinkhorn_solve(ctxs[s], x, y, p.eps, mode="online", f_init=f0)
        res[s].append((r["solve_ms"], r["iterations"]))
for s in specs:
    print(s, "solve ms", [round(v[0], 2) for v in res[s]], "L", res[s][0][1])
