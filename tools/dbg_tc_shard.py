"""Where do the tensor-core (K3) sharded solves stop being bit-identical across W?  Runs the
emulated sharded solver for W = 1, 2, 8 for 1..S sweeps on a C5-shaped problem and prints the
first sweep whose f or g differ (and by how much).

    python tools/dbg_tc_shard.py [n] [d] [sweeps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_07630_b200 as sk  # noqa: E402
from workloads import gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
S = int(sys.argv[3]) if len(sys.argv) > 3 else 5
p = gen.c5(n=n, d=d)
ctx = sk.Context(0)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
out = []
for seeded in (1, 0):
    ctx.set_tuning("seeded", seeded)
    for L in range(1, S + 1):
        res = {}
        for W in (1, 2, 8):
            f, g, r = sk.sinkhorn_solve_sharded_emulated(ctx, W, x, y, p.eps, tol=1e-12, max_iter=L, mode="online")
            res[W] = (f.clone(), g.clone())
        row = {"seeded": seeded, "L": L}
        for W in (2, 8):
            row[f"f_eq_w{W}"] = bool(torch.equal(res[W][0], res[1][0]))
            row[f"g_eq_w{W}"] = bool(torch.equal(res[W][1], res[1][1]))
            row[f"f_maxdiff_w{W}"] = float((res[W][0] - res[1][0]).abs().max())
            row[f"g_maxdiff_w{W}"] = float((res[W][1] - res[1][1]).abs().max())
            if not row[f"g_eq_w{W}"]:
                idx = torch.nonzero(res[W][1] != res[1][1]).flatten()
                row[f"g_ndiff_w{W}"] = int(idx.numel())
                row[f"g_first_w{W}"] = idx[:8].tolist()
            if not row[f"f_eq_w{W}"]:
                idx = torch.nonzero(res[W][0] != res[1][0]).flatten()
                row[f"f_ndiff_w{W}"] = int(idx.numel())
                row[f"f_first_w{W}"] = idx[:8].tolist()
        out.append(row)
        print(json.dumps(row), flush=True)
