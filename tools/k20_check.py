"""K20 vs the multi-kernel inner solve on a slowly contracting problem run to tol (1431 sweeps):
both against the oracle's lockstep (how far fp32 drifts, per path).
    python tools/k20_check.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_07630_b200 as sk  # noqa: E402
from oracle import oracle as O  # noqa: E402
from parity import centred, rel_inf  # noqa: E402
from workloads import gen  # noqa: E402

n, m, d, ns, ms, eps_f = 6000, 6000, 2, 700, 800, 0.003
rng = np.random.default_rng(n + d)
x = rng.random((n, d)).astype(np.float32)
y = (rng.random((m, d)) * 0.9 + 0.05).astype(np.float32)
ix = np.sort(rng.choice(n, ns, replace=False)).astype(np.int32)
iy = np.sort(rng.choice(m, ms, replace=False)).astype(np.int32)
eps = float(np.float32(eps_f * gen.mean_sq_cost(x, y)))
ctx = sk.Context(0)
w, z = x[ix], y[iy]
c = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
for gs in (1, 0):
    ctx.set_tuning("grid_solver", gs)
    for cap in (60, 300, 0):
        tol, mi = (1e-12, cap) if cap else (1e-4, 10000)
        pot, _, inner = sk.sinkhorn_init_subsample(ctx, c(x), c(y), c(ix), c(iy), eps, tol, inner_max_iter=mi)
        lock = O.sinkhorn(w, z, eps, tol=0, max_iter=inner["iterations"])
        ex = O.subsample_extrapolate(x, z, lock.g, eps)
        print(json.dumps({"grid_solver": gs, "L": inner["iterations"], "pot_rel_inf": rel_inf(centred(pot.cpu().numpy()), centred(ex), eps),
                          "E": inner["dual_objective"], "E_oracle": lock.E}), flush=True)
