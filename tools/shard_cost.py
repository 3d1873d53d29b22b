"""Per-sweep cost of the row-sharded algorithm on one GPU: the unsharded solve
vs sinkhorn_solve_sharded_emulated(W) on C4 (or C5), zero init, a fixed number of sweeps.
Emulated W runs the W rank slices one after another on this GPU, so its per-sweep time is the
1-GPU cost of the W-rank launch configuration (the 8-rank per-GPU time is about 1/W of it).

    python tools/shard_cost.py [c4|c5] [sweeps]
"""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_07630_b200 as sk  # noqa: E402
from workloads import gen  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c4"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 12
p = gen.c4() if wl == "c4" else gen.c5()
ctx = sk.Context(0)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
out = {"workload": wl, "sweeps": L}


def run(tag, fn):
    fn()  # warm-up (allocations)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f, g, rep = fn()
    e1.record()
    torch.cuda.synchronize()
    out[tag] = {"ms_per_sweep": e0.elapsed_time(e1) / rep["iterations"], "iterations": rep["iterations"],
                "solve_ms": rep["solve_ms"]}
    return f, g


fu, gu = run("unsharded", lambda: sk.sinkhorn_solve(ctx, x, y, p.eps, tol=1e-12, max_iter=L, mode="online"))
for W in (1, 2, 8):
    f, g = run(f"emulated_w{W}", lambda: sk.sinkhorn_solve_sharded_emulated(ctx, W, x, y, p.eps, tol=1e-12,
                                                                             max_iter=L, mode="online"))
    out[f"emulated_w{W}"]["bit_identical_to_unsharded"] = bool(torch.equal(f, fu) and torch.equal(g, gu))
u = out["unsharded"]["ms_per_sweep"]
for W in (1, 2, 8):
    out[f"emulated_w{W}"]["ratio_to_unsharded"] = out[f"emulated_w{W}"]["ms_per_sweep"] / u
print(json.dumps(out))
