"""C2 schedule study for K13's queue tail: per-problem sweep counts L and the errors err_{K-2},
err_{K-1} after K-2 / K-1 sweeps (sort1d init), then the makespan on 296 slots of
  FIFO (today's dynamic queue), LPT with the true L, and the two-phase park/resume schedule:
  phase 1 = K sweeps per problem in queue order (or to convergence), phase 2 = the parked
  problems in decreasing predicted remaining sweeps log(err_{K-1}/tol) / log(err_{K-2}/err_{K-1}).
    python tools/c2_park_sim.py
"""
import heapq
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_07630_b200 as sk  # noqa: E402
from workloads import gen  # noqa: E402

p = gen.c2()
ctx = sk.Context(0)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
f0 = sk.sinkhorn_init_sort1d(ctx, x.view(1024, 1024), y.view(1024), y_shared=True)
_, _, reps = sk.sinkhorn_solve(ctx, x, y, p.eps, y_shared=True, f_init=f0)
L = np.array([r["iterations"] for r in reps])
errs = {}
for k in range(1, 53):
    _, _, rk = sk.sinkhorn_solve(ctx, x, y, p.eps, y_shared=True, f_init=f0, tol=1e-30, max_iter=k)
    errs[k] = np.array([r["marginal_error"] for r in rk])
SLOTS = 296
cost = 2 * L + 1
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/c2_park_trace.npz", L=L, **{f"e{k}": v for k, v in errs.items()}, tol=p.tol)


def makespan_list(jobs):   # jobs: list of durations in start order
    h = [0.0] * SLOTS
    for d in jobs:
        t = heapq.heappop(h)
        heapq.heappush(h, t + d)
    return max(h)


ideal = cost.sum() / SLOTS
out = {"L_mean": float(L.mean()), "L_max": int(L.max()), "ideal": ideal,
       "fifo_eff": ideal / makespan_list(list(cost)),
       "lpt_true_eff": ideal / makespan_list(list(np.sort(cost)[::-1]))}
for K in (8, 12, 16):
    # phase 1: every problem min(L, K) sweeps (2 per sweep), FIFO; phase 2: the parked remainder
    h = [0.0] * SLOTS
    for i in range(1024):
        t = heapq.heappop(h)
        heapq.heappush(h, t + 2 * min(L[i], K) + (1 if L[i] <= K else 0))
    e1, e2 = errs[K - 2], errs[K - 1]
    rho = np.clip(e2 / e1, 1e-6, 0.999999)
    pred = np.log(np.maximum(e2, 1e-30) / p.tol) / -np.log(rho)
    parked = [i for i in range(1024) if L[i] > K]
    order = sorted(parked, key=lambda i: -pred[i])
    # phase 2 starts as slots free up (the heap continues)
    for i in order:
        t = heapq.heappop(h)
        heapq.heappush(h, t + 2 * (L[i] - K) + 1)
    rem = np.array([L[i] - K for i in parked])
    out[f"park_K{K}_eff"] = ideal / max(h)
    # the same with a perfect predictor (upper bound of the two-phase schedule)
    h2 = [0.0] * SLOTS
    for i in range(1024):
        t = heapq.heappop(h2)
        heapq.heappush(h2, t + 2 * min(L[i], K) + (1 if L[i] <= K else 0))
    for i in sorted(parked, key=lambda i: -(L[i] - K)):
        t = heapq.heappop(h2)
        heapq.heappush(h2, t + 2 * (L[i] - K) + 1)
    out[f"park_K{K}_perfect_eff"] = ideal / max(h2)
    out[f"park_K{K}_pred_corr"] = float(np.corrcoef(pred[parked], rem)[0, 1])
print(json.dumps(out))
