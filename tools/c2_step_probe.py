"""Where the C2 bench step's time outside the K13 launch goes: CUDA events on the library's
stream around the initializer and the solve, host wall time per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07630_b200 as sk
from workloads import gen
p = gen.c2()
st = torch.cuda.Stream()
ctx = sk.Context(0, st)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
B, n, m = p.batch, p.n, p.m
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
with torch.cuda.stream(st):
    for it in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev[0].record(st)
        f0 = sk.sinkhorn_init_sort1d(ctx, x.view(B, n), y.view(m), y_shared=True)
        ev[1].record(st)
        t1 = time.perf_counter()
        f, g, reps = sk.sinkhorn_solve(ctx, x, y, p.eps, y_shared=True, f_init=f0)
        ev[2].record(st)
        t2 = time.perf_counter()
        torch.cuda.synchronize()
        if it >= 3:
            print("init %.3f ms (host %.3f)  solve %.3f ms (host %.3f, loop %.3f)  total %.3f" % (
                ev[0].elapsed_time(ev[1]), 1e3 * (t1 - t0), ev[1].elapsed_time(ev[2]), 1e3 * (t2 - t1),
                reps[0]["solve_ms"], ev[0].elapsed_time(ev[2])))
