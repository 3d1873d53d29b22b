"""d in (64, 256]: per-sweep time and K3's tensor-pipe rate on a BJ.cfg5-shaped problem
(embedding-like, L2-normalised) at n = m = 65536 for d = 64 .. 256, and the wide FFMA pass (K2,
tc = 0) at n = m = 16384, a fixed number of sweeps from zero init, eps = 0.01 mean(C).
K3 MMA flops per entry: 2 x 16 x (3 ksteps + 1) (3-product fp16 split plus the extra-column step).

    python tools/wide_perf.py [sweeps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_07630_b200 as sk  # noqa: E402
from workloads import gen  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
out = []
for d, n, tc in [(64, 65536, 1), (128, 65536, 1), (192, 65536, 1), (256, 65536, 1), (128, 16384, 0), (256, 16384, 0)]:
    p = gen.c5(n=n, d=d)
    ctx = sk.Context(0)
    ctx.set_tuning("tc", tc)
    ctx.set_timing(True)
    x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
    sk.sinkhorn_solve(ctx, x, y, p.eps, tol=1e-12, max_iter=2, mode="online")   # warm-up
    torch.cuda.synchronize()
    ctx.reset_counters()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f, g, rep = sk.sinkhorn_solve(ctx, x, y, p.eps, tol=1e-12, max_iter=L, mode="online")
    e1.record()
    torch.cuda.synchronize()
    c = ctx.counters()
    ms = e0.elapsed_time(e1)
    r = {"d": d, "n": n, "kernel": "K3" if tc else "K2 wide", "sweeps": rep["iterations"], "ms_per_sweep": ms / rep["iterations"],
         "entries_per_s": 2.0 * n * n * rep["iterations"] / (ms * 1e-3)}
    if c["dom_launches"]:
        avg = c["dom_ms"] / c["dom_launches"]
        r["dom_avg_ms"] = avg
        if tc:
            ks = (d + 15) // 16
            tf = 2.0 * 16 * (3 * ks + 1) * n * n / (avg * 1e-3) / 1e12
            r["tensor_tflops"] = tf
            r["frac_burst"] = tf / peak["bf16_tflops"]
            r["frac_sustained"] = tf / peak["bf16_tflops_sustained"]
        else:
            r["ffma_per_s"] = d * n * n / (avg * 1e-3)
    out.append(r)
    print(json.dumps(r), flush=True)
    ctx.close()
