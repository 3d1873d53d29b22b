"""Small instances of every kernel path, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_07630_b200 as sk  # noqa: E402
from workloads import gen  # noqa: E402

ctx = sk.Context(0)
c = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
rng = np.random.default_rng(0)
# on-chip batched (d=1, shared y) + sort1d closed form and paper mode
p = gen.c2(B=6, n=300)
f0 = sk.sinkhorn_init_sort1d(ctx, c(p.x).view(6, 300), c(p.y).view(-1))
f0j = sk.sinkhorn_init_sort1d(ctx, c(p.x).view(6, 300), c(p.y).view(-1), dualsort_iters=2)
sk.sinkhorn_solve(ctx, c(p.x), c(p.y), p.eps, y_shared=True, f_init=f0, max_iter=50)
sk.sinkhorn_sort1d_batched(ctx, c(p.x).view(6, 300))
# single small on-chip (d=2) with weights
p1 = gen.c1(n=100)
g0, _ = sk.sinkhorn_init_gaussian(ctx, c(p1.x), c(p1.y))
sk.sinkhorn_solve(ctx, c(p1.x), c(p1.y), p1.eps, f_init=g0, a=c(gen.random_weights(100, rng)))
# online FFMA (d=3), ragged
x = rng.random((1300, 3)).astype(np.float32); y = rng.random((777, 3)).astype(np.float32)
sk.sinkhorn_solve(ctx, c(x), c(y), 0.05, mode="online", max_iter=20)
# tensor-core path (d=64 and d=20), ragged
p5 = gen.c5(n=700, eps_factor=0.1)
sk.sinkhorn_solve(ctx, c(p5.x), c(p5.y[:515]), p5.eps, mode="online", max_iter=10)
x20 = rng.standard_normal((300, 20)).astype(np.float32)
sk.sinkhorn_solve(ctx, c(x20), c(x20[:257] + 0.1), 2.0, mode="online", max_iter=10)
# stored (d=16) + GMM init
p3 = gen.c3(n=1100, eps_factor=0.05)
gx = {k: c(v) for k, v in p3.extra["gmm_x"].items()}; gy = {k: c(v) for k, v in p3.extra["gmm_y"].items()}
fg, _ = sk.sinkhorn_init_gmm(ctx, c(p3.x), c(p3.y), gx, gy, p3.eps)
sk.sinkhorn_solve(ctx, c(p3.x), c(p3.y), p3.eps, mode="stored", f_init=fg, max_iter=20)
# subsample init + emulated sharding
p4 = gen.c4(n=3000, ns=200)
sk.sinkhorn_init_subsample(ctx, c(p4.x), c(p4.y), c(p4.extra["idx_x"]), c(p4.extra["idx_y"]), p4.eps, 1e-3)
sk.sinkhorn_solve_sharded_emulated(ctx, 2, c(p4.x), c(p4.y), p4.eps, max_iter=10)
# relaxation / eps-decay on the on-chip and merge paths, the CTA-pair on-chip variant (C1 size)
sk.sinkhorn_solve(ctx, c(p1.x), c(p1.y), p1.eps, omega=1.5, eps_decay=(5.0, 0.8), max_iter=30)
sk.sinkhorn_solve(ctx, c(x), c(y), 0.05, mode="online", omega=1.3, max_iter=12)
sk.sinkhorn_solve(ctx, c(x), c(y), 0.05, mode="online", eps_decay=(5.0, 0.8), max_iter=14)
# soft ranks / sort, general 1D initializer, GMM fit, VJP
fb, gb, _ = sk.sinkhorn_solve(ctx, c(p.x), c(p.y), p.eps, y_shared=True, f_init=f0, max_iter=30)
sk.sinkhorn_soft_rank_sort(ctx, c(p.x).view(6, 300), c(p.y).view(-1), p.eps, fb, gb, y_shared=True)
xw = c(rng.random((3, 250)).astype(np.float32)); yw = c(np.sort(rng.random(170)).astype(np.float32))
sk.sinkhorn_init_nw1d(ctx, xw, yw, a=c(np.stack([gen.random_weights(250, rng) for _ in range(3)])))
sk.sinkhorn_init_nw1d(ctx, xw, yw)
sk.sinkhorn_fit_gmm(ctx, c(p3.x), 4, gen.gmm_start_idx(p3.n, 4, 3), iters=3)
fv, gv, _ = sk.sinkhorn_solve(ctx, c(x), c(y), 0.05, mode="online", max_iter=20)
sk.sinkhorn_vjp(ctx, c(x), c(y), 0.05, fv, gv, c(rng.standard_normal(1300).astype(np.float32)),
                c(rng.standard_normal(777).astype(np.float32)), cg_max_iter=10)
torch.cuda.synchronize()
print("sanitize smoke ok")
