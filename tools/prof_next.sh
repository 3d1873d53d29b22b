# ncu summaries of the NEXT-row kernels (K15 soft rank/sort, K16 EM, K17 VJP plan pass, K18 NW 1D)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
cat > /tmp/next_probe.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2206_07630_b200 as sk
from workloads import gen
ctx = sk.Context(0)
c2 = gen.c2()
xb, yb = torch.from_numpy(c2.x).cuda(), torch.from_numpy(c2.y).cuda()
pot = sk.sinkhorn_init_sort1d(ctx, xb.view(1024, 1024), yb.view(-1))
f, g, _ = sk.sinkhorn_solve(ctx, xb, yb, c2.eps, y_shared=True, f_init=pot)
sk.sinkhorn_soft_rank_sort(ctx, xb.view(1024, 1024), yb.view(-1), c2.eps, f, g, y_shared=True)
p3 = gen.c3()
sk.sinkhorn_fit_gmm(ctx, torch.from_numpy(p3.x).cuda(), 8, gen.gmm_start_idx(p3.n, 8, 3), iters=5)
p4 = gen.c4(n=16384)
x4, y4 = torch.from_numpy(p4.x).cuda(), torch.from_numpy(p4.y).cuda()
f4, g4, _ = sk.sinkhorn_solve(ctx, x4, y4, p4.eps, mode="online")
n = p4.n
sk.sinkhorn_vjp(ctx, x4, y4, p4.eps, f4, g4, torch.full((n,), 1 / n, device="cuda"), torch.full((n,), 1 / n, device="cuda"), cg_max_iter=16)
rng = np.random.default_rng(0)
xn = torch.from_numpy(rng.random((64, 2000)).astype(np.float32)).cuda()
yn = torch.from_numpy(np.sort(rng.random(1500)).astype(np.float32)).cuda()
sk.sinkhorn_init_nw1d(ctx, xn, yn)
torch.cuda.synchronize()
print("ok")
PY
python /tmp/next_probe.py && \
timeout 600 ncu --set full --clock-control none -k regex:"k_soft_rank_sort|k_em_estep|k_plan_pass|k_nw1d" -c 5 -o gpurun_out/prof_next -f python /tmp/next_probe.py > gpurun_out/prof_next.log 2>&1; tail -2 gpurun_out/prof_next.log
