"""C3 (n = m = 16384, d = 16) solved in stored mode (K4 build + K5 fused sweeps) and in online mode
(K3 tensor-core passes, compact K = 16 images), same init / eps / tol: time to tol and sweeps.
    python tools/c3_modes.py [eps_factor]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_07630_b200 as sk  # noqa: E402
from workloads import gen  # noqa: E402

ef = float(sys.argv[1]) if len(sys.argv) > 1 else 0.01
p = gen.c3(eps_factor=ef)
ctx = sk.Context(0)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
f0, side = sk.sinkhorn_init_gaussian(ctx, x, y)
res = {}
for mode in ("stored", "online", "online_tc", "stored", "online", "online_tc"):
    ctx.set_tuning("tc_min_d", 1 if mode == "online_tc" else 17)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f, g, rep = sk.sinkhorn_solve(ctx, x, y, p.eps, tol=p.tol, mode=mode.split("_")[0], f_init=f0)
    e1.record()
    torch.cuda.synchronize()
    res[mode] = {"ms": e0.elapsed_time(e1), "L": rep["iterations"], "err": rep["marginal_error"],
                 "E": rep["dual_objective"], "f": f.clone()}
out = {m: {k: v for k, v in r.items() if k != "f"} for m, r in res.items()}
fs = res["stored"]["f"].double()
for mo in ("online", "online_tc"):
    fo = res[mo]["f"].double()
    out[f"f_rel_inf_{mo}_vs_stored"] = float(((fs - fs.mean()) - (fo - fo.mean())).abs().max() / max(float((fs - fs.mean()).abs().max()), p.eps))
out["eps"] = p.eps
print(json.dumps(out))
