python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
[ -z "$NOTEST" ] && timeout 600 python -m pytest tests/test_gpu_sort1d.py tests/test_gpu_adaptive.py tests/test_gpu_relax.py tests/test_gpu_solve.py -q 2>&1 | tail -3
for park in ${PARKS:-8 0 6 12 8 0}; do timeout 300 python - <<PY
import sys, json, torch; sys.path.insert(0,'.')
import paper_2206_07630_b200 as sk
from workloads import gen
p = gen.c2(); c = sk.Context(0); c.set_tuning("batched_park", $park)
x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
def step():
    f0 = sk.sinkhorn_init_sort1d(c, x.view(1024, 1024), y.view(1024), y_shared=True)
    return sk.sinkhorn_solve(c, x, y, p.eps, y_shared=True, f_init=f0)
for _ in range(3): step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): step()
e1.record(); torch.cuda.synchronize()
print("park", $park, "ms/step %.3f" % (e0.elapsed_time(e1) / 10))
PY
done
