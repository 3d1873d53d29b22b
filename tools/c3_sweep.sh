python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_large.py -k "stored or c3 or sharded" -x -q 2>&1 | tail -5
for f in 1 0; do SK_FUSED=$f timeout 400 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --no-k14 > gpurun_out/bench_c3_f$f.json 2>gpurun_out/bench_c3_f$f.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_c3_f$f.json').read().strip().splitlines()[-1]); r=d['roofline']
print('fused $f', 'value %.3e ms %.2f'%(d['value'], d['ms_per_step']), 'its', d['solve']['iterations'], 'frac %.3f avg_ms %.3f share %.3f'%(r['frac'], r['avg_launch_ms'], r['share_of_step']), d['clocks'])"; done
