python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "stored or c3 or sharded or gmm" 2>&1 | tail -4
for pz in 1 0; do SK_PERSIST=$pz timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --no-k14 > gpurun_out/bench_c3_p$pz.json 2>gpurun_out/bench_c3_p$pz.err; tail -2 gpurun_out/bench_c3_p$pz.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_c3_p$pz.json').read().strip().splitlines()[-1]); r=d['roofline']
print('persist $pz', 'value %.3e ms %.2f'%(d['value'], d['ms_per_step']), 'solve', d['solve'], 'frac %.3f avg_ms %.3f share %.3f'%(r['frac'], r['avg_launch_ms'], r['share_of_step']), 'ttt', d['time_to_tol_ms'])"; done
