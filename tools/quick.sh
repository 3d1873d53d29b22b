python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q ${TESTK:+-k "$TESTK"} 2>&1 | tail -4
for w in ${WLS:-c3}; do timeout 600 python bench.py --workload $w --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-k14 > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_$w.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', 'value %.3e ms %.2f'%(d['value'], d['ms_per_step']), 'solve', d['solve'], 'frac %.3f avg_ms %.3f share %.3f'%(r['frac'], r['avg_launch_ms'], r['share_of_step']), 'ttt', d['time_to_tol_ms'], d['clocks'])"; done
