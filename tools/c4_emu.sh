python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for e in 2 1 0; do SK_LSE_EMU8=$e timeout 600 python bench.py --workload c4 --init zero --steps 3 --warmup 3 --no-cpu-baseline --no-k14 > gpurun_out/bench_c4_e$e.json 2>gpurun_out/bench_c4_e$e.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_c4_e$e.json').read().strip().splitlines()[-1]); r=d['roofline']
print('emu8 $e', 'value %.3e ms %.2f'%(d['value'], d['ms_per_step']), 'its', d['solve']['iterations'], 'frac %.3f avg_ms %.3f share %.3f'%(r['frac'], r['avg_launch_ms'], r['share_of_step']), d['clocks'])"; done
