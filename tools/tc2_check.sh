# K3 variants on C5: parity tests, then the bench per (SK_TC_EPI, SK_TC_EMU)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for ep in ${EPIS:-162 16}; do
SK_TC_EPI=$ep timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -1
for e in ${EMUS:-1 2}; do SK_TC_EPI=$ep SK_TC_EMU=$e timeout 300 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-k14 > gpurun_out/bench_c5_x${ep}e$e.json 2>gpurun_out/bench_c5_x${ep}e$e.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_c5_x${ep}e$e.json').read().strip().splitlines()[-1]); r=d['roofline']
print('epi $ep emu $e', 'value %.3e'%d['value'], 'its', d['solve']['iterations'], 'frac %.3f mufu %.3f avg_ms %.3f share %.3f'%(r['frac'], r['mufu_frac'], r['avg_launch_ms'], r['share_of_step']), d['clocks'])"; done
done
