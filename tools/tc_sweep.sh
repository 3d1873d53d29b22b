python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_large.py -k "tc or sharded or c5" -x -q 2>&1 | tail -5
for ab in 2 1; do
SK_TC_ABUF=$ab python -c "
import sys; sys.path.insert(0,'.')
import paper_2206_07630_b200 as sk
c=sk.Context(0)
for k in ['tc','tc_noload']: print('abuf $ab', k, c.microbench(k)/1e12)
"
for e in ${EMUS:-0 2}; do SK_TC_ABUF=$ab SK_TC_EMU=$e timeout 400 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-k14 > gpurun_out/bench_c5_emu$e.json 2>gpurun_out/bench_c5_emu$e.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_c5_emu$e.json').read().strip().splitlines()[-1]); r=d['roofline']
print('abuf $ab emu $e', 'value %.3e'%d['value'], 'its', d['solve']['iterations'], 'frac %.3f mufu %.3f avg_ms %.3f share %.3f'%(r['frac'], r['mufu_frac'], r['avg_launch_ms'], r['share_of_step']), d['clocks'])"; done
done
