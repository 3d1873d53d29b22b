python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -c "
import sys; sys.path.insert(0,'.')
import paper_2206_07630_b200 as sk
c=sk.Context(0)
for shape in (0, 1):
    for mode in (0, 2, 4, 12, 6, 14): print('shape', shape, 'mode', mode, c.microbench(100 + shape + 4 * mode))
for k in ['tc_clk','tc_noload_clk']: print(k, c.microbench(k))
"
EMUS="0" bash tools/tc_sweep.sh
