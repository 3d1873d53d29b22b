# K14 MMA probes: raw tcgen05 rates (flop per SM clock) of the probe shapes, and the K3 kernel's
# MMA pipeline with the epilogue reduced to buffer releases (tc_clk) and without B reloads.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2206_07630_b200 as sk
c=sk.Context(0)
for shape in (0, 1):
    for mode in (0, 1, 2, 4, 12): print('shape', shape, 'mode', mode, '%.0f flop/clk/SM' % c.microbench(100 + shape + 4 * mode))
for k in ['tc','tc_noload']: print(k, '%.1f TF/s' % (c.microbench(k) / 1e12))
for k in ['tc_clk','tc_noload_clk']: print(k, '%.0f flop/clk/SM' % c.microbench(k))
"
SK_TC_PAIR=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2206_07630_b200 as sk
c=sk.Context(0)
for k in ['tc','tc_clk']: print('pair', k, '%.1f' % (c.microbench(k) / (1e12 if k == 'tc' else 1)))
"
