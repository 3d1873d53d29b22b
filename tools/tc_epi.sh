# K3 pair kernel on the 32768^2 probe: cycles per 256x256 pair tile of the MMA pipeline alone
# (tc_clk), the epilogue alone (tc_epi) and the bare TMEM loads (tc_tmem)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for ne in ${EPIS:-162 16 8}; do for e in ${EMUS:-1}; do SK_TC_EPI=$ne SK_TC_EMU=$e timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import paper_2206_07630_b200 as sk
c=sk.Context(0)
tile = 3*2*64*256*128   # flops per SM per pair tile
for k in ['tc_clk', 'tc_epi', 'tc_math']:
    v = c.microbench(k)
    print('ne $ne emu $e %-8s %.0f cycles per tile' % (k, tile / v))
"; done; done
