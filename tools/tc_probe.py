"""K3 probes (K14 kinds 9-14 on the 32768^2 probe, d = 64): cycles per 256 x 256 pair tile of the
whole seeded kernel (tc_full), the MMAs with the operand stream (tc_clk), the MMA pipeline alone (tc_noload_clk), the epilogue alone (tc_epi), the bare
TMEM loads + releases (tc_tmem) and the epilogue arithmetic without loads (tc_math), for each
epilogue organisation / FMA-pipe exponential share given on the command line.
    python tools/tc_probe.py [epi,emu[,pipe] ...]   (default: 162,2 16,2)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_07630_b200 as sk  # noqa: E402

tile = 3 * 2 * 64 * 256 * 128   # flops per SM per pair tile
for spec in (sys.argv[1:] or ["162,2", "16,2"]):
    v = [int(t) for t in spec.split(",")]
    epi, emu, pipe = v[0], v[1], (v[2] if len(v) > 2 else 0)
    c = sk.Context(0)
    c.set_tuning("tc_epi", epi)
    c.set_tuning("tc_emu", emu)
    c.set_tuning("tc_pipe", pipe)
    out = {k: tile / c.microbench(k) for k in ("tc_full", "tc_clk", "tc_noload_clk", "tc_epi", "tc_tmem", "tc_math")}
    print(f"epi {epi} emu {emu} pipe {pipe}: " + "  ".join(f"{k} {v:.0f}" for k, v in out.items()), flush=True)
    c.close()
