"""K14: print the measured roofline denominators of this device (JSON)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_07630_b200 as sk  # noqa: E402

ctx = sk.Context(0)
out = {k: ctx.microbench(k) for k in ("ex2", "ffma", "hbm", "tc")}
out = {"ex2_per_s": out["ex2"], "ffma_per_s": out["ffma"], "hbm_read_GBps": out["hbm"] / 1e9,
       "tc_f16_TFLOPs": out["tc"] / 1e12}
print(json.dumps(out))
