"""One launch of the K3 epilogue-only probe (K14 kind 11) or the whole seeded kernel (kind 14) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_07630_b200 as sk
c = sk.Context(0)
print(c.microbench(sys.argv[1] if len(sys.argv) > 1 else "tc_epi"))
