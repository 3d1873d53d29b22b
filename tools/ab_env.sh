#!/usr/bin/env bash
# A/B of the C2 bench step across environment settings ("VAR=val VAR2=val" strings), alternating.
set -u
for k in 1 2 3; do
  for e in "$@"; do
    env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-k14 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$e', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), round(d['solve']['anderson5']['time_to_tol_ms'],3))"
  done
done
