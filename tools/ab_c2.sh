#!/usr/bin/env bash
# A/B(/C) of a bench step (WL, default c2) across source trees (e.g. . ab_old ab_new), alternating.
set -u
TREES=${*:-. ab_old}
for k in 1 2 3; do
  for t in $TREES; do
    (cd "$t" && timeout 300 python bench.py --workload ${WL:-c2} --steps 10 --warmup 3 --no-cpu-baseline --no-k14 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$t', round(d['ms_per_step'],3), round(d['roofline']['frac'],4))")
  done
done
