#!/usr/bin/env bash
# A/B of sk_set_tuning settings on one workload's bench step, alternating:
#   WL=c4 STEPS=5 bash tools/ab_tune.sh "lse_emu8=1" "lse_emu8=2"
set -u
WL=${WL:-c4}
for k in 1 2 3; do
  for spec in "$@"; do
    args=""
    for kv in $spec; do args="$args --tune $kv"; done
    timeout 600 python bench.py --workload $WL --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-k14 --no-anderson $args 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$spec', round(d['ms_per_step'],3), round(d['roofline']['frac'],4))"
  done
done
