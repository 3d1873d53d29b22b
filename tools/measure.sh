#!/usr/bin/env bash
# One GPU call: the default bench (C4) plus every other BASELINE.json config through bench.py,
# the sharded per-sweep cost, ncu launch lists and one `--set full` capture of each workload's
# dominant kernel.  Output under gpurun_out/$TAG/.
#   gpurun --timeout 3600 -- 'bash tools/measure.sh r02a'
set -u
TAG=${1:-rXX}
O=gpurun_out/$TAG
mkdir -p "$O"
python -c "import __graft_entry__ as g; g.build()" > "$O/build.log" 2>&1 || { echo build failed; tail "$O/build.log"; exit 1; }
B="timeout 900 python bench.py"
$B > "$O/bench_c4.json" 2> "$O/bench_c4.err"; echo "c4 (default) rc=$?"
$B --impl reference > "$O/bench_reference.json" 2> "$O/bench_reference.err"; echo "reference rc=$?"
$B --no-k14 --workload c2 > "$O/bench_c2.json" 2> "$O/bench_c2.err"; echo "c2 rc=$?"
$B --no-k14 --workload c1 --steps 20 --warmup 3 > "$O/bench_c1.json" 2> "$O/bench_c1.err"; echo "c1 rc=$?"
$B --no-k14 --workload c3 --steps 10 --warmup 3 > "$O/bench_c3.json" 2> "$O/bench_c3.err"; echo "c3 rc=$?"
$B --no-k14 --workload c3 --init gaussian --eps-factor 0.05 --no-cpu-baseline --steps 10 --warmup 3 > "$O/bench_c3_g05.json" 2> "$O/bench_c3_g05.err"; echo "c3g rc=$?"
$B --no-k14 --workload c5 --steps 5 --warmup 3 > "$O/bench_c5.json" 2> "$O/bench_c5.err"; echo "c5 rc=$?"
$B --no-k14 --workload c5 --eps-factor 0.1 --no-cpu-baseline --steps 5 --warmup 3 > "$O/bench_c5_e1.json" 2> "$O/bench_c5_e1.err"; echo "c5e1 rc=$?"
$B --no-k14 --workload c5 --eps-factor 0.001 --no-cpu-baseline --steps 3 --warmup 3 > "$O/bench_c5_e3.json" 2> "$O/bench_c5_e3.err"; echo "c5e3 rc=$?"
for dd in 128 256; do
  $B --no-k14 --workload c5 --d $dd --no-cpu-baseline --steps 3 --warmup 3 > "$O/bench_c5_d$dd.json" 2> "$O/bench_c5_d$dd.err"; echo "c5 d=$dd rc=$?"
done
timeout 300 python tools/shard_cost.py c4 12 > "$O/shard_cost_c4.json" 2>&1; echo "shard c4 rc=$?"
timeout 300 python tools/shard_cost.py c5 8 > "$O/shard_cost_c5.json" 2>&1; echo "shard c5 rc=$?"
# launch lists (cold-cache, serialised: shares only) of the default bench command and the others
NCU="timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv"
$NCU -c 3000 --log-file "$O/launches_c4.csv" python bench.py --steps 2 --warmup 1 --no-k14 --no-cpu-baseline --no-anderson > "$O/ncu_c4.log" 2>&1; echo "ncu c4 rc=$?"
$NCU -c 400 --log-file "$O/launches_c2.csv" python bench.py --workload c2 --steps 2 --warmup 1 --no-k14 --no-cpu-baseline > "$O/ncu_c2.log" 2>&1; echo "ncu c2 rc=$?"
for w in c3 c5; do
  $NCU -c 200 --log-file "$O/launches_$w.csv" python tools/prof_c4.py $w > "$O/ncu_$w.log" 2>&1; echo "ncu $w rc=$?"
done
FULL="timeout 900 ncu --set full --clock-control none --import-source on"
$FULL -k regex:k_lse -s 4 -c 1 -o "$O/full_c4" python tools/prof_c4.py c4 > "$O/full_c4.log" 2>&1; echo "full c4 rc=$?"
$FULL -k regex:k_batched -c 1 -o "$O/full_c2" python bench.py --workload c2 --steps 1 --warmup 0 --no-k14 --no-cpu-baseline > "$O/full_c2.log" 2>&1; echo "full c2 rc=$?"
$FULL -k regex:k_stored_fused -s 2 -c 1 -o "$O/full_c3" python tools/prof_c4.py c3 > "$O/full_c3.log" 2>&1; echo "full c3 rc=$?"
$FULL -k regex:k_lse_tc -s 4 -c 1 -o "$O/full_c5" python tools/prof_c4.py c5 > "$O/full_c5.log" 2>&1; echo "full c5 rc=$?"
for f in "$O"/bench_*.json; do echo "== $f"; tail -c 600 "$f"; echo; done
