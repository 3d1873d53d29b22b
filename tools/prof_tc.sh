# ncu --set full of one K3 launch (C5), variant chosen by SK_TC_PAIR
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export SK_TC_PAIR=${SK_TC_PAIR:-1}
timeout 300 python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline --no-k14 > gpurun_out/prof_tc_plain.json 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lse_tc -s 20 -c 1 -o gpurun_out/prof_tc${SK_TC_PAIR} -f \
  python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline --no-k14 > gpurun_out/prof_tc_ncu.log 2>&1
tail -3 gpurun_out/prof_tc_ncu.log
