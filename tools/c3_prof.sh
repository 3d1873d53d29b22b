python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 2000 --log-file gpurun_out/launches_c3b.csv python bench.py --workload c3 --steps 1 --warmup 0 --no-k14 --no-cpu-baseline > gpurun_out/ncu_c3b.log 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_c3b.csv
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 2000 --log-file gpurun_out/launches_c1.csv python bench.py --workload c1 --steps 1 --warmup 0 --no-k14 --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_c1.csv
