python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_wide.py tests/test_gpu_tc.py -m gpu -x -q ${PYARGS:-} > gpurun_out/wide.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/wide.log
