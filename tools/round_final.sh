#!/usr/bin/env bash
# Build, the whole GPU suite, then tools/measure.sh TAG (bench lines, launch lists, ncu captures).
TAG=${1:-rXX}
mkdir -p gpurun_out/$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/$TAG/build0.log 2>&1 || { tail gpurun_out/$TAG/build0.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/$TAG/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/$TAG/gputest.log
bash tools/measure.sh $TAG
