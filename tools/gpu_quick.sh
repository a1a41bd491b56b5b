#!/bin/bash
# usage (GPU box): tools/gpu_quick.sh TAG [pytest args...] -- build, a pytest selection, default bench (both dtypes)
mkdir -p gpurun_out
tag=${1:-q}; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
if [ $# -gt 0 ]; then timeout 1500 python -m pytest "$@" -q -m gpu > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log; fi
timeout 900 python bench.py --no-cpu > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$tag.log
