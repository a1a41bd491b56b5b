#!/bin/bash
# usage (on the GPU box via gpurun): tools/gpu_r2b.sh TAG [pytest args...]
# build + smoke + pytest -m gpu (no -x: every failure is listed) [+ bench unless NOBENCH=1]
mkdir -p gpurun_out
tag=${1:-r}; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
timeout 2400 python -m pytest -q -m gpu --durations=30 "${@:-tests}" > gpurun_out/pytest_gpu_$tag.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
if [ -z "$NOBENCH" ]; then
  timeout 900 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$tag.log
fi
