#!/bin/bash
# usage (GPU box): tools/gpu_teams.sh TAG -- parity subset, then c128 bench with 1 vs 2 compute teams
# (interleaved repeats) and the c64 bench
mkdir -p gpurun_out
tag=${1:-t}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 1500 python -m pytest tests/test_config4_parity.py tests/test_gpu_parity.py tests/test_sharded.py -q -m gpu > gpurun_out/pytest_$tag.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
for run in T2a T1a T2b T1b; do
  case $run in T2*) e=PTSBE_TEAMS=2;; T1*) e=PTSBE_TEAMS=1;; esac
  env $e timeout 600 python bench.py --no-cpu --dtype c128 --secondary none --steps 4 --warmup 3 > gpurun_out/teams_${tag}_$run.log 2>&1
done
timeout 600 python bench.py --no-cpu --dtype c64 --secondary none --steps 4 --warmup 3 > gpurun_out/teams_${tag}_c64.log 2>&1
