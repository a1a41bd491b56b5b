#!/bin/bash
# usage (GPU box): tools/gpu_teams2.sh TAG -- c128 parity, then c128 bench: auto teams vs one team (interleaved)
mkdir -p gpurun_out
tag=${1:-t}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 900 python -m pytest tests/test_config4_parity.py -q -m gpu -k c128 > gpurun_out/pytest_$tag.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
for run in A1 B1 A2 B2; do
  case $run in A*) e=PTSBE_X=0;; B*) e=PTSBE_TEAMS=1;; esac
  env $e timeout 600 python bench.py --no-cpu --dtype c128 --secondary none --steps 4 --warmup 3 > gpurun_out/teams_${tag}_$run.log 2>&1
done
