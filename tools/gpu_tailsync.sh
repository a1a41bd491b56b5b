#!/bin/bash
# usage (GPU box): tools/gpu_tailsync.sh TAG -- team tail barrier: parity subset + interleaved c128 bench A/B
# (A = team barrier after each store PTSBE_TEAM_TAIL_SYNC=1, B = none (default))
mkdir -p gpurun_out
tag=${1:-w}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 1200 python -m pytest -x -q -m gpu tests/test_config4_parity.py tests/test_gpu_parity.py \
  -k "config4 or shared_trunk or tree_schedule or tile_sizes or config3 or active or prepared or fused" \
  > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
for run in A1 B1 A2 B2; do
  case $run in A*) e="PTSBE_TEAM_TAIL_SYNC=1";; B*) e="PTSBE_X=0";; esac
  env $e timeout 600 python bench.py --no-cpu --dtype c128 --secondary none > gpurun_out/ab_${tag}_$run.log 2>&1
done
