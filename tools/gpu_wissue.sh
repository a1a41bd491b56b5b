#!/bin/bash
# usage (GPU box): tools/gpu_wissue.sh TAG -- warp-uniform TMA issue: parity subset + interleaved c128 bench A/B
# (A = per-lane issue PTSBE_TMA_LANES=32, B = warp-uniform default)
mkdir -p gpurun_out
tag=${1:-w}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 1200 python -m pytest -x -q -m gpu tests/test_config4_parity.py tests/test_gpu_parity.py \
  -k "config4 or shared_trunk or tree_schedule or tile_sizes or config3 or active or prepared or fused" \
  > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
for run in A1 B1 A2 B2; do
  case $run in A*) e="PTSBE_TMA_LANES=32";; B*) e="PTSBE_TMA_LANES=0";; esac
  env $e timeout 600 python bench.py --no-cpu --dtype c128 --secondary none > gpurun_out/ab_${tag}_$run.log 2>&1
done
