#!/bin/bash
# usage (GPU box): tools/gpu_wissue2.sh TAG -- warp-uniform TMA issue from a __constant__ row table:
# interleaved c128 bench A/B (A = per-lane issue, default; B = PTSBE_TMA_LANES=0), then the c128 parity subset under B
mkdir -p gpurun_out
tag=${1:-w}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
for run in A1 B1 A2 B2; do
  case $run in A*) e="PTSBE_X=0";; B*) e="PTSBE_TMA_LANES=0";; esac
  env $e timeout 600 python bench.py --no-cpu --dtype c128 --secondary none > gpurun_out/ab_${tag}_$run.log 2>&1
done
PTSBE_TMA_LANES=0 timeout 1200 python -m pytest -x -q -m gpu tests/test_config4_parity.py tests/test_gpu_parity.py \
  -k "config4 or shared_trunk or tile_sizes or prepared" > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
