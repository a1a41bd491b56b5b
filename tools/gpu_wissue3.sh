#!/bin/bash
# usage (GPU box): tools/gpu_wissue3.sh TAG -- warp-uniform TMA issue from a __constant__ row table:
# interleaved c128 bench A/B (A = per-lane issue everywhere PTSBE_TMA_LANES=32; B = a build whose default is warp-uniform on light non-last passes (measured, not adopted)), then the c128 parity subset under B
mkdir -p gpurun_out
tag=${1:-w}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
for run in A1 B1 A2 B2; do
  case $run in A*) e="PTSBE_TMA_LANES=32";; B*) e="PTSBE_X=0";; esac
  env $e timeout 600 python bench.py --no-cpu --dtype c128 --secondary none > gpurun_out/ab_${tag}_$run.log 2>&1
done
timeout 1200 python -m pytest -x -q -m gpu tests/test_config4_parity.py tests/test_gpu_parity.py \
  -k "config4 or shared_trunk or tile_sizes or prepared or tma_issue_forms" > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
