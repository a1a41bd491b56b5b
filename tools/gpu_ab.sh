#!/bin/bash
# usage (GPU box): tools/gpu_ab.sh TAG "ENV_A" "ENV_B" [bench args]  -- bench A then B (then A again) on one box
mkdir -p gpurun_out
tag=$1; a=$2; b=$3; shift 3
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for run in A1 B1 A2 B2; do
  case $run in A*) e=$a;; B*) e=$b;; esac
  env $e timeout 900 python bench.py --no-cpu "$@" > gpurun_out/ab_${tag}_$run.log 2>&1
done
