#!/bin/bash
# usage (GPU box): tools/gpu_abc.sh TAG "ENV_B" "ENV_C" -- c128 bench: default (A) vs ENV_B vs ENV_C, interleaved twice
mkdir -p gpurun_out
tag=$1; eb=$2; ec=$3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
for run in A1 B1 C1 A2 B2 C2; do
  case $run in A*) e=PTSBE_X=0;; B*) e=$eb;; C*) e=$ec;; esac
  env $e timeout 600 python bench.py --no-cpu --dtype c128 --secondary none > gpurun_out/abc_${tag}_$run.log 2>&1
done
