#!/bin/bash
# usage (GPU box): tools/gpu_abc.sh TAG "ENV0" "ENV1" "ENV2" [bench args] -- variants interleaved, twice each
mkdir -p gpurun_out
tag=$1; v0=$2; v1=$3; v2=$4; shift 4
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
  for i in 0 1 2; do
    case $i in 0) e=$v0;; 1) e=$v1;; 2) e=$v2;; esac
    env $e timeout 900 python bench.py --no-cpu "$@" > gpurun_out/abc_${tag}_v${i}_$rep.log 2>&1
  done
done
