#!/bin/bash
# usage (GPU box): tools/gpu_ab2.sh TAG "ENV_B" [pytest args] -- pytest selection, then c128 bench default (A) vs ENV_B (B)
# interleaved A B A B (default steps), then the c64 bench once
mkdir -p gpurun_out
tag=$1; eb=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
if [ $# -gt 0 ]; then timeout 1500 python -m pytest "$@" -q -m gpu > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log; fi
for run in A1 B1 A2 B2; do
  case $run in A*) e=PTSBE_X=0;; B*) e=$eb;; esac
  env $e timeout 600 python bench.py --no-cpu --dtype c128 --secondary none > gpurun_out/ab_${tag}_$run.log 2>&1
done
timeout 600 python bench.py --no-cpu --dtype c64 --secondary none > gpurun_out/ab_${tag}_c64.log 2>&1
