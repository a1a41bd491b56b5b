#!/bin/bash
# usage (GPU box): tools/gpu_exp.sh TAG "ENV|ARGS" ... -- each variant twice, interleaved
mkdir -p gpurun_out
tag=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
  i=0
  for v in "$@"; do
    e=${v%%|*}; a=${v#*|}
    env $e timeout 900 python bench.py --no-cpu $a > gpurun_out/exp_${tag}_v${i}_$rep.log 2>&1
    i=$((i+1))
  done
done
