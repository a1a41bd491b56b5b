#!/bin/bash
# usage (GPU box): tools/gpu_sweep.sh TAG "ENV=.. ENV=..|--bench-args" ...   -- one bench (no CPU leg) per entry
mkdir -p gpurun_out
tag=$1; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
for e in "$@"; do
  envs=${e%%|*}; args=""
  [[ "$e" == *"|"* ]] && args=${e#*|}
  echo "== $e" >> gpurun_out/sweep_$tag.log
  env $envs timeout 600 python bench.py --no-cpu $args >> gpurun_out/sweep_$tag.log 2>&1
done
