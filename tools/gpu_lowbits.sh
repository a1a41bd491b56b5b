#!/bin/bash
# usage (GPU box): tools/gpu_lowbits.sh TAG -- c128 / c64 bench at several contiguous low-bit runs (interleaved)
mkdir -p gpurun_out
tag=${1:-lo}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
for rep in 1 2; do
  for lb in 3 5; do timeout 600 python bench.py --no-cpu --dtype c128 --secondary none --low-bits $lb > gpurun_out/lo_${tag}_c128_${lb}_$rep.log 2>&1; done
done
for lb in 4 5; do timeout 600 python bench.py --no-cpu --dtype c64 --secondary none --low-bits $lb > gpurun_out/lo_${tag}_c64_${lb}.log 2>&1; done
