#!/bin/bash
# usage (GPU box): tools/gpu_tiles_r2.sh TAG -- tile-size experiments, interleaved twice
mkdir -p gpurun_out
tag=$1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
  timeout 900 python bench.py --no-cpu --secondary none > gpurun_out/tl_${tag}_c128L11_$rep.log 2>&1
  timeout 900 python bench.py --no-cpu --secondary none --tile-bits 12 > gpurun_out/tl_${tag}_c128L12_$rep.log 2>&1
  PTSBE_NO_TMA=1 timeout 900 python bench.py --no-cpu --secondary none --tile-bits 12 > gpurun_out/tl_${tag}_c128L12cpa_$rep.log 2>&1
  PTSBE_TMA=1 timeout 900 python bench.py --no-cpu --dtype c64 --secondary none --tile-bits 13 > gpurun_out/tl_${tag}_c64L13tma_$rep.log 2>&1
  timeout 900 python bench.py --no-cpu --dtype c64 --secondary none --tile-bits 13 > gpurun_out/tl_${tag}_c64L13_$rep.log 2>&1
done
