#!/bin/bash
mkdir -p gpurun_out
tag=$1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
i=0
for e in "PTSBE_X=1 TB=11" "PTSBE_X=1" "PTSBE_NO_TMA=1" "PTSBE_MIN_BLOCKS=2" "PTSBE_MIN_BLOCKS=2 PTSBE_NO_TMA=1" "PTSBE_STAGES=2" "PTSBE_STAGES=2 PTSBE_NO_TMA=1"; do
  tb=12; case "$e" in *TB=11*) tb=11;; esac
  for rep in 1 2; do
    env $e timeout 900 python bench.py --no-cpu --secondary none --tile-bits $tb > gpurun_out/L12_${tag}_e${i}_$rep.log 2>&1
  done
  i=$((i+1))
done
