#!/bin/bash
mkdir -p gpurun_out
tag=$1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
i=0
for e in "PTSBE_X=1 TB=12" "PTSBE_X=1" "PTSBE_TMA=1" "PTSBE_MIN_BLOCKS=2" "PTSBE_MIN_BLOCKS=2 PTSBE_TMA=1" "PTSBE_MIN_BLOCKS=3 PTSBE_TMA=1"; do
  tb=13; case "$e" in *TB=12*) tb=12;; esac
  for rep in 1 2; do
    env $e timeout 900 python bench.py --no-cpu --dtype c64 --secondary none --tile-bits $tb > gpurun_out/L13_${tag}_e${i}_$rep.log 2>&1
  done
  i=$((i+1))
done
