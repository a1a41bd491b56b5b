#!/bin/bash
# usage (GPU box): tools/ncu_pass.sh TAG PASS DTYPE [ENV...] -- ncu --set full of one pass launch of the bench, raw CSV
mkdir -p gpurun_out
tag=$1; pass=$2; d=$3; shift 3
if [ $d = c128 ]; then np=17; else np=12; fi
env "$@" timeout 900 ncu --set full --clock-control none -k regex:"ptsbe_pass_${pass}\$" -s 3 -c 1 -o /tmp/p_$tag -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --dtype $d --secondary none > gpurun_out/ncu_${tag}.log 2>&1
ncu -i /tmp/p_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${tag}.csv
