#!/bin/bash
# usage (GPU box): tools/ncu_pass_sass.sh TAG PASS [ENV...]  -- full ncu of one pass launch, SASS source page + raw CSV
mkdir -p gpurun_out
tag=$1; pass=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
env "$@" timeout 900 ncu --set full --clock-control none -k regex:"ptsbe_pass_${pass}\$" -s 3 -c 1 -o /tmp/p$pass -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_p${pass}_$tag.log 2>&1
ncu -i /tmp/p$pass.ncu-rep --page source --csv --print-source=sass > gpurun_out/p${pass}_sass_$tag.csv
ncu -i /tmp/p$pass.ncu-rep --page raw --csv > gpurun_out/p${pass}_raw_$tag.csv
