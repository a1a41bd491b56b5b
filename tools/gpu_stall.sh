#!/bin/bash
# usage (GPU box): tools/gpu_stall.sh TAG PASS -- c128 bench line + ncu --set full of one pass kernel with
# per-SASS-instruction stall samples (source page), to locate the heavy passes' stall sites
mkdir -p gpurun_out
tag=${1:-r}; pass=${2:-5}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 600 python bench.py --dtype c128 --secondary none --no-cpu > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$tag.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ptsbe_pass_${pass}\$" -s 3 -c 1 -o /tmp/st_$tag -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --dtype c128 --secondary none > gpurun_out/ncu_st_$tag.log 2>&1
ncu -i /tmp/st_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_st_raw_$tag.csv 2>/dev/null
ncu -i /tmp/st_$tag.ncu-rep --page details > gpurun_out/ncu_st_details_$tag.txt 2>/dev/null
ncu -i /tmp/st_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_st_sass_$tag.csv 2>gpurun_out/ncu_st_sass_err_$tag.txt
