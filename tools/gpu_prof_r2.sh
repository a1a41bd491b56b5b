#!/bin/bash
# usage (GPU box): tools/gpu_prof_r2.sh TAG -- launch lists + per-pass DRAM bytes of the bench, c128 and c64
mkdir -p gpurun_out
tag=${1:-r}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
for d in c128 c64; do
  np=$(python -c "
import sys; sys.path.insert(0, '.')
import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import workloads
from paper_2504_16297_b200.program import compile_circuit
c = workloads.build(4, P.parse_circuit, P.parse_noise_model, P.attach_noise)
print(compile_circuit(c, '$d').n_passes)")
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
    --log-file gpurun_out/launches_${d}_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu --dtype $d --secondary none \
    > gpurun_out/ncu_launch_${d}_$tag.log 2>&1
  # every pass launch of a short bench run, with the engine's own log of each launch's
  # algorithmic bytes (same process, same order) -> DRAM traffic / algorithmic bytes
  rm -f gpurun_out/launchlog_${d}_$tag.txt
  PTSBE_LAUNCH_LOG=gpurun_out/launchlog_${d}_$tag.txt timeout 1200 ncu --metrics \
    dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:ptsbe_pass --csv --log-file gpurun_out/pass_dram_${d}_$tag.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --dtype $d --secondary none > gpurun_out/ncu_dram_${d}_$tag.log 2>&1
done
