#!/bin/bash
# usage (GPU box): tools/gpu_final_r2.sh TAG -- the round's evidence: smoke, full GPU suite, bench (both arms),
# torchrun path, launch lists + per-pass DRAM bytes (c128 / c64), ncu --set full of the heaviest c128 pass
mkdir -p gpurun_out
tag=${1:-r}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > gpurun_out/gpu_$tag.txt
nproc >> gpurun_out/gpu_$tag.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
timeout 2700 python -m pytest tests -q -m gpu --durations=25 > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$tag.log
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/bench_ref_$tag.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_$tag.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_torchrun_$tag.log 2>&1; echo "torchrun rc=$?" >> gpurun_out/bench_torchrun_$tag.log
bash tools/gpu_prof_r2.sh $tag
heavy=${HEAVY:-7}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ptsbe_pass_${heavy}\$" -s 3 -c 1 -o /tmp/full_$tag -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --dtype c128 --secondary none > gpurun_out/ncu_full_$tag.log 2>&1
ncu -i /tmp/full_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_full_raw_$tag.csv 2>/dev/null
ncu -i /tmp/full_$tag.ncu-rep --page details > gpurun_out/ncu_full_details_$tag.txt 2>/dev/null
