#!/bin/bash
# usage (on the GPU box via gpurun): tools/gpu_round.sh TAG [ncu]
# smoke + pytest -m gpu + bench + reference arm (+ ncu launch list of the bench and one
# --set full capture of every pass kernel of one step, exported as raw CSV)
mkdir -p gpurun_out
tag=${1:-r}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$tag.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$tag.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$tag.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_$tag.log
if [ "$2" = "ncu" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch_$tag.log 2>&1
  timeout 1500 ncu --set full --clock-control none -k regex:ptsbe_pass -s 36 -c 12 -o /tmp/pass_$tag -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full_$tag.log 2>&1
  ncu -i /tmp/pass_$tag.ncu-rep --page raw --csv > gpurun_out/pass_raw_$tag.csv
  timeout 900 ncu --set full --clock-control none -k regex:sample_blocksum -s 3 -c 1 -o /tmp/bs_$tag -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_bs_$tag.log 2>&1
  ncu -i /tmp/bs_$tag.ncu-rep --page raw --csv > gpurun_out/blocksum_raw_$tag.csv
fi
