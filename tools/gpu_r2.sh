#!/bin/bash
# usage (on the GPU box via gpurun): tools/gpu_r2.sh TAG [tests-expr]
# build + smoke + pytest -m gpu (optionally -k expr) + default bench (c128 headline + c64) + reference arm
mkdir -p gpurun_out
tag=${1:-r}
kexpr=${2:-}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$tag.txt
free -g >> gpurun_out/gpu_$tag.txt; nproc >> gpurun_out/gpu_$tag.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
if [ -n "$kexpr" ]; then
  timeout 1800 python -m pytest tests -q -m gpu -x -k "$kexpr" --durations=15 > gpurun_out/pytest_gpu_$tag.log 2>&1
else
  timeout 1800 python -m pytest tests -q -m gpu -x --durations=25 > gpurun_out/pytest_gpu_$tag.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$tag.log
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/bench_ref_$tag.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_$tag.log
