#!/bin/bash
# GPU suite + dataset-path timing (tools/dataset_speed.py)
mkdir -p gpurun_out
tag=${1:-r}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 600 python tools/dataset_speed.py 3 256 > gpurun_out/dataset_$tag.log 2>&1
timeout 600 python tools/dataset_speed.py 4 96 >> gpurun_out/dataset_$tag.log 2>&1
nproc >> gpurun_out/dataset_$tag.log
