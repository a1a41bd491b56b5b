#!/bin/bash
# usage (GPU box): tools/sanitize.sh TAG -- compute-sanitizer memcheck / racecheck / synccheck on small GPU
# parity cases (generic kernel: 10 q config 1; generated kernels: 17 q config 2; sampler; shared trunk)
mkdir -p gpurun_out
tag=$1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
sel='config2 or config1 or tiny or uneven or general_channel or permuted'
for tool in memcheck racecheck synccheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 99 \
    python -m pytest tests/test_gpu_parity.py -q -x -k "$sel" > gpurun_out/sanitize_${tool}_$tag.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_${tool}_$tag.log
done
