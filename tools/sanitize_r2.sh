#!/bin/bash
# usage (GPU box): tools/sanitize_r2.sh TAG -- compute-sanitizer memcheck / racecheck / synccheck over:
# generic + generated kernels (config 1/2, config 3 at 20 q incl. c128 TMA staging), sampler (exact
# numpy CDF and fixed point), shared trunk, conventional Algorithm 1, virtual shards (swaps, cross-shard
# norms), the NCCL 1-rank shard group, the device-pointer (host mirror) path
mkdir -p gpurun_out
tag=$1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
sel='config2 or config1 or tiny or uneven or general_channel or permuted or config3_20q or specialised_kernels'
for tool in memcheck racecheck synccheck; do
  log=gpurun_out/sanitize_${tool}_$tag.log
  : > $log
  for spec in "tests/test_gpu_parity.py -k" "tests/test_conventional.py -k" "tests/test_sharded.py -k" "tests/test_pipeline.py -k"; do
    case "$spec" in
      *gpu_parity*) k="$sel";;
      *conventional*) k="not 20_qubits";;
      *sharded*) k="not 28_qubits";;
      *pipeline*) k="device_pointer";;
    esac
    echo "### $tool: $spec \"$k\"" >> $log
    timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 99 \
      python -m pytest $spec "$k" -q -x -m gpu -p no:cacheprovider >> $log 2>&1
    echo "$tool rc=$?" >> $log
  done
done
