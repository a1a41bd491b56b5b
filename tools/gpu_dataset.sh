mkdir -p gpurun_out
timeout 600 python tools/dataset_speed.py 3 256 > gpurun_out/dataset_r1bb.log 2>&1
timeout 600 python tools/dataset_speed.py 4 96 >> gpurun_out/dataset_r1bb.log 2>&1
nproc >> gpurun_out/dataset_r1bb.log
