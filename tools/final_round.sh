bash tools/gpu_round.sh r1az ncu
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:ptsbe_pass -s 36 -c 12 --csv --log-file gpurun_out/pass_dram_r1az.csv python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
