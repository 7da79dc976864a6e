D=gpurun_out/r1e
mkdir -p $D
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_quantize" -c 6 --csv --log-file $D/launches_qq.csv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_qq.log 2>&1
