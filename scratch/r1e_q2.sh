D=gpurun_out/r1e
mkdir -p $D
python bench.py --config conv-large --no-cpu --no-e2e > $D/bench_conv_q2.json 2> $D/bench_conv_q2.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_quantize -c 20 --csv --log-file $D/launches_conv_q2.csv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_conv_q2.log 2>&1
