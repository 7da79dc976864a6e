D=gpurun_out/r1e
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3 > $D/tests_e16.txt
python bench.py --config conv-large --no-cpu --no-e2e > $D/bench_conv_e16.json 2> $D/bench_conv_e16.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"band_kernel" -c 6 --csv --log-file $D/launches_e16.csv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_e16.log 2>&1
