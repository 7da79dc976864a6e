D=gpurun_out/r1e
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3 > $D/tests_b3.txt
python bench.py --config conv-large --no-cpu --no-e2e > $D/bench_conv_b3.json 2> $D/bench_conv_b3.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"band_kernel|k_quantize" -c 12 --csv --log-file $D/launches_b3.csv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_b3.log 2>&1
