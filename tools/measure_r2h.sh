set -x
D=gpurun_out/r2h
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "conv or fir or band or smoke" 2>&1 | tail -15 > $D/tests_conv.txt
timeout 600 python bench.py --config conv-large --no-cpu > $D/bench_conv.json 2> $D/bench_conv.err
timeout 600 python bench.py --config conv-large --no-cpu --no-e2e --precision ozaki24 > $D/bench_conv24.json 2> $D/bench_conv24.err
COFEM_CONV_UNFUSED=1 timeout 600 python bench.py --config conv-large --no-cpu --no-e2e > $D/bench_conv_unfused.json 2> $D/bench_conv_unfused.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $D/launches_conv.csv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_conv.log 2>&1
ls -la $D
