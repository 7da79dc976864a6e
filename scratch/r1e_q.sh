D=gpurun_out/r1e
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -5 > $D/tests_q.txt
python bench.py --config conv-large --no-cpu --no-e2e > $D/bench_conv_q.json 2> $D/bench_conv_q.err
python bench.py --no-cpu --no-e2e > $D/bench_dense_q.json 2> $D/bench_dense_q.err
python bench.py --config dct-large --no-cpu --no-e2e > $D/bench_dct_q.json 2> $D/bench_dct_q.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_conv_q.csv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_conv_q.log 2>&1
