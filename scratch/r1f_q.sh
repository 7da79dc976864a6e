D=gpurun_out/r1f
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3 > $D/tests_q.txt
python bench.py --config conv-large --no-cpu --no-e2e > $D/bench_conv_q.json 2> $D/bench_conv_q.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_quantize" -c 6 --csv --log-file $D/launches_q.csv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_q.log 2>&1
