D=gpurun_out/r1f
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -4 > $D/tests_x2.txt
python bench.py --config conv-large --no-cpu --no-e2e > $D/bench_conv_x2.json 2> $D/bench_conv_x2.err
python bench.py --no-cpu --no-e2e > $D/bench_dense_x2.json 2> $D/bench_dense_x2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_direction" -c 8 --csv --log-file $D/launches_x2.csv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_x2.log 2>&1
