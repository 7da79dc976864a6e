D=gpurun_out/r1f
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -k "conv or sharded or fresh or distributed" 2>&1 | tail -15 > $D/tests_fu.txt
python bench.py --config conv-large --no-cpu --no-e2e > $D/bench_conv_fu.json 2> $D/bench_conv_fu.err
COFEM_CONV_UNFUSED=1 python bench.py --config conv-large --no-cpu --no-e2e > $D/bench_conv_unfu.json 2> $D/bench_conv_unfu.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $D/launches_fu.csv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_fu.log 2>&1
