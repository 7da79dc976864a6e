D=gpurun_out/r1e
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -15 > $D/tests_x.txt
python bench.py --config conv-large --no-cpu --no-e2e > $D/bench_conv_x.json 2> $D/bench_conv_x.err
python bench.py --no-cpu --no-e2e > $D/bench_dense_x.json 2> $D/bench_dense_x.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_quantize|k_update|k_direction" -s 20 -c 4 -o $D/full_conv_tail python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncuf_conv_tail.log 2>&1
