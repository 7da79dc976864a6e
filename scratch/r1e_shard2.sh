D=gpurun_out/r1e
mkdir -p $D
timeout 900 python -m pytest tests/test_distributed.py tests/test_sharded_gpu.py -q -x --timeout 400 2>&1 | tail -5 > $D/shard_tests2.txt
python bench.py --config conv-large --no-cpu > $D/bench_conv2.json 2> $D/bench_conv2.err
