D=gpurun_out/r1e
mkdir -p $D
timeout 900 python -m pytest tests/test_sharded_gpu.py -q -x --timeout 400 2>&1 | tail -30 > $D/shard_tests.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "conv or fir" 2>&1 | tail -5 >> $D/shard_tests.txt
