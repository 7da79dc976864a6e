set -x
D=gpurun_out/r2q
mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1
timeout 1200 python -m pytest tests/test_sharded_gpu.py tests/test_distributed.py tests/test_baseline_configs_gpu.py -q -m gpu -s -k "not config3" 2>&1 | tail -30 > $D/tests.txt
timeout 600 python bench.py --config conv-large > $D/bench_conv.json 2> $D/bench_conv.err
timeout 600 python bench.py --config dct-large > $D/bench_dct.json 2> $D/bench_dct.err
ls -la $D
