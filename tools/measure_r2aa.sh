set -x
D=gpurun_out/r2aa
mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_baseline_configs_gpu.py -q -m gpu -x -k "dct or config5 or staged" 2>&1 | tail -5 > $D/tests.txt
timeout 600 python bench.py --config dct-large > $D/bench_dct.json 2> $D/bench_dct.err
timeout 600 python bench.py --config dct-large > $D/bench_dct_b.json 2> $D/bench_dct_b.err
ls -la $D
