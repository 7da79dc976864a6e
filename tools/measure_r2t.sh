set -x
D=gpurun_out/r2t
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_baseline_configs_gpu.py -q -m gpu -x -s -k "dct2 or config5" 2>&1 | tail -15 > $D/tests.txt
timeout 600 python bench.py --config dct-large > $D/bench_dct.json 2> $D/bench_dct.err
COFEM_DCT_SMEM=1 timeout 600 python bench.py --config dct-large > $D/bench_dct_old.json 2> $D/bench_dct_old.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $D/launches_dct.csv python bench.py --config dct-large --steps 1 --warmup 1 > $D/ncu.log 2>&1
ls -la $D
