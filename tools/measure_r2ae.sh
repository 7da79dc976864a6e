set -x
D=gpurun_out/r2ae
mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_baseline_configs_gpu.py -q -m gpu -x -s -k "dct or config5 or staged" 2>&1 | tail -8 > $D/tests.txt
timeout 600 python bench.py --config dct-large --no-cpu > $D/bench_dct.json 2> $D/bench_dct.err
COFEM_DCT_PSI=1 timeout 600 python bench.py --config dct-large --no-cpu > $D/bench_dct_psi.json 2> $D/bench_dct_psi.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $D/launches_dct-large.csv python bench.py --config dct-large --steps 2 --warmup 1 --no-e2e --no-cpu > $D/ncu.log 2>&1
ls -la $D
