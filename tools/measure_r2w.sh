set -x
D=gpurun_out/r2w
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_baseline_configs_gpu.py -q -m gpu -x -s -k "dct2 or config5 or conv" 2>&1 | tail -15 > $D/tests.txt
timeout 600 python bench.py --config dct-large > $D/bench_dct.json 2> $D/bench_dct.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dct_pass --launch-skip 6 -c 3 -o $D/dct python bench.py --config dct-large --steps 1 --warmup 1 > $D/ncu.log 2>&1
ncu -i $D/dct.ncu-rep --page raw --csv > $D/dct_raw.csv 2>/dev/null
ls -la $D
