D=gpurun_out/r1e
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3 > $D/tests_aty.txt
python bench.py --config dct-large --no-cpu > $D/bench_dct_aty.json 2> $D/bench_dct_aty.err
python bench.py --config conv-large --no-cpu > $D/bench_conv_aty.json 2> $D/bench_conv_aty.err
