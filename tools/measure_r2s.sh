set -x
D=gpurun_out/r2s
mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -30 > $D/tests.txt
timeout 600 python bench.py > $D/bench_dense.json 2> $D/bench_dense.err
timeout 600 python bench.py --config conv-large > $D/bench_conv.json 2> $D/bench_conv.err
timeout 600 python bench.py --config dct-large > $D/bench_dct.json 2> $D/bench_dct.err
ls -la $D
