set -x
D=gpurun_out/r2al
mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > $D/tests.txt
timeout 600 python bench.py > $D/bench_dense.json 2> $D/bench_dense.err
timeout 600 python bench.py --config conv-large > $D/bench_conv.json 2> $D/bench_conv.err
timeout 600 python bench.py --config dct-large > $D/bench_dct.json 2> $D/bench_dct.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $D/bench_ref.json 2> $D/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_dct-large.csv python bench.py --config dct-large --steps 2 --warmup 1 --no-e2e > $D/ncu.log 2>&1
ls -la $D
