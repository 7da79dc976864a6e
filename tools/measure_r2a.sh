set -x
D=gpurun_out/r2a
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $D/smi.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x 2>&1 | tail -30 > $D/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1
timeout 600 python bench.py > $D/bench_dense.json 2> $D/bench_dense.err
COFEM_NO_PERSISTENT=1 timeout 600 python bench.py --no-cpu --no-e2e > $D/bench_dense_multi.json 2> $D/bench_dense_multi.err
timeout 600 python bench.py --config conv-large --no-cpu > $D/bench_conv.json 2> $D/bench_conv.err
timeout 600 python bench.py --config dct-large --no-cpu > $D/bench_dct.json 2> $D/bench_dct.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $D/launches_dense-large.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_dense.log 2>&1
ls -la $D
