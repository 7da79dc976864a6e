D=gpurun_out/r1k
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -12 > $D/tests.txt
python bench.py --no-cpu --no-e2e > $D/bench_dense.json 2> $D/bench_dense.err
COFEM_NO_SPLIT_FIXUP=1 python bench.py --no-cpu --no-e2e > $D/bench_dense_nofix.json 2> $D/bench_dense_nofix.err
python bench.py --no-cpu --no-e2e > $D/bench_dense2.json 2> $D/bench_dense2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu.log 2>&1
