set -x
D=gpurun_out/r2c
mkdir -p $D
timeout 600 python bench.py --precision ozaki24 > $D/bench_dense24.json 2> $D/bench_dense24.err
COFEM_PHASE_DUMP=1 timeout 600 python bench.py --precision ozaki24 --no-cpu --no-e2e --steps 3 > $D/bench_dense24_phase.json 2> $D/bench_dense24_phase.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $D/launches_dense-large24.csv python bench.py --precision ozaki24 --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_dense.log 2>&1
ls -la $D
