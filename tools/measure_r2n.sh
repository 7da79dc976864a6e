set -x
D=gpurun_out/r2n
mkdir -p $D
timeout 300 python tools/timing_overhead.py dct-large 5 > $D/timing_dct.txt 2>&1
timeout 300 python tools/timing_overhead.py conv-large 2 > $D/timing_conv.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $D/launches_dct.csv python bench.py --config dct-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_dct.log 2>&1
ls -la $D
