D=gpurun_out/r1i_q
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -3 > $D/tests.txt
python bench.py --config conv-large --no-cpu --no-e2e > $D/bench_conv.json 2> $D/bench_conv.err
python bench.py --no-cpu --no-e2e > $D/bench_dense.json 2> $D/bench_dense.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_quantize" -c 6 --csv --log-file $D/launches_q.csv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_q.log 2>&1
