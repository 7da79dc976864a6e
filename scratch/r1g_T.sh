D=gpurun_out/r1g
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -4 > $D/tests_T.txt
python bench.py --no-cpu > $D/bench_dense_T.json 2> $D/bench_dense_T.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"contract_kernel|k_planes" -c 8 --csv --log-file $D/launches_T.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_T.log 2>&1
